// fast_kernels.cuh -- host glue of the specialised hot path.
//
// The fused7 kernel (fused7.cuh) serves time-shear / separable lattices with p = 1, q = 4,
// d = M in {256, 512}, complex64 (BASELINE configs 3 and 5).  This file decides whether a
// plan qualifies (checking on the host, exactly, every identity the kernel relies on), builds
// the plan-time window table G', sizes the ring of intermediate slots and the look-ahead,
// and launches the persistent kernel.  Every other lattice runs the generic kernels of dgt.cu.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include <cudaTypedefs.h>

#include "../../include/nsdgt.h"
#include "cplx.cuh"
#include "fused7.cuh"
#include "fused7_adj.cuh"
#include "fused8.cuh"

namespace nsdgt {

template <typename T>
__global__ void k_window_factor(cx<T>* G, const double2* gt, int64_t L, int64_t c, int64_t d, int64_t p, int64_t q);

struct FastPlan {
    int kind = 0;  // 0 = none (generic path); 2 = fused persistent kernel (fused8, or fused7)
    int xdb = 0;   // fused7t: double-buffered exchange (NSDGT_XDB=1)
    int early = 0; // fused7 D = 512: half-tile-early prefetch (NSDGT_EARLY=1)
    int gpersist = 0;   // experiment: G' in a persisting L2 access-policy window (NSDGT_GPERSIST=1)
    int cst = 0;        // fused7: TMA coefficient stores (NSDGT_CST=1; measured slower, off by default)
    int ver = 7;   // forward kernel: 7 = fused7 (default), 9 = fused7t (TMA tile loads), 8 = fused8 (NSDGT_FUSED)
    const char* name = "none";
    int D = 0, MM = 0, Q = 0, c = 0, N = 0;
    int64_t L = 0;
    int nA = 0, nB = 0;          // A jobs (8 columns j) and B jobs (16 columns n) per signal
    int grid = 0;                // persistent grid: CTAs per SM (occupancy) x SMs
    size_t smem = 0;
    size_t esz = 8;
    int Kmod = 0, beta = 0;      // chirp rate K mod D, rotation slope beta (fused7.cuh header)
    int S = 8, lag = 5;          // ring slots, look-ahead (signals)
    int minb = 3;                // CTAs per SM the kernel is compiled for
    const void* E = nullptr;     // Alg. 1 column phases (plan-owned)
    void* Gp = nullptr;          // G' (owned)
    void* Gpa = nullptr;         // G' in the adjoint kernel's order (owned)
    size_t smem_adj = 0;
    int grid_adj = 0, lag_adj = 0;   // synthesis kernel grid and look-ahead
    int grid_real = 0;               // real-input forward kernel grid
    int dbg = 0;                 // experiment knobs (NSDGT_DBG, read once at plan time; fused7.cuh)
    unsigned long long* tracelog = nullptr;   // dbg & 16: per-CTA phase stamps of a -DNSDGT_TRACE build
    int* counters = nullptr;     // job queue + per-slot completion counters (owned)
};

template <int D, int MINB>
static void launch7(const v7::Args& a, const CUtensorMap& cm, int grid, size_t smem, cudaStream_t st) {
    v7::fused7_kernel<D, MINB><<<grid, v7::Cfg<D>::NT, smem, st>>>(a, cm);
}
static void launch7e(const v7::Args& a, const CUtensorMap& cm, int grid, size_t smem, cudaStream_t st) {
    v7::fused7_kernel<512, 3, true, false, true><<<grid, v7::Cfg<512>::NT, smem, st>>>(a, cm);
}
// TMA coefficient stores (the default occupancy)
template <int D, int MINB>
static void launch7c(const v7::Args& a, const CUtensorMap& cm, int grid, size_t smem, cudaStream_t st) {
    v7::fused7_kernel<D, MINB, (MINB <= 3), false, false, true><<<grid, v7::Cfg<D>::NT, smem, st>>>(a, cm);
}
// real input (promoted on load): the default CTAs-per-SM variants only
template <int D, int MINB>
static void launch7r(const v7::Args& a, const CUtensorMap& cm, int grid, size_t smem, cudaStream_t st) {
    v7::fused7_kernel<D, MINB, (MINB <= 3), true><<<grid, v7::Cfg<D>::NT, smem, st>>>(a, cm);
}
// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
    }
    return fn;
}
// 2-D map over a row-major array of 8-byte elements: cols x rows, row pitch in bytes, boxes of
// box_cols x box_rows
static bool encode_map_2d(CUtensorMap* m, const void* base, uint64_t cols, uint64_t rows, uint64_t pitch,
                          uint32_t box_cols, uint32_t box_rows) {
    auto fn = tensor_map_encoder();
    if (!fn) return false;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {pitch};
    cuuint32_t box[2] = {box_cols, box_rows};
    cuuint32_t es[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, const_cast<void*>(base), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// 3-D map over the coefficients c[W][M][N] viewed as [W M / R1][R1][N] (m = R1 (m div R1) +
// m mod R1): boxes of 8 columns x 16 rows m mod R1 x 16 rows m div R1 -- one exchange round
// of a B tile (CST)
static bool encode_cmap(CUtensorMap* m, const void* c, int64_t W, int64_t M, int64_t N, int64_t R1) {
    auto fn = tensor_map_encoder();
    if (!fn) return false;
    cuuint64_t dims[3] = {(cuuint64_t)N, (cuuint64_t)R1, (cuuint64_t)(W * M / R1)};
    cuuint64_t strides[2] = {(cuuint64_t)N * 8, (cuuint64_t)R1 * N * 8};
    cuuint32_t box[3] = {8, 16, 16};
    cuuint32_t es[3] = {1, 1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, const_cast<void*>(c), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
template <int D, int MINB, bool XDB = false>
static void launch7t(const v7::Args& a, const v7::Maps& m, int grid, size_t smem, cudaStream_t st) {
    v7::fused7t_kernel<D, MINB, XDB><<<grid, v7::Cfg<D>::NT, smem, st>>>(a, m);
}
template <int D, int MINB, bool REAL = false>
static void launch8(const v7::Args& a, int grid, size_t smem, cudaStream_t st) {
    v8::fused8_kernel<D, MINB, REAL><<<grid, v8::Cfg<D>::NT, smem, st>>>(a);
}
template <int D, int MINB>
static void launch7a(const v7::Args& a, int grid, size_t smem, cudaStream_t st) {
    v7::fused7a_kernel<D, MINB><<<grid, v7::Cfg<D>::NT, smem, st>>>(a);
}

// Decide and build.  Returns DGT_OK with fp->kind == 0 when the lattice does not qualify.
template <typename T>
int build_fast(FastPlan* fp, const dgt_lattice_info& I, const double2* gt, const void* E, bool force_generic,
               cudaStream_t st) {
    fp->kind = 0;
    fp->name = "none";
    if (force_generic) return DGT_OK;
    if constexpr (!std::is_same<T, float>::value) return DGT_OK;
    if (I.branch == DGT_BRANCH_FREQ || I.p != 1 || I.q != 4 || I.d != I.iM || (I.d != 512 && I.d != 256)) return DGT_OK;
    if (I.c % 16 != 0 || I.N % 16 != 0 || I.iM != I.M || I.N != I.q * I.d) return DGT_OK;
    const int64_t L = I.L, twoL = 2 * L, D = I.d, M = I.M, Q = I.q, N = I.N;
    const int64_t sigma = ((I.chirp_sigma % twoL) + twoL) % twoL;
    const int64_t K = (int64_t)((unsigned __int128)sigma * (unsigned __int128)((L + 1) % twoL) % (unsigned __int128)twoL);
    if (((unsigned __int128)K * ((unsigned __int128)M * M % twoL)) % twoL != 0) return DGT_OK;  // R(s) == 1 required
    // rotation identity rot(n(tau)) = alpha_{l,u} - beta tau (mod M), n(tau) = (l - u - q tau) mod N,
    // verified for every (l, u, tau) with the same integer formula the generic path uses
    if ((I.s1 * I.a * Q) % I.b != 0) return DGT_OK;
    const int64_t beta = ((I.s1 * I.a * Q / I.b) % M + M) % M;
    auto rotm = [&](int64_t n) {
        const __int128 x = (__int128)I.s1 * I.a * n;
        const int64_t r = (int64_t)(((x + I.b - 1) / I.b) % M);
        return ((r % M) + M) % M;
    };
    v7::GpArgs ga{};
    for (int l = 0; l < Q; ++l)
        for (int u = 0; u < Q; ++u) {
            const int64_t alpha = rotm((((l - u) % N) + N) % N);
            ga.alpha[l * Q + u] = (int)alpha;
            for (int64_t tau = 0; tau < D; ++tau) {
                const int64_t n = (((l - u - Q * tau) % N) + N) % N;
                if (rotm(n) != (((alpha - beta * tau) % M) + M) % M) return DGT_OK;
            }
        }
    // kernel variant: CTAs per SM, measured best 3 for D = 512 (more CTAs leave too little L1
    // next to 3 x 53 KB of shared memory: the ring stores use it), 5 for D = 256 (36 KB, 91
    // registers).  NSDGT_CTAS overrides (experiments).
    fp->ver = 7;
    if (const char* e = std::getenv("NSDGT_FUSED")) {
        const int v = std::atoi(e);
        fp->ver = (v == 7 || v == 9) ? v : 8;
    }
    const bool v8k = fp->ver == 8;
    fp->xdb = (fp->ver == 9 && std::getenv("NSDGT_XDB") && std::atoi(std::getenv("NSDGT_XDB"))) ? 1 : 0;
    int minb = v8k ? 2 : D == 512 ? 3 : 5;
    if (const char* e = std::getenv("NSDGT_CTAS"))
        minb = v8k ? std::max(2, std::min(D == 512 ? 2 : 3, std::atoi(e))) : std::max(3, std::min(D == 512 ? 4 : 5, std::atoi(e)));
    fp->early = (fp->ver == 7 && D == 512 && minb == 3 && std::getenv("NSDGT_EARLY") && std::atoi(std::getenv("NSDGT_EARLY"))) ? 1 : 0;
    fp->cst = (fp->ver == 7 && !fp->early && D == 512 && minb == 3 &&
               std::getenv("NSDGT_CST") && std::atoi(std::getenv("NSDGT_CST"))) ? 1 : 0;
    if (fp->cst && cudaFuncSetAttribute((const void*)v7::fused7_kernel<512, 3, true, false, false, true>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)v7::Cfg<512>::SMEM) != cudaSuccess)
        return DGT_ECUDA;
    if (fp->early &&
        cudaFuncSetAttribute((const void*)v7::fused7_kernel<512, 3, true, false, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)v7::Cfg<512>::SMEM) != cudaSuccess)
        return DGT_ECUDA;
    {
        const void* ka = D == 512 ? (const void*)v7::fused7a_kernel<512, 3> : (const void*)v7::fused7a_kernel<256, 5>;
        const size_t sm = D == 512 ? v7::Cfg<512>::SMEM : v7::Cfg<256>::SMEM;
        if (cudaFuncSetAttribute(ka, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess) return DGT_ECUDA;
        fp->smem_adj = sm;
    }
    const void* kfn = v8k ? (D == 512   ? (const void*)v8::fused8_kernel<512, 2>
                             : minb == 3 ? (const void*)v8::fused8_kernel<256, 3>
                                         : (const void*)v8::fused8_kernel<256, 2>)
                      : fp->ver == 9 && fp->xdb ? (D == 512 ? (const void*)v7::fused7t_kernel<512, 3, true>
                                                            : (const void*)v7::fused7t_kernel<256, 4, true>)
                      : fp->ver == 9 ? (D == 512 ? (minb == 4 ? (const void*)v7::fused7t_kernel<512, 4>
                                                              : (const void*)v7::fused7t_kernel<512, 3>)
                                                 : (minb == 5 ? (const void*)v7::fused7t_kernel<256, 5>
                                                              : (const void*)v7::fused7t_kernel<256, 4>))
                      : D == 512 ? (minb == 4 ? (const void*)v7::fused7_kernel<512, 4> : (const void*)v7::fused7_kernel<512, 3>)
                                 : (minb == 5   ? (const void*)v7::fused7_kernel<256, 5>
                                    : minb == 4 ? (const void*)v7::fused7_kernel<256, 4>
                                                : (const void*)v7::fused7_kernel<256, 3>);
    const size_t smem = v8k ? (D == 512 ? v8::Cfg<512>::SMEM : v8::Cfg<256>::SMEM)
                            : (D == 512 ? v7::Cfg<512>::SMEM + (fp->xdb ? v7::Cfg<512>::XE * 8 : 0)
                                        : v7::Cfg<256>::SMEM + (fp->xdb ? v7::Cfg<256>::XE * 8 : 0));
    const int nthreads = v8k ? v8::Cfg<512>::NT : v7::Cfg<512>::NT;
    if (cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return DGT_ECUDA;
    int per_sm = 0, dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, nthreads, smem) != cudaSuccess || per_sm < 1)
        return DGT_OK;   // cannot host the persistent kernel: generic path
    // persistent kernel: every CTA must be resident (the occupancy query bounds the grid)
    if (const char* e = std::getenv("NSDGT_PER_SM")) per_sm = std::max(1, std::min(per_sm, std::atoi(e)));
    // fp64 window factors G64[(r q + u) d + nu] = conj(Gamma)/d, then G' (fused7.cuh)
    double2* G64 = nullptr;
    if (cudaMalloc(&G64, sizeof(double2) * L) != cudaSuccess) return DGT_ENOMEM;
    k_window_factor<double><<<(unsigned)std::min<int64_t>((L + 255) / 256, 148 * 64), 256, 0, st>>>(G64, gt, L, I.c, I.d, 1, Q);
    if (cudaMalloc(&fp->Gp, sizeof(float2) * (size_t)M * Q * D) != cudaSuccess) { cudaFree(G64); return DGT_ENOMEM; }
    ga.Gp = (float4*)fp->Gp; ga.G64 = G64; ga.L = L; ga.K = K;
    ga.M = (int)M; ga.D = (int)D; ga.Q = (int)Q; ga.c = (int)I.c; ga.beta = (int)beta; ga.R1 = (int)(D / 16);
    ga.layout = 0;
    if (v8k) v8::k_gprime8<<<(unsigned)std::min<int64_t>((M * Q * D + 255) / 256, 148 * 64), 256, 0, st>>>(ga);
    else v7::k_gprime<<<(unsigned)std::min<int64_t>((M * Q * D + 255) / 256, 148 * 64), 256, 0, st>>>(ga);
    // the same table in the synthesis kernel's order
    if (cudaMalloc(&fp->Gpa, sizeof(float2) * (size_t)M * Q * D) != cudaSuccess) { cudaFree(G64); return DGT_ENOMEM; }
    ga.Gp = (float4*)fp->Gpa;
    ga.layout = 1;
    v7::k_gprime<<<(unsigned)std::min<int64_t>((M * Q * D + 255) / 256, 148 * 64), 256, 0, st>>>(ga);
    const cudaError_t err = cudaStreamSynchronize(st);
    cudaFree(G64);
    if (err != cudaSuccess) return DGT_ECUDA;
    fp->minb = minb;
    fp->grid = per_sm * sms;
    fp->smem = smem;
    fp->D = (int)D; fp->MM = (int)M; fp->Q = (int)Q; fp->c = (int)I.c; fp->N = (int)N; fp->L = L;
    fp->nA = (int)(M / (v8k ? v8::Cfg<512>::ACOL : v7::Cfg<512>::ACOL));
    fp->nB = (int)(N / 16);
    fp->Kmod = (int)(K % D);
    fp->beta = (int)beta;
    // Look-ahead: B(w) is queued lag signals after A(w).  An A job spans several tiles, so about
    // 3 x (CTAs / jobs per signal) signals of look-ahead hide the A -> B dependency; the ring
    // (S signals of intermediate) is capped at ~80 MB so that it stays mostly in L2, with
    // 4 + lag/2 slots beyond the look-ahead where it fits (config 5: S = 10, lag = 6, 5.78 ms;
    // the earlier 64 MB cap gave S = 8, lag = 5, 5.91 ms).
    {
        const int jps = fp->nA + fp->nB;
        const size_t per_sig = (size_t)M * Q * D * sizeof(float2);
        const int smax = std::max(6, (int)((80ull << 20) / per_sig));
        fp->lag = std::max(2, std::min(smax - 4, (3 * fp->grid + jps / 2) / jps));
        fp->S = std::min(smax, fp->lag + 4 + fp->lag / 2);   // config 3: S = 38 (0.341 ms; 31: 0.354)
    }
    if (const char* e = std::getenv("NSDGT_S")) fp->S = std::max(1, std::atoi(e));
    if (const char* e = std::getenv("NSDGT_LAG")) fp->lag = std::max(0, std::atoi(e));
    if (fp->lag >= fp->S) fp->lag = fp->S - 1;
    if (std::getenv("NSDGT_VERBOSE"))
        std::fprintf(stderr, "fused%d: D=%d CTAs/SM=%d grid=%d smem/CTA=%zu B ring S=%d lag=%d\n", fp->ver, (int)D, per_sm,
                     fp->grid, smem, fp->S, fp->lag);
    // job queue + per-slot completion counters (allocated here: execute allocates nothing)
    if (cudaMalloc(&fp->counters, sizeof(int) * (1 + 2 * fp->S)) != cudaSuccess) return DGT_ENOMEM;
    // Synthesis (fused7_adj.cuh): B' jobs are short (2 tiles) and the long A' jobs (5 tiles)
    // free the ring slots, so A'(w) needs less lag behind B'(w) than fused7's B behind A, and a
    // shorter lag leaves more slots between B'(w) and the A'(w - S) it waits for.  Measured:
    // config 5 lag 2 (S = 8) 6.24 ms against 8.07 ms at fused7's lag 5; config 3 lag 6 (S = 20)
    // 0.39 ms against 0.48 ms at lag 14.  Its grid: every CTA resident (occupancy query).
    fp->lag_adj = std::max(1, std::min(fp->S - 1, (2 * fp->lag + 2) / 5));
    if (const char* e = std::getenv("NSDGT_LAG_ADJ")) fp->lag_adj = std::max(0, std::min(fp->S - 1, std::atoi(e)));
    {
        int per_sm_a = 0;
        const void* ka = D == 512 ? (const void*)v7::fused7a_kernel<512, 3> : (const void*)v7::fused7a_kernel<256, 5>;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_a, ka, v7::Cfg<512>::NT, fp->smem_adj) != cudaSuccess ||
            per_sm_a < 1)
            return DGT_ECUDA;
        fp->grid_adj = v8k ? per_sm_a * sms : std::min(per_sm * sms, per_sm_a * sms);
    }
    {   // real-input variant (default occupancy): attribute + resident grid
        const void* kr = v8k ? (D == 512 ? (const void*)v8::fused8_kernel<512, 2, true>
                                         : (const void*)v8::fused8_kernel<256, 2, true>)
                             : D == 512 ? (const void*)v7::fused7_kernel<512, 3, true, true>
                                        : (const void*)v7::fused7_kernel<256, 5, false, true>;
        int per_sm_r = 0;
        if (cudaFuncSetAttribute(kr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess ||
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_r, kr, nthreads, smem) != cudaSuccess ||
            per_sm_r < 1)
            return DGT_ECUDA;
        fp->grid_real = std::min(per_sm * sms, per_sm_r * sms);
    }
    fp->dbg = std::getenv("NSDGT_DBG") ? std::atoi(std::getenv("NSDGT_DBG")) : 0;   // experiment knobs
    fp->gpersist = std::getenv("NSDGT_GPERSIST") ? std::atoi(std::getenv("NSDGT_GPERSIST")) : 0;
    if (fp->gpersist) cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)M * Q * D * 8);
    if (fp->dbg & 16) {   // phase trace of a -DNSDGT_TRACE build (tools/v7trace.py, dgt_debug_trace_log)
        if (cudaMalloc(&fp->tracelog, sizeof(unsigned long long) * 8 * 4096) != cudaSuccess) return DGT_ENOMEM;
    }
    fp->E = E;
    fp->esz = sizeof(float2);
    fp->kind = 2;
    fp->name = v8k ? "fused8_t_p1" : fp->ver == 9 ? "fused7t_t_p1" : "fused7_t_p1";
    return DGT_OK;
}

inline void free_fast(FastPlan* fp) {
    if (fp->tracelog) cudaFree(fp->tracelog);
    fp->tracelog = nullptr;
    if (fp->Gp) cudaFree(fp->Gp);
    if (fp->Gpa) cudaFree(fp->Gpa);
    fp->Gpa = nullptr;
    if (fp->counters) cudaFree(fp->counters);
    fp->Gp = nullptr;
    fp->counters = nullptr;
}

// ring of S intermediate slots
inline size_t fast_workspace_bytes(const FastPlan* fp, int64_t /*Wc*/) {
    return (size_t)fp->S * fp->MM * fp->Q * fp->D * fp->esz;
}

// the fused kernel consumes the whole batch in one launch
// (the kernel's 32-bit job indices bound one launch to W (nA + nB) < 2^31 signals' jobs)
inline int64_t fast_chunk(const FastPlan* fp) { return (((int64_t)1 << 31) - 1) / (fp->nA + fp->nB); }
inline int64_t fast_launches_per_chunk(const FastPlan*) { return 1; }

template <typename T>
int launch_fast(FastPlan* fp, const void* f, int real_in, void* ws, void* c, int64_t W, cudaStream_t st) {
    if (fp->kind != 2) return DGT_EUNSUPPORTED;
    if (W * (int64_t)(fp->nA + fp->nB) >= (int64_t)1 << 31) return DGT_EUNSUPPORTED;   // 32-bit job indices
    const int nctr = 1 + 2 * fp->S;
    if (!fp->counters) return DGT_EINVAL;   // allocated by build_fast
    if (cudaMemsetAsync(fp->counters, 0, sizeof(int) * nctr, st) != cudaSuccess) return DGT_ECUDA;
    v7::Args a{};
    a.f = (const float2*)f; a.out = (float2*)c; a.ws = (float2*)ws; a.Gp = (const float4*)fp->Gp;
    a.E = (const float2*)fp->E; a.ctr = fp->counters; a.W = (int)W; a.N = fp->N; a.c = fp->c; a.Kmod = fp->Kmod;
    a.beta = fp->beta; a.S = fp->S; a.lag = fp->lag; a.nA = fp->nA; a.nB = fp->nB;
    a.sig0 = ((fp->beta - fp->Kmod) & (fp->D - 1)) == 0 ? 1 : 0;
    a.dbg = fp->dbg;
    if (fp->tracelog) {
        cudaMemsetAsync(fp->tracelog, 0, sizeof(unsigned long long) * 8 * 4096, st);
        a.log = fp->tracelog;
    }
    if (fp->gpersist) {   // experiment: keep G' resident (the ring and c stream normally)
        cudaStreamAttrValue v{};
        v.accessPolicyWindow.base_ptr = fp->Gp;
        v.accessPolicyWindow.num_bytes = (size_t)fp->MM * fp->Q * fp->D * 8;
        v.accessPolicyWindow.hitRatio = 1.0f;
        v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &v);
    }
    if (fp->ver == 9 && !real_in) {
        v7::Maps m;
        const int64_t D = fp->D, M = fp->MM, Q = fp->Q;
        if (!encode_map_2d(&m.f, f, (uint64_t)M, (uint64_t)(W * D), (uint64_t)M * 8, 8, 256) ||
            !encode_map_2d(&m.ws, ws, (uint64_t)(Q * D), (uint64_t)fp->S * M, (uint64_t)Q * D * 8, 8, 256))
            return DGT_ECUDA;
        if (fp->xdb) (fp->D == 512 ? launch7t<512, 3, true> : launch7t<256, 4, true>)(a, m, fp->grid, fp->smem, st);
        else if (fp->D == 512) (fp->minb == 4 ? launch7t<512, 4> : launch7t<512, 3>)(a, m, fp->grid, fp->smem, st);
        else (fp->minb == 5 ? launch7t<256, 5> : launch7t<256, 4>)(a, m, fp->grid, fp->smem, st);
    } else if (fp->ver == 8) {
        if (real_in) {
            if (fp->D == 512) launch8<512, 2, true>(a, fp->grid_real, fp->smem, st);
            else launch8<256, 2, true>(a, fp->grid_real, fp->smem, st);
        } else if (fp->D == 512) {
            launch8<512, 2>(a, fp->grid, fp->smem, st);
        } else {
            (fp->minb == 3 ? launch8<256, 3> : launch8<256, 2>)(a, fp->grid, fp->smem, st);
        }
    } else {
        CUtensorMap cm{};
        const bool cst = fp->cst && !real_in;
        if (cst && !encode_cmap(&cm, c, W, fp->MM, fp->N, fp->D / 16)) return DGT_ECUDA;
        if (real_in) {   // the real variants are compiled for the default occupancy only
            if (fp->D == 512) launch7r<512, 3>(a, cm, fp->grid_real, fp->smem, st);
            else launch7r<256, 5>(a, cm, fp->grid_real, fp->smem, st);
        } else if (cst) {
            launch7c<512, 3>(a, cm, fp->grid, fp->smem, st);
        } else if (fp->D == 512) {
            if (fp->early) launch7e(a, cm, fp->grid, fp->smem, st);
            else (fp->minb == 4 ? launch7<512, 4> : launch7<512, 3>)(a, cm, fp->grid, fp->smem, st);
        } else {
            (fp->minb == 5 ? launch7<256, 5> : fp->minb == 4 ? launch7<256, 4> : launch7<256, 3>)(a, cm, fp->grid, fp->smem, st);
        }
    }
    if (fp->gpersist) {
        cudaStreamAttrValue v{};
        v.accessPolicyWindow.num_bytes = 0;
        cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &v);
    }
    return DGT_OK;
}

// synthesis (fused7_adj.cuh): c (device, W x M x N) -> f (device, W x L), the ring as workspace.
// The grid is the forward kernel's: 3 CTAs/SM for D = 512, 5 for D = 256 (both kernels use the
// same shared memory and fewer registers for the adjoint; the occupancy query checks it).
inline int launch_fast_adj(FastPlan* fp, const void* c, void* ws, void* f, int64_t W, cudaStream_t st) {
    if (fp->kind != 2) return DGT_EUNSUPPORTED;
    if (W * (int64_t)(fp->nA + fp->nB) >= (int64_t)1 << 31) return DGT_EUNSUPPORTED;
    const int nctr = 1 + 2 * fp->S;
    if (!fp->counters) return DGT_EINVAL;   // allocated by build_fast
    if (cudaMemsetAsync(fp->counters, 0, sizeof(int) * nctr, st) != cudaSuccess) return DGT_ECUDA;
    v7::Args a{};
    a.f = (const float2*)c; a.out = (float2*)f; a.ws = (float2*)ws; a.Gp = (const float4*)fp->Gpa;
    a.E = (const float2*)fp->E; a.ctr = fp->counters; a.W = (int)W; a.N = fp->N; a.c = fp->c; a.Kmod = fp->Kmod;
    a.beta = fp->beta; a.S = fp->S; a.lag = fp->lag; a.nA = fp->nA; a.nB = fp->nB;
    a.lag = fp->lag_adj;
    a.dbg = fp->dbg;
    const int grid = fp->grid_adj;
    if (fp->D == 512) launch7a<512, 3>(a, grid, fp->smem_adj, st);
    else launch7a<256, 5>(a, grid, fp->smem_adj, st);
    return DGT_OK;
}

}  // namespace nsdgt
