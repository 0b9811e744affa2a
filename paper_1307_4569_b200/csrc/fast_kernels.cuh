// fast_kernels.cuh -- the specialised hot path.
//
// One persistent kernel per execute for the time-shear / separable branch with p = 1
// (BASELINE configs 3 and 5): every CTA loops over a global job queue holding two job
// kinds per signal w,
//   A(w, rg): Zak columns j = 4rg+rho + c*l (rho<4, l<q) -> DFT_d over s (the Zak DFT),
//             chirp by factorisation, products with the window factors, DFT_d over nu,
//             -> intermediate C(j, n) in an L2-resident ring of S signal slots;
//   B(w, t) : 16 consecutive columns n of C -> M-point FFT over j, Alg. 1 phase E(n) and
//             row rotation, coalesced streaming stores of c[w][m][n].
// Jobs are dequeued in an order where every dependency (B(w) on all A(w); A(w) on all
// B(w-S) before reusing the slot) was dequeued earlier, so spinning on the per-signal
// counters cannot deadlock (all CTAs are co-resident: grid = occupancy x SM count).
//
// FFTs are warp-level, register resident: N = 32*E points, lane t holds x[t + 32k];
// pass 1 = DFT-E in registers + twiddle W_N^{t k1}; one shared-memory exchange; pass 2 =
// DFT-E in registers + twiddle W_32^{h k'} + a cross-lane DFT-(32/E) with shuffles.
//
// Chirp by factorisation (T-branch, p = 1, x = j + s M, L = d M):
//   P_sigma(j + sM) = C(j) R(s) exp(2 pi i (K j mod d) s / d),  K = sigma (L+1) mod 2L,
//   C(j) = exp(i pi (K j^2 mod 2L)/L),  R(s) = exp(i pi (K s^2 M^2 mod 2L)/L),
// so DFT_s[P f](nu, j) = C(j) DFT_s[R f](nu - K j mod d, j): a column phase and a cyclic
// index shift, no per-sample sincos.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <type_traits>

#include "../../include/nsdgt.h"
#include "cplx.cuh"
#include "fft_smem.cuh"

namespace nsdgt {

// ------------------------------------------------------------------------------------
// warp FFT, N = 32*E, forward (exp(-2 pi i jk/N))
// ------------------------------------------------------------------------------------
template <int E> struct WarpFftShape {
    static constexpr int N = 32 * E;
    static constexpr int H = 32 / E;
    static constexpr int SROW = (E == 16) ? 33 : 36;  // padded scratch row (bank-conflict free)
    static constexpr int SCRATCH = E * SROW;           // complex elements per warp
};

template <typename T, int E>
struct WarpFft {
    using S = WarpFftShape<E>;
    cx<T> tw1[E];  // W_N^{lane*k1}
    cx<T> tw2[E];  // W_32^{h*k'}, h = lane / E

    __device__ __forceinline__ void init(int lane) {
        const int h = lane / E;
#pragma unroll
        for (int k = 0; k < E; ++k) {
            double s, c;
            sincospi(-2.0 * (double)((lane * k) % S::N) / (double)S::N, &s, &c);
            tw1[k] = mk<T>((T)c, (T)s);
            sincospi(-2.0 * (double)((h * k) % 32) / 32.0, &s, &c);
            tw2[k] = mk<T>((T)c, (T)s);
        }
    }
    // output index j-block of this lane (cross-lane DFT-H leaves outputs bit reversed)
    static __device__ __forceinline__ int out_jo(int lane) {
        const int h = lane / E;
        if constexpr (S::H == 4) return ((h & 1) << 1) | (h >> 1);
        else return h;
    }
    // v[k] = x[lane + 32k] on entry.  On exit v[k'] = X[k1 + E k' + E^2 jo], lane = k1 + E h.
    __device__ __forceinline__ void run(cx<T>* v, cx<T>* scr, int lane) const {
        dft_fixed<T, E>(v);
#pragma unroll
        for (int k = 1; k < E; ++k) v[k] = cmul(v[k], tw1[k]);
#pragma unroll
        for (int k = 0; k < E; ++k) scr[k * S::SROW + lane] = v[k];
        __syncwarp();
        const int k1 = lane % E, h = lane / E;
#pragma unroll
        for (int m = 0; m < E; ++m) v[m] = scr[k1 * S::SROW + h + S::H * m];
        __syncwarp();
        dft_fixed<T, E>(v);
#pragma unroll
        for (int k = 1; k < E; ++k) v[k] = cmul(v[k], tw2[k]);
        if constexpr (S::H >= 4) {
            // DIF radix-2 on lane bit 2E: lanes h<2 keep Z_h + Z_{h+2}; h>=2 get (Z_{h-2} - Z_h) W4^{h-2}
            const bool hi = (h & 2) != 0;
            const bool rot = (h & 1) != 0;
#pragma unroll
            for (int k = 0; k < E; ++k) {
                cx<T> o;
                o.x = __shfl_xor_sync(0xffffffffu, v[k].x, 2 * E);
                o.y = __shfl_xor_sync(0xffffffffu, v[k].y, 2 * E);
                cx<T> r = hi ? (o - v[k]) : (v[k] + o);
                v[k] = (hi && rot) ? mul_mi(r) : r;
            }
        }
        if constexpr (S::H >= 2) {
            const bool odd = (h & 1) != 0;
            const T sg = odd ? T(-1) : T(1);
#pragma unroll
            for (int k = 0; k < E; ++k) {
                cx<T> o;
                o.x = __shfl_xor_sync(0xffffffffu, v[k].x, E);
                o.y = __shfl_xor_sync(0xffffffffu, v[k].y, E);
                v[k] = mk<T>(fma(sg, v[k].x, o.x), fma(sg, v[k].y, o.y));
            }
        }
    }
};

// ------------------------------------------------------------------------------------
// fused persistent kernel (T-branch / separable, p = 1)
// ------------------------------------------------------------------------------------
struct FusedArgs {
    const void* f;
    void* ws;           // S slots x [iM][Q][D]
    void* out;          // [W][M][N]
    const void* G;      // [c][Q][D] = conj(Gamma)/d
    const void* Cj;     // [iM] column chirp phase (null = 1)
    const void* Rs;     // [D] row chirp factor (null = 1)
    int Kmod;           // K mod D
    const void* E;      // [N] Alg. 1 column phase
    const int* rot;     // [N] Alg. 1 row rotation
    int* counters;      // [1 + 2W]
    int64_t W, L;
    int c, N, S, lag, nA, nB;
};

struct Job {
    int isA, w, idx;
};

__host__ __device__ __forceinline__ Job decode_job(int64_t p, int64_t W, int lag, int nA, int nB) {
    const int64_t lagE = lag < W ? lag : W;
    const int64_t seg1 = lagE * nA, seg2 = (W - lagE) * (nA + nB);
    Job j;
    if (p < seg1) {
        j.isA = 1; j.w = (int)(p / nA); j.idx = (int)(p % nA);
    } else if (p < seg1 + seg2) {
        const int64_t q = p - seg1;
        const int64_t t = lagE + q / (nA + nB), r = q % (nA + nB);
        if (r < nA) { j.isA = 1; j.w = (int)t; j.idx = (int)r; }
        else { j.isA = 0; j.w = (int)(t - lagE); j.idx = (int)(r - nA); }
    } else {
        const int64_t q = p - seg1 - seg2;
        j.isA = 0; j.w = (int)(W - lagE + q / nB); j.idx = (int)(q % nB);
    }
    return j;
}

__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

template <typename T> __device__ __forceinline__ cx<T> ldcg(const cx<T>* p);
template <> __device__ __forceinline__ float2 ldcg<float>(const float2* p) { return __ldcg(p); }
template <> __device__ __forceinline__ double2 ldcg<double>(const double2* p) { return __ldcg(p); }

template <typename T, int D, int MM, int Q>
struct FusedCfg {
    static constexpr int ED = D / 32, EM = MM / 32;
    static constexpr int NWARP = 16, NTHR = 512;
    static constexpr int SF = D + 1;        // Fh row stride
    static constexpr int SI = MM + 1;       // In row stride
    static constexpr int SO = 18;           // Out row stride (16 cols + pad, 16-byte aligned rows)
    static constexpr int SCR = (WarpFftShape<ED>::SCRATCH > WarpFftShape<EM>::SCRATCH ? WarpFftShape<ED>::SCRATCH
                                                                                       : WarpFftShape<EM>::SCRATCH);
    // A: Fh[16][SF] + scratch[16][SCR];  B: max(In[16][SI], scratch[16][SCR]) + Out[MM][SO]
    static constexpr size_t A_ELEMS = (size_t)16 * SF + (size_t)NWARP * SCR;
    static constexpr size_t B_ELEMS = ((size_t)16 * SI > (size_t)NWARP * SCR ? (size_t)16 * SI : (size_t)NWARP * SCR) +
                                      (size_t)MM * SO;
    static constexpr size_t SMEM = sizeof(cx<T>) * (A_ELEMS > B_ELEMS ? A_ELEMS : B_ELEMS);
};

template <typename T, int D, int MM, int Q>
__global__ void __launch_bounds__(512, 1) fused_t_kernel(FusedArgs A) {
    using C = cx<T>;
    using Cfg = FusedCfg<T, D, MM, Q>;
    constexpr int ED = Cfg::ED, EM = Cfg::EM;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C* sm = (C*)smem_raw;
    __shared__ int s_job;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    WarpFft<T, ED> fftD;
    fftD.init(lane);
    WarpFft<T, EM> fftM;
    if constexpr (EM != ED) fftM.init(lane);
    const WarpFft<T, EM>& fM = [&]() -> const WarpFft<T, EM>& {
        if constexpr (EM == ED) return fftD; else return fftM;
    }();
    const int64_t total = A.W * (int64_t)(A.nA + A.nB);
    int* queue = A.counters;
    int* doneA = A.counters + 1;
    int* doneB = A.counters + 1 + A.W;
    const C* __restrict__ f = (const C*)A.f;
    const C* __restrict__ G = (const C*)A.G;
    const int c = A.c;
    const int64_t slot_elems = (int64_t)MM * Q * D;

    for (;;) {
        if (tid == 0) s_job = atomicAdd(queue, 1);
        __syncthreads();
        const int64_t p = s_job;
        if (p >= total) break;
        const Job jb = decode_job(p, A.W, A.lag, A.nA, A.nB);
        if (tid == 0) {
            if (jb.isA) {
                if (jb.w >= A.S)
                    while (ld_acquire(&doneB[jb.w - A.S]) < A.nB) __nanosleep(100);
            } else {
                while (ld_acquire(&doneA[jb.w]) < A.nA) __nanosleep(100);
            }
        }
        __syncthreads();
        C* ws = (C*)A.ws + (int64_t)(jb.w % A.S) * slot_elems;
        if (jb.isA) {
            // ---------------- A job: 16 Zak columns (4 residues x Q=4 l) ----------------
            C* Fh = sm;
            C* scr = sm + 16 * Cfg::SF + warp * Cfg::SCR;
            const int rho = warp & 3, l = warp >> 2;
            const int r = 4 * jb.idx + rho;
            const int j = r + c * l;
            const C* fw = f + (int64_t)jb.w * A.L;
            C v[ED];
#pragma unroll
            for (int k = 0; k < ED; ++k) v[k] = __ldg(fw + (int64_t)(lane + 32 * k) * MM + j);
            if (A.Rs) {
                const C* Rs = (const C*)A.Rs;
#pragma unroll
                for (int k = 0; k < ED; ++k) v[k] = cmul(v[k], __ldg(Rs + lane + 32 * k));
            }
            fftD.run(v, scr, lane);
            if (A.Cj) {
                const C cj = __ldg((const C*)A.Cj + j);
#pragma unroll
                for (int k = 0; k < ED; ++k) v[k] = cmul(v[k], cj);
            }
            {
                const int k1 = lane % ED, jo = WarpFft<T, ED>::out_jo(lane);
#pragma unroll
                for (int k = 0; k < ED; ++k) Fh[warp * Cfg::SF + k1 + ED * k + ED * ED * jo] = v[k];
            }
            __syncthreads();
            const int shift = (int)(((int64_t)A.Kmod * j) % D);
            const C* Frow = Fh + warp * Cfg::SF;
#pragma unroll 1
            for (int u = 0; u < Q; ++u) {
                const C* Gr = G + ((int64_t)r * Q + u) * D;
#pragma unroll
                for (int k = 0; k < ED; ++k) {
                    const int nu = lane + 32 * k;
                    v[k] = cmul(Frow[(nu - shift) & (D - 1)], __ldg(Gr + nu));
                }
                fftD.run(v, scr, lane);
                // T_r(l,u;tau) -> C[j][kappa][n'], kappa = (l-u) mod Q, n' = (-tau - [l<u]) mod D
                const int kappa = (l - u + Q) % Q;
                const int off = (l < u) ? 1 : 0;
                C* dst = ws + ((int64_t)j * Q + kappa) * D;
                const int k1 = lane % ED, jo = WarpFft<T, ED>::out_jo(lane);
#pragma unroll
                for (int k = 0; k < ED; ++k) {
                    const int tau = k1 + ED * k + ED * ED * jo;
                    __stcg(dst + ((-tau - off) & (D - 1)), v[k]);
                }
            }
        } else {
            // ---------------- B job: 16 consecutive columns n ----------------
            C* In = sm;
            C* scr = sm + warp * Cfg::SCR;  // aliases In after the columns are in registers
            C* Out = sm + (16 * Cfg::SI > 16 * Cfg::SCR ? 16 * Cfg::SI : 16 * Cfg::SCR);
            const int t = jb.idx;
            const int n0p = 4 * t;  // n' block
            // load C[j][kappa][n0p..n0p+4) for all j, kappa -> In[col][j], col = kappa + 4 n''
            for (int e = tid; e < MM * Q * 2; e += Cfg::NTHR) {
                const int half = e & 1, kap = (e >> 1) % Q, jj = (e >> 1) / Q;
                const C* src = ws + ((int64_t)jj * Q + kap) * D + n0p + 2 * half;
                const C a0 = ldcg<T>(src), a1 = ldcg<T>(src + 1);
                In[(kap + Q * (2 * half)) * Cfg::SI + jj] = a0;
                In[(kap + Q * (2 * half + 1)) * Cfg::SI + jj] = a1;
            }
            __syncthreads();
            C v[EM];
#pragma unroll
            for (int k = 0; k < EM; ++k) v[k] = In[warp * Cfg::SI + lane + 32 * k];
            __syncthreads();
            fM.run(v, scr, lane);
            const int n = 16 * t + warp;
            const C e = __ldg((const C*)A.E + n);
            const int rt = __ldg(A.rot + n);
            const int k1 = lane % EM, jo = WarpFft<T, EM>::out_jo(lane);
#pragma unroll
            for (int k = 0; k < EM; ++k) {
                const int m = k1 + EM * k + EM * EM * jo;
                const int mo = (m - rt) & (MM - 1);
                Out[mo * Cfg::SO + warp] = cmul(e, v[k]);
            }
            __syncthreads();
            C* cw = (C*)A.out + (int64_t)jb.w * MM * A.N + 16 * t;
            constexpr int VPR = 16 * (int)sizeof(C) / 16;  // 16-byte vectors per output row
            for (int e2 = tid; e2 < MM * VPR; e2 += Cfg::NTHR) {
                const int mo = e2 / VPR, part = e2 % VPR;
                const float4 val = *(const float4*)((const char*)(Out + mo * Cfg::SO) + 16 * part);
                __stcs((float4*)((char*)(cw + (int64_t)mo * A.N) + 16 * part), val);
            }
        }
        __syncthreads();
        if (tid == 0) {
            __threadfence();
            atomicAdd(jb.isA ? &doneA[jb.w] : &doneB[jb.w], 1);
        }
    }
}

// ------------------------------------------------------------------------------------
// plan-side glue
// ------------------------------------------------------------------------------------
struct FastPlan {
    int kind = 0;  // 0 = none (generic path); 1 = fused T-branch p=1
    const char* name = "none";
    int D = 0, MM = 0, Q = 0, c = 0, N = 0;
    int64_t L = 0;
    int S = 4, lag = 2, nA = 0, nB = 0;
    int grid = 0;
    size_t smem = 0;
    size_t esz = 8;
    void* Cj = nullptr;
    void* Rs = nullptr;
    int Kmod = 0;
    const void* G = nullptr;
    const void* E = nullptr;
    const int* rot = nullptr;
    int* counters = nullptr;
    int64_t counters_W = 0;
    void (*launch)(const FusedArgs&, int grid, size_t smem, cudaStream_t) = nullptr;
};

template <typename T, int D, int MM, int Q>
void launch_fused(const FusedArgs& a, int grid, size_t smem, cudaStream_t st) {
    fused_t_kernel<T, D, MM, Q><<<grid, 512, smem, st>>>(a);
}

template <typename T>
__global__ void k_chirp_factors(cx<T>* Cj, cx<T>* Rs, int64_t K, int64_t L, int64_t M, int64_t D) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const unsigned __int128 twoL = 2 * L;
    if (i < M) {
        const unsigned __int128 e = ((unsigned __int128)K * (((unsigned __int128)i * i) % twoL)) % twoL;
        double s, c;
        sincospi((double)(int64_t)e / (double)L, &s, &c);
        Cj[i] = mk<T>((T)c, (T)s);
    }
    if (Rs && i < D) {
        const unsigned __int128 mm = ((unsigned __int128)M * M) % twoL;
        const unsigned __int128 e = ((unsigned __int128)K * ((((unsigned __int128)i * i) % twoL) * mm % twoL)) % twoL;
        double s, c;
        sincospi((double)(int64_t)e / (double)L, &s, &c);
        Rs[i] = mk<T>((T)c, (T)s);
    }
}

template <typename T, int D, int MM, int Q>
static int setup_fused(FastPlan* fp) {
    using Cfg = FusedCfg<T, D, MM, Q>;
    fp->smem = Cfg::SMEM;
    if (cudaFuncSetAttribute(fused_t_kernel<T, D, MM, Q>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fp->smem) !=
        cudaSuccess)
        return DGT_ECUDA;
    int per_sm = 0, dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fused_t_kernel<T, D, MM, Q>, 512, fp->smem) !=
            cudaSuccess ||
        per_sm < 1)
        return DGT_EUNSUPPORTED;
    fp->grid = per_sm * sms;
    fp->launch = &launch_fused<T, D, MM, Q>;
    return DGT_OK;
}

template <typename T>
int build_fast(FastPlan* fp, const dgt_lattice_info& I, void* G, void* /*chirp*/, void* E, int* rot,
               bool force_generic, cudaStream_t st) {
    fp->kind = 0;
    fp->name = "none";
    if (force_generic) return DGT_OK;
    if (I.branch == DGT_BRANCH_FREQ || I.p != 1 || I.q != 4 || I.c % 4 != 0) return DGT_OK;
    const int64_t D = I.d, MM = I.iM;
    int rc = DGT_OK;
    if constexpr (std::is_same<T, float>::value) {
        if (D == 512 && MM == 512) rc = setup_fused<T, 512, 512, 4>(fp);
        else if (D == 256 && MM == 256) rc = setup_fused<T, 256, 256, 4>(fp);
        else return DGT_OK;
    } else {
        return DGT_OK;  // c128 uses the generic kernels (round 1)
    }
    if (rc) return DGT_OK;  // fall back to the generic kernels (still CUDA)
    fp->D = (int)D; fp->MM = (int)MM; fp->Q = (int)I.q; fp->c = (int)I.c; fp->N = (int)I.N; fp->L = I.L;
    fp->nA = (int)(I.c / 4);
    fp->nB = (int)(D / 4);
    fp->esz = sizeof(cx<T>);
    fp->G = G; fp->E = E; fp->rot = rot;
    // chirp factorisation: K = sigma (L+1) mod 2L
    const int64_t L = I.L, twoL = 2 * L;
    const int64_t sigma = ((I.chirp_sigma % twoL) + twoL) % twoL;
    const int64_t K = (int64_t)((unsigned __int128)sigma * (unsigned __int128)((L + 1) % twoL) % (unsigned __int128)twoL);
    fp->Kmod = (int)(K % D);
    if (K != 0) {
        const bool r_trivial = ((unsigned __int128)K * ((unsigned __int128)MM * MM % twoL)) % twoL == 0;
        if (cudaMalloc(&fp->Cj, sizeof(cx<T>) * MM) != cudaSuccess) return DGT_ENOMEM;
        if (!r_trivial && cudaMalloc(&fp->Rs, sizeof(cx<T>) * D) != cudaSuccess) return DGT_ENOMEM;
        const int64_t n = std::max<int64_t>(MM, D);
        k_chirp_factors<T><<<(unsigned)((n + 255) / 256), 256, 0, st>>>((cx<T>*)fp->Cj, (cx<T>*)fp->Rs, K, L, MM, D);
    }
    fp->kind = 1;
    fp->name = "fused_t_p1";
    return DGT_OK;
}

inline void free_fast(FastPlan* fp) {
    if (fp->Cj) cudaFree(fp->Cj);
    if (fp->Rs) cudaFree(fp->Rs);
    if (fp->counters) cudaFree(fp->counters);
    fp->Cj = fp->Rs = nullptr;
    fp->counters = nullptr;
}

inline size_t fast_workspace_bytes(const FastPlan* fp, int64_t /*Wc*/) {
    return (size_t)fp->S * fp->MM * fp->Q * fp->D * fp->esz;
}

// the fused kernel consumes the whole batch in one launch
inline int64_t fast_chunk(const FastPlan*) { return (int64_t)1 << 40; }
inline int64_t fast_launches_per_chunk(const FastPlan*) { return 1; }

template <typename T>
int launch_fast(FastPlan* fp, const void* f, int real_in, void* ws, void* c, int64_t W, cudaStream_t st) {
    if (real_in) return DGT_EUNSUPPORTED;
    if (fp->counters_W < W) {
        if (fp->counters) cudaFree(fp->counters);
        fp->counters = nullptr;
        fp->counters_W = 0;
        if (cudaMalloc(&fp->counters, sizeof(int) * (1 + 2 * W)) != cudaSuccess) return DGT_ENOMEM;
        fp->counters_W = W;
    }
    if (cudaMemsetAsync(fp->counters, 0, sizeof(int) * (1 + 2 * W), st) != cudaSuccess) return DGT_ECUDA;
    FusedArgs a{};
    a.f = f; a.ws = ws; a.out = c; a.G = fp->G; a.Cj = fp->Cj; a.Rs = fp->Rs; a.Kmod = fp->Kmod;
    a.E = fp->E; a.rot = fp->rot; a.counters = fp->counters;
    a.W = W; a.L = fp->L; a.c = fp->c; a.N = fp->N; a.S = fp->S; a.lag = fp->lag; a.nA = fp->nA; a.nB = fp->nB;
    const int64_t total = W * (int64_t)(fp->nA + fp->nB);
    const int grid = (int)std::min<int64_t>(fp->grid, total);
    fp->launch(a, grid, fp->smem, st);
    return DGT_OK;
}

}  // namespace nsdgt
