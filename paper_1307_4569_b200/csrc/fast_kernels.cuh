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
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "../../include/nsdgt.h"
#include "cplx.cuh"
#include "fft_smem.cuh"
#include "fused7.cuh"

namespace nsdgt {

template <typename T>
__global__ void k_window_factor(cx<T>* G, const double2* gt, int64_t L, int64_t c, int64_t d, int64_t p, int64_t q);

// ------------------------------------------------------------------------------------
// warp FFT, N = 32*E, forward (exp(-2 pi i jk/N))
// ------------------------------------------------------------------------------------
template <int E> struct WarpFftShape {
    static constexpr int N = 32 * E;
    static constexpr int H = 32 / E;
    static constexpr int SROW = (E == 16) ? 33 : 36;  // padded scratch row (bank-conflict free)
    static constexpr int SCRATCH = E * SROW;           // complex elements per warp
};

// W_32^k as compile-time constants (pass-2 twiddles when H = 2: only lanes h = 1 multiply)
__device__ __forceinline__ float2 w32(int k) {
    // table of exp(-2 pi i k/32), k < 16 (constant memory broadcast: k is warp-uniform)
    constexpr float c[16] = {1.0f, 0.98078528040323044913f, 0.92387953251128675613f, 0.83146961230254523708f,
                             0.70710678118654752440f, 0.55557023301960222474f, 0.38268343236508977173f,
                             0.19509032201612826785f, 0.0f, -0.19509032201612826785f, -0.38268343236508977173f,
                             -0.55557023301960222474f, -0.70710678118654752440f, -0.83146961230254523708f,
                             -0.92387953251128675613f, -0.98078528040323044913f};
    return make_float2(c[k], c[(k + 8) & 15] * (k < 8 ? 1.0f : -1.0f));  // (cos, -sin)
}

template <typename T, int E>
struct WarpFft {
    using S = WarpFftShape<E>;
    cx<T> tw1[E];                   // W_N^{lane*k1}
    cx<T> tw2[S::H == 2 ? 1 : E];   // W_32^{h*k'}, h = lane / E (registers only when H > 2)

    __device__ __forceinline__ void init(int lane) {
        const int h = lane / E;
#pragma unroll
        for (int k = 0; k < E; ++k) {
            double s, c;
            sincospi(-2.0 * (double)((lane * k) % S::N) / (double)S::N, &s, &c);
            tw1[k] = mk<T>((T)c, (T)s);
            if constexpr (S::H != 2) {
                sincospi(-2.0 * (double)((h * k) % 32) / 32.0, &s, &c);
                tw2[k] = mk<T>((T)c, (T)s);
            }
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
        if constexpr (S::H == 2) {
            if (h) {
#pragma unroll
                for (int k = 1; k < E; ++k) v[k] = cmul(v[k], w32(k));
            }
        } else {
#pragma unroll
            for (int k = 1; k < E; ++k) v[k] = cmul(v[k], tw2[k]);
        }
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
    int* counters;      // [ngroups] group-barrier counters (zeroed per launch)
    int64_t W, L;
    int c, N, nA, nB;
    int GS, ngroups;    // CTAs per group; groups (each group owns one signal at a time)
    int dbg;            // experiment knobs (0 in production)
    int tma;            // 1: c leaves through TMA bulk-tensor stores (NCOL = 16 only)
    int discard;        // 1: discard dead intermediate lines from L2 before rewriting them
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

template <typename T, int D, int MM, int Q, int NCOL>
struct FusedCfg {
    static constexpr int ED = D / 32, EM = MM / 32;
    static constexpr int NWARP = NCOL, NTHR = 32 * NCOL;   // one warp per column
    static constexpr int ROWS = D > MM ? D : MM;
    static constexpr int TILE = ROWS * NCOL;  // row-major, NCOL complex per row, 16-byte chunks XOR-swizzled
    static constexpr int SCR = (WarpFftShape<ED>::SCRATCH > WarpFftShape<EM>::SCRATCH ? WarpFftShape<ED>::SCRATCH
                                                                                       : WarpFftShape<EM>::SCRATCH);
    static constexpr int FH = NCOL * (D + 1);   // per-warp F^ rows (A jobs)
    static constexpr int OUT = MM * NCOL;       // output staging (B jobs), aliases FH
    static constexpr int U = FH > OUT ? FH : OUT;
    static constexpr size_t ELEMS = (size_t)TILE + (size_t)NWARP * SCR + (size_t)U;
    static constexpr size_t SMEM = sizeof(cx<T>) * ELEMS;
    static constexpr int LPJ = NCOL / 4;        // values of l per A job (4 residues each)
    static constexpr int NPK = NCOL / 4;        // n' values per kappa per B job
};

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
// TMA (bulk tensor) store of one 2-D box from shared memory; asynchronous (bulk group)
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* smem, int x, int y) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];\n" ::"l"(map), "r"(sa),
                 "r"(x), "r"(y)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// Group barrier over the GS CTAs of one group (all CTAs are co-resident: persistent grid).
__device__ __forceinline__ void group_barrier(int* cnt, int target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(cnt, 1);
        while (ld_acquire(cnt) < target) __nanosleep(32);
    }
    __syncthreads();
}

// Static schedule of one CTA: for each signal of its group, its A jobs, a group barrier,
// its B jobs, a group barrier.  Position k -> (w, isA, job); false past the end.
struct CtaSchedule {
    int64_t W;
    int ngroups, g, q, GS, perA, perB;
    __device__ __forceinline__ bool at(int64_t k, int64_t* w, int* isA, int* job) const {
        const int per = perA + perB;
        const int64_t round = k / per;
        const int r = (int)(k % per);
        *w = g + round * ngroups;
        if (*w >= W) return false;
        if (r < perA) { *isA = 1; *job = q + r * GS; }
        else { *isA = 0; *job = q + (r - perA) * GS; }
        return true;
    }
};

// Tile element (row, col): row-major rows of NCOL complex; the 16-byte chunk index is
// XOR-swizzled with the row so that column reads are at most 4-way bank conflicted.
template <int NCOL>
__device__ __forceinline__ int tile_pos(int row, int col) {
    return row * NCOL + ((((col >> 1) ^ (row & (NCOL / 2 - 1))) << 1) | (col & 1));
}

// Issue the cp.async copies of one job's tile (16-byte chunks, whole 32-byte sectors).
//  A job (4 residues r0.. x LPJ values of l from l0): row s, col = rho + 4 (l - l0)
//        <- f[w][s M + c l + r0 + rho];  chunk ch = 2 (l - l0) + hf holds rho = 2hf, 2hf+1
//  B job (NCOL columns n = NCOL t + kappa + 4 n''): row j, col = 2 chunk + (n'' & 1)
//        <- C[j][kappa][NPK t + n''];  chunk ch = kappa (NPK/2) + (n'' >> 1)
template <typename T, int D, int MM, int Q, int NCOL>
__device__ __forceinline__ void issue_tile(cx<T>* tile, const FusedArgs& A, const cx<T>* ws, int64_t w, int isA,
                                           int job) {
    using Cfg = FusedCfg<T, D, MM, Q, NCOL>;
    constexpr int NT = Cfg::NTHR, CPR = NCOL / 2;   // chunks per row
    const int tid = threadIdx.x;
    if (isA) {
        if (A.dbg & 16) { cp_async_commit(); return; }
        constexpr int JPR = 16 / NCOL;               // A jobs per residue group
        const int r0 = 4 * (job / JPR), l0 = (job % JPR) * Cfg::LPJ;
        const cx<T>* fw = (const cx<T>*)A.f + w * A.L + r0;
#pragma unroll
        for (int i = 0; i < D * CPR / NT; ++i) {
            const int e = tid + NT * i;
            const int s = e / CPR, ch = e % CPR, ll = ch >> 1, hf = ch & 1;
            cp_async16(tile + s * NCOL + ((ch ^ (s & (CPR - 1))) << 1),
                       fw + (int64_t)s * MM + A.c * (l0 + ll) + 2 * hf);
        }
    } else {
        if (A.dbg & 32) { cp_async_commit(); return; }
        constexpr int HPK = Cfg::NPK / 2;            // chunks per kappa
        const cx<T>* src = ws + Cfg::NPK * job;
#pragma unroll
        for (int i = 0; i < MM * CPR / NT; ++i) {
            const int e = tid + NT * i;
            const int jj = e / CPR, ch = e % CPR, kap = ch / HPK, hf = ch % HPK;
            cp_async16(tile + jj * NCOL + ((ch ^ (jj & (CPR - 1))) << 1),
                       src + ((int64_t)jj * Q + kap) * D + 2 * hf);
        }
    }
    cp_async_commit();
}

template <typename T, int D, int MM, int Q, int NCOL>
__global__ void __launch_bounds__(32 * NCOL, (D <= 256 ? 2 : 1) * (NCOL == 8 ? 2 : 1))
    fused_t_kernel(FusedArgs A, const __grid_constant__ CUtensorMap cmap) {
    using C = cx<T>;
    using Cfg = FusedCfg<T, D, MM, Q, NCOL>;
    constexpr int ED = Cfg::ED, EM = Cfg::EM, NT = Cfg::NTHR;
    static_assert(sizeof(C) == 8, "fused path is complex64");
    static_assert(Q == 4, "fused path assumes q = 4");
    static_assert(NCOL == 8 || NCOL == 16, "8 or 16 columns per job");
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    C* sm = (C*)smem_raw;
    C* tile = sm;
    C* scr = sm + Cfg::TILE + (threadIdx.x >> 5) * Cfg::SCR;
    C* uni = sm + Cfg::TILE + Cfg::NWARP * Cfg::SCR;   // 1024-byte aligned (TMA 128B swizzle)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    WarpFft<T, ED> fftD;
    fftD.init(lane);
    WarpFft<T, EM> fftM;
    if constexpr (EM != ED) fftM.init(lane);
    const WarpFft<T, EM>& fM = [&]() -> const WarpFft<T, EM>& {
        if constexpr (EM == ED) return fftD; else return fftM;
    }();
    CtaSchedule sch;
    sch.W = A.W; sch.ngroups = A.ngroups; sch.g = blockIdx.x / A.GS; sch.q = blockIdx.x % A.GS; sch.GS = A.GS;
    sch.perA = A.nA > sch.q ? (A.nA - sch.q + A.GS - 1) / A.GS : 0;
    sch.perB = A.nB > sch.q ? (A.nB - sch.q + A.GS - 1) / A.GS : 0;
    if (sch.g >= A.ngroups) return;
    int* bar = A.counters + sch.g;
    int epoch = 0;
    const C* __restrict__ G = (const C*)A.G;
    const int c = A.c;
    C* ws = (C*)A.ws + (int64_t)sch.g * MM * Q * D;   // this group's intermediate C[j][kappa][n']

    if (sch.perA + sch.perB == 0) {   // no jobs: still take part in the group's barriers
        for (int64_t w = sch.g; w < A.W; w += A.ngroups) {
            group_barrier(bar, (++epoch) * A.GS);
            group_barrier(bar, (++epoch) * A.GS);
        }
        return;
    }
    if ((A.dbg >> 8) && (sch.g & 1)) {   // experiment: delay odd groups by dbg>>8 microseconds
        unsigned long long t0;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        for (;;) {
            unsigned long long t1;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
            if (t1 - t0 > (unsigned long long)(A.dbg >> 8) * 1000ull) break;
            __nanosleep(1000);
        }
    }
    int64_t w;
    int isA, job;
    int64_t k = 0;
    bool have = sch.at(0, &w, &isA, &job);
    bool issued = false;
    if (have && isA) { issue_tile<T, D, MM, Q, NCOL>(tile, A, ws, w, 1, job); issued = true; }
    int64_t cur_w = sch.g;   // signal whose phases we are in
    int phase = 0;           // 0 = A phase of cur_w, 1 = B phase of cur_w
    while (have) {
        while (cur_w != w || phase != (isA ? 0 : 1)) {   // pass the group barriers up to this job
            group_barrier(bar, (++epoch) * A.GS);
            if (phase == 0) phase = 1; else { phase = 0; cur_w += A.ngroups; }
        }
        if (!issued) issue_tile<T, D, MM, Q, NCOL>(tile, A, ws, w, isA, job);
        cp_async_wait_all();
        __syncthreads();  // tile k visible; previous job's Out fully stored
        int64_t w2; int isA2, job2;
        const bool more = sch.at(k + 1, &w2, &isA2, &job2);
        // the next tile may be prefetched now unless it is a B tile behind a group barrier
        const bool can_pf = more && (isA2 || (!isA && w2 == w));
        if (isA) {
            // -------- A job: NCOL Zak columns = 4 residues (rho) x LPJ values of l --------
            constexpr int JPR = 16 / NCOL;
            const int rho = warp & 3;
            const int l = (job % JPR) * Cfg::LPJ + (warp >> 2);
            const int r = 4 * (job / JPR) + rho;
            const int j = r + c * l;
            C v[ED];
#pragma unroll
            for (int kk = 0; kk < ED; ++kk) v[kk] = tile[tile_pos<NCOL>(lane + 32 * kk, warp)];
            if (A.discard) {
                // The previous signal's intermediate rows this job is about to overwrite are dead
                // (its B phase ended at the last group barrier): drop them from L2 without
                // writing them back to HBM.  Only this CTA writes these rows.
                C* row = ws + (int64_t)j * Q * D;   // this warp's column j: Q*D complex
                constexpr int LINES = Q * D * (int)sizeof(C) / 128;
                for (int i = lane; i < LINES; i += 32)
                    asm volatile("discard.global.L2 [%0], 128;" ::"l"((const char*)row + 128 * i) : "memory");
            }
            __syncthreads();  // tile consumed
            issued = false;
            if (can_pf) { issue_tile<T, D, MM, Q, NCOL>(tile, A, ws, w2, isA2, job2); issued = true; }
            if (A.Rs) {
                const C* Rs = (const C*)A.Rs;
#pragma unroll
                for (int kk = 0; kk < ED; ++kk) v[kk] = cmul(v[kk], __ldg(Rs + lane + 32 * kk));
            }
            if (!(A.dbg & 1)) fftD.run(v, scr, lane);
            if (A.Cj) {
                const C cj = __ldg((const C*)A.Cj + j);
#pragma unroll
                for (int kk = 0; kk < ED; ++kk) v[kk] = cmul(v[kk], cj);
            }
            C* Frow = uni + warp * (D + 1);
            if (tid == 0) bulk_wait_read0();   // the previous output box has left uni
            __syncthreads();
            {
                const int k1 = lane % ED, jo = WarpFft<T, ED>::out_jo(lane);
#pragma unroll
                for (int kk = 0; kk < ED; ++kk) Frow[k1 + ED * kk + ED * ED * jo] = v[kk];
            }
            __syncwarp();
            const int shift = (int)(((int64_t)A.Kmod * j) % D);
#pragma unroll 1
            for (int u = 0; u < Q; ++u) {
                const C* Gr = G + ((int64_t)r * Q + u) * D;
#pragma unroll
                for (int kk = 0; kk < ED; ++kk) {
                    const int nu = lane + 32 * kk;
                    v[kk] = (A.dbg & 64) ? Frow[(nu - shift) & (D - 1)] : cmul(Frow[(nu - shift) & (D - 1)], __ldg(Gr + nu));
                }
                if (!(A.dbg & 1)) fftD.run(v, scr, lane);
                // T_r(l,u;tau) -> C[j][kappa][n'], kappa = (l-u) mod Q, n' = (-tau - [l<u]) mod D
                const int kappa = (l - u + Q) % Q;
                const int off = (l < u) ? 1 : 0;
                C* dst = ws + ((int64_t)j * Q + kappa) * D;
                const int k1 = lane % ED, jo = WarpFft<T, ED>::out_jo(lane);
                const int base = -(k1 + ED * ED * jo) - off;
#pragma unroll
                if (!(A.dbg & 4))
                    for (int kk = 0; kk < ED; ++kk) __stcg(dst + ((base - ED * kk) & (D - 1)), v[kk]);
            }
        } else {
            // -------- B job: NCOL consecutive columns n = NCOL t + col, col = kappa + 4 n'' --------
            const int t = job;
            const int kap = warp & 3, nn = warp >> 2;
            const int cl = 2 * (kap * (Cfg::NPK / 2) + (nn >> 1)) + (nn & 1);
            const int n = NCOL * t + warp;   // warp = kappa + 4 n''
            const C e = __ldg((const C*)A.E + n);
            const int rt = __ldg(A.rot + n);
            C v[EM];
#pragma unroll
            for (int kk = 0; kk < EM; ++kk) v[kk] = tile[tile_pos<NCOL>(lane + 32 * kk, cl)];
            __syncthreads();  // tile consumed
            issued = false;
            if (can_pf) { issue_tile<T, D, MM, Q, NCOL>(tile, A, ws, w2, isA2, job2); issued = true; }
            if (!(A.dbg & 2)) fM.run(v, scr, lane);
            C* Out = uni;
            if (tid == 0) bulk_wait_read0();   // the previous output box has left uni
            __syncthreads();
            const int k1 = lane % EM, jo = WarpFft<T, EM>::out_jo(lane);
            if (NCOL == 16 && A.tma) {
                // TMA SWIZZLE_128B layout: row mo = 128 B, 16-byte chunk index XOR (mo & 7)
#pragma unroll
                for (int kk = 0; kk < EM; ++kk) {
                    const int m = k1 + EM * kk + EM * EM * jo;
                    const int mo = (m - rt) & (MM - 1);
                    Out[mo * 16 + ((((warp >> 1) ^ (mo & 7)) << 1) | (warp & 1))] = cmul(e, v[kk]);
                }
                fence_proxy_async_smem();
                __syncthreads();
                if (tid == 0 && !(A.dbg & 8)) {
#pragma unroll
                    for (int bx = 0; bx < MM / 256; ++bx)
                        tma_store_2d(&cmap, Out + bx * 256 * 16, 32 * t, (int)(w * MM) + 256 * bx);
                    bulk_commit();
                }
            } else {
#pragma unroll
                for (int kk = 0; kk < EM; ++kk) {
                    const int m = k1 + EM * kk + EM * EM * jo;
                    const int mo = (m - rt) & (MM - 1);
                    const int x = NCOL == 16 ? (mo & 15) : ((mo >> 1) & 7);
                    Out[mo * NCOL + (warp ^ x)] = cmul(e, v[kk]);
                }
                __syncthreads();
                C* cw = (C*)A.out + w * MM * A.N + NCOL * t;
                constexpr int VPR = NCOL / 2;               // float4 per output row
                constexpr int PER2 = MM * VPR / NT;
#pragma unroll
                for (int i = 0; i < PER2; ++i) {
                    const int e2 = tid + NT * i;
                    const int mo = e2 / VPR, pp = e2 % VPR;
                    const int x = NCOL == 16 ? (mo & 15) : ((mo >> 1) & 7);
                    float4 val = *(const float4*)(Out + mo * NCOL + 2 * (pp ^ (x >> 1)));
                    if (x & 1) val = make_float4(val.z, val.w, val.x, val.y);
                    if (!(A.dbg & 8)) __stcs((float4*)(cw + (int64_t)mo * A.N + 2 * pp), val);
                }
            }
        }
        ++k;
        have = more;
        if (have) { w = w2; isA = isA2; job = job2; }
    }
    while (cur_w < A.W) {   // this CTA's remaining barriers
        group_barrier(bar, (++epoch) * A.GS);
        if (phase == 0) phase = 1; else { phase = 0; cur_w += A.ngroups; }
    }
    cp_async_wait_all();
    if (tid == 0) bulk_wait0();
}

// ------------------------------------------------------------------------------------
// plan-side glue
// ------------------------------------------------------------------------------------
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

struct FastPlan {
    int kind = 0;  // 0 = none (generic path); 1 = fused T-branch p=1
    const char* name = "none";
    int D = 0, MM = 0, Q = 0, c = 0, N = 0;
    int64_t L = 0;
    int nA = 0, nB = 0, GS = 16, ngroups = 1, ncol = 16;
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
    void (*launch)(const FusedArgs&, const CUtensorMap&, int grid, size_t smem, cudaStream_t, const cudaAccessPolicyWindow*) = nullptr;
    bool persist = false;   // L2 persisting window over the intermediate workspace
    // kind 2 (fused7): per-column window table G', ring of S7 slots, look-ahead lag7
    void* Gp7 = nullptr;
    int beta7 = 0, S7 = 8, lag7 = 5, minb7 = 3;
};

template <typename T, int D, int MM, int Q, int NCOL>
void launch_fused(const FusedArgs& a, const CUtensorMap& cmap, int grid, size_t smem, cudaStream_t st,
                  const cudaAccessPolicyWindow* apw) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(FusedCfg<T, D, MM, Q, NCOL>::NTHR);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    int na = 0;
    if (apw) {
        // keep the intermediate ring L2 resident while c streams through
        attr[na].id = cudaLaunchAttributeAccessPolicyWindow;
        attr[na].val.accessPolicyWindow = *apw;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    cudaLaunchKernelEx(&cfg, fused_t_kernel<T, D, MM, Q, NCOL>, a, cmap);
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

template <typename T, int D, int MM, int Q, int NCOL>
static int setup_fused(FastPlan* fp) {
    using Cfg = FusedCfg<T, D, MM, Q, NCOL>;
    fp->smem = Cfg::SMEM;
    if (cudaFuncSetAttribute(fused_t_kernel<T, D, MM, Q, NCOL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fp->smem) !=
        cudaSuccess)
        return DGT_ECUDA;
    int per_sm = 0, dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fused_t_kernel<T, D, MM, Q, NCOL>, Cfg::NTHR, fp->smem) !=
            cudaSuccess ||
        per_sm < 1)
        return DGT_EUNSUPPORTED;
    fp->grid = per_sm * sms;
    fp->launch = &launch_fused<T, D, MM, Q, NCOL>;
    fp->ncol = NCOL;
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
        const int ncol = std::getenv("NSDGT_NCOL") ? std::atoi(std::getenv("NSDGT_NCOL")) : 16;
        if (D == 512 && MM == 512) rc = ncol == 16 ? setup_fused<T, 512, 512, 4, 16>(fp) : setup_fused<T, 512, 512, 4, 8>(fp);
        else if (D == 256 && MM == 256) rc = ncol == 16 ? setup_fused<T, 256, 256, 4, 16>(fp) : setup_fused<T, 256, 256, 4, 8>(fp);
        else return DGT_OK;
    } else {
        return DGT_OK;  // c128 uses the generic kernels (round 1)
    }
    if (rc) return DGT_OK;  // fall back to the generic kernels (still CUDA)
    fp->D = (int)D; fp->MM = (int)MM; fp->Q = (int)I.q; fp->c = (int)I.c; fp->N = (int)I.N; fp->L = I.L;
    fp->nA = (int)(I.c / 4) * (16 / fp->ncol);   // ncol columns (4 residues x ncol/4 l) per A job
    fp->nB = (int)(D * 4 / fp->ncol);            // ncol consecutive columns n per B job
    // groups of GS CTAs each own one signal at a time; the intermediates of the signals in
    // flight (ngroups x per-signal bytes) must stay L2 resident
    {
        const size_t per_sig = (size_t)MM * I.q * D * sizeof(cx<T>);
        const int max_inflight = (int)std::max<size_t>(1, (size_t)(72u << 20) / per_sig);
        int gs = 4;
        while (gs < 64 && (fp->grid / gs) > max_inflight) gs *= 2;
        if (const char* e = std::getenv("NSDGT_GS")) gs = std::max(1, std::atoi(e));
        fp->GS = std::min(gs, fp->grid);
        fp->ngroups = std::max(1, fp->grid / fp->GS);
    }
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
    fp->persist = std::getenv("NSDGT_PERSIST") != nullptr;  // experiment only
    fp->kind = 1;
    fp->name = "fused_t_p1";
    return DGT_OK;
}

inline void free_fast(FastPlan* fp) {
    if (fp->Cj) cudaFree(fp->Cj);
    if (fp->Rs) cudaFree(fp->Rs);
    if (fp->counters) cudaFree(fp->counters);
    if (fp->Gp7) cudaFree(fp->Gp7);
    fp->Gp7 = nullptr;
    fp->Cj = fp->Rs = nullptr;
    fp->counters = nullptr;
}

inline size_t fast_workspace_bytes(const FastPlan* fp, int64_t /*Wc*/) {
    if (fp->kind == 2) return (size_t)fp->S7 * fp->MM * fp->Q * fp->D * fp->esz;
    return (size_t)fp->ngroups * fp->MM * fp->Q * fp->D * fp->esz;
}

// the fused kernel consumes the whole batch in one launch
inline int64_t fast_chunk(const FastPlan*) { return (int64_t)1 << 40; }
inline int64_t fast_launches_per_chunk(const FastPlan*) { return 1; }

template <int D, int MINB>
static void launch7(const v7::Args& a, int grid, size_t smem, cudaStream_t st, const cudaAccessPolicyWindow* apw) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(v7::Cfg<D>::NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    int na = 0;
    if (apw) {
        // keep the intermediate ring L2 resident while f and c stream through
        attr[na].id = cudaLaunchAttributeAccessPolicyWindow;
        attr[na].val.accessPolicyWindow = *apw;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    cudaLaunchKernelEx(&cfg, v7::fused7_kernel<D, MINB>, a);
}

// kind 2: the fused7 kernel (fused7.cuh).  Builds G' from the fp64 window factors and checks,
// on the host, the identities the kernel relies on; returns DGT_OK with
// fp->kind unchanged when the lattice does not qualify.
template <typename T>
int build_fast7(FastPlan* fp, const dgt_lattice_info& I, const double2* gt, const void* E, cudaStream_t st) {
    if constexpr (!std::is_same<T, float>::value) return DGT_OK;
    if (std::getenv("NSDGT_V6")) return DGT_OK;
    if (I.branch == DGT_BRANCH_FREQ || I.p != 1 || I.q != 4 || I.d != I.iM || (I.d != 512 && I.d != 256)) return DGT_OK;
    if (I.c % 16 != 0 || I.N % 16 != 0 || I.iM != I.M || I.N != I.q * I.d) return DGT_OK;
    const int64_t L = I.L, twoL = 2 * L, D = I.d, M = I.M, Q = I.q, N = I.N;
    const int64_t sigma = ((I.chirp_sigma % twoL) + twoL) % twoL;
    const int64_t K = (int64_t)((unsigned __int128)sigma * (unsigned __int128)((L + 1) % twoL) % (unsigned __int128)twoL);
    if (((unsigned __int128)K * ((unsigned __int128)M * M % twoL)) % twoL != 0) return DGT_OK;  // R(s) == 1 required
    // rotation identity rot(n(tau)) = alpha_{l,u} - beta tau (mod M), n(tau) = (l - u - q tau) mod N
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
    // fp64 window factors G64[(r q + u) d + nu] = conj(Gamma)/d, then G'
    double2* G64 = nullptr;
    if (cudaMalloc(&G64, sizeof(double2) * L) != cudaSuccess) return DGT_ENOMEM;
    k_window_factor<double><<<(unsigned)std::min<int64_t>((L + 255) / 256, 148 * 64), 256, 0, st>>>(G64, gt, L, I.c, I.d, 1, Q);
    const size_t gp_bytes = sizeof(float2) * (size_t)M * Q * D;
    if (cudaMalloc(&fp->Gp7, gp_bytes) != cudaSuccess) { cudaFree(G64); return DGT_ENOMEM; }
    ga.Gp = (float4*)fp->Gp7; ga.G64 = G64; ga.L = L; ga.K = K;
    ga.M = (int)M; ga.D = (int)D; ga.Q = (int)Q; ga.c = (int)I.c; ga.beta = (int)beta; ga.R1 = (int)(D / 16);
    v7::k_gprime<<<(unsigned)std::min<int64_t>((M * Q * D + 255) / 256, 148 * 64), 256, 0, st>>>(ga);
    if (cudaStreamSynchronize(st) != cudaSuccess) { cudaFree(G64); return DGT_ECUDA; }
    cudaFree(G64);
    size_t smem = D == 512 ? v7::Cfg<512>::SMEM : v7::Cfg<256>::SMEM;
    // CTAs per SM: 3 (no register spills) by default; NSDGT_CTAS=4 trades spills for warps
    // CTAs per SM (each 128 threads): measured best 3 for D = 512 (more CTAs leave too little
    // L1 next to 3 x 53 KB of shared memory), 5 for D = 256 (36 KB, 91 registers).  NSDGT_CTAS overrides.
    fp->minb7 = D == 512 ? 3 : 5;
    if (const char* e = std::getenv("NSDGT_CTAS")) fp->minb7 = std::max(3, std::min(5, std::atoi(e)));
    if (D == 512 && fp->minb7 == 5) fp->minb7 = 4;
    const void* kfn = D == 512 ? (fp->minb7 == 4 ? (const void*)v7::fused7_kernel<512, 4> : (const void*)v7::fused7_kernel<512, 3>)
                               : (fp->minb7 == 5   ? (const void*)v7::fused7_kernel<256, 5>
                                  : fp->minb7 == 4 ? (const void*)v7::fused7_kernel<256, 4>
                                                   : (const void*)v7::fused7_kernel<256, 3>);
    if (cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return DGT_ECUDA;
    int per_sm = 0, dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, v7::Cfg<512>::NT, smem) != cudaSuccess || per_sm < 1)
        return DGT_EUNSUPPORTED;
    // persistent kernel: every CTA must be resident (the occupancy query bounds the grid)
    if (const char* e = std::getenv("NSDGT_PER_SM")) per_sm = std::max(1, std::min(per_sm, std::atoi(e)));
    fp->grid = per_sm * sms;
    fp->smem = smem;
    if (std::getenv("NSDGT_VERBOSE"))
        std::fprintf(stderr, "fused7: D=%d CTAs/SM=%d grid=%d smem/CTA=%zu B S=%d\n", (int)D, per_sm, fp->grid, smem, fp->S7);
    fp->D = (int)D; fp->MM = (int)M; fp->Q = (int)Q; fp->c = (int)I.c; fp->N = (int)N; fp->L = L;
    fp->nA = (int)(M / v7::Cfg<512>::ACOL); fp->nB = (int)(N / 16);
    fp->Kmod = (int)(K % D);
    fp->beta7 = (int)beta;
    // Look-ahead: B(w) is queued lag signals after A(w).  An A job spans a few tiles, so
    // about 3 x (CTAs / jobs per signal) signals of look-ahead hide the A -> B dependency;
    // the ring (S signals of intermediate) is capped at ~64 MB so it stays mostly in L2.
    {
        const int jps = fp->nA + fp->nB;
        const size_t per_sig = (size_t)M * Q * D * sizeof(float2);
        const int smax = std::max(4, (int)((64ull << 20) / per_sig));
        fp->lag7 = std::max(2, std::min(smax - 3, (3 * fp->grid + jps / 2) / jps));
        fp->S7 = std::min(smax, fp->lag7 + 3 + fp->lag7 / 4);
    }
    if (const char* e = std::getenv("NSDGT_S")) fp->S7 = std::max(1, std::atoi(e));
    if (const char* e = std::getenv("NSDGT_LAG")) fp->lag7 = std::max(0, std::atoi(e));
    if (fp->lag7 >= fp->S7) fp->lag7 = fp->S7 - 1;
    fp->E = E;
    fp->esz = sizeof(float2);
    // No persisting-L2 carve-out: consumed ring lines are discarded (fused7.cuh), and a
    // device-wide set-aside measurably slows the kernel and everything else in the process.
    fp->persist = false;
    fp->kind = 2;
    fp->name = "fused7_t_p1";
    return DGT_OK;
}

template <typename T>
int launch_fast(FastPlan* fp, const void* f, int real_in, void* ws, void* c, int64_t W, cudaStream_t st) {
    if (real_in) return DGT_EUNSUPPORTED;
    if (fp->kind == 2) {
        const int nctr = 1 + 2 * fp->S7;
        if (!fp->counters) {
            if (cudaMalloc(&fp->counters, sizeof(int) * nctr) != cudaSuccess) return DGT_ENOMEM;
        }
        if (cudaMemsetAsync(fp->counters, 0, sizeof(int) * nctr, st) != cudaSuccess) return DGT_ECUDA;
        v7::Args a{};
        a.f = (const float2*)f; a.out = (float2*)c; a.ws = (float2*)ws; a.Gp = (const float4*)fp->Gp7;
        if (W * (int64_t)(fp->nA + fp->nB) >= (int64_t)1 << 31) return DGT_EUNSUPPORTED;
        a.E = (const float2*)fp->E; a.ctr = fp->counters; a.W = (int)W; a.N = fp->N; a.c = fp->c; a.Kmod = fp->Kmod;
        a.dbg = std::getenv("NSDGT_DBG") ? std::atoi(std::getenv("NSDGT_DBG")) : 0;
        if (a.dbg & 16) {
            static unsigned long long* logbuf = nullptr;
            if (!logbuf) cudaMalloc(&logbuf, sizeof(unsigned long long) * 8 * 4096);
            cudaMemsetAsync(logbuf, 0, sizeof(unsigned long long) * 8 * 4096, st);
            a.log = logbuf;
            if (const char* e = std::getenv("NSDGT_LOGPTR")) *(unsigned long long**)std::strtoull(e, nullptr, 10) = logbuf;
        }
        a.beta = fp->beta7; a.S = fp->S7; a.lag = fp->lag7; a.nA = fp->nA; a.nB = fp->nB;
        cudaAccessPolicyWindow apw{};
        apw.base_ptr = ws;
        apw.num_bytes = fast_workspace_bytes(fp, W);
        apw.hitRatio = 1.0f;
        apw.hitProp = cudaAccessPropertyPersisting;
        apw.missProp = cudaAccessPropertyStreaming;
        const cudaAccessPolicyWindow* pw = fp->persist ? &apw : nullptr;
        if (fp->D == 512) (fp->minb7 == 4 ? launch7<512, 4> : launch7<512, 3>)(a, fp->grid, fp->smem, st, pw);
        else (fp->minb7 == 5 ? launch7<256, 5> : fp->minb7 == 4 ? launch7<256, 4> : launch7<256, 3>)(a, fp->grid, fp->smem, st, pw);
        return DGT_OK;
    }
    if (!fp->counters) {
        if (cudaMalloc(&fp->counters, sizeof(int) * fp->ngroups) != cudaSuccess) return DGT_ENOMEM;
    }
    if (cudaMemsetAsync(fp->counters, 0, sizeof(int) * fp->ngroups, st) != cudaSuccess) return DGT_ECUDA;
    FusedArgs a{};
    a.f = f; a.ws = ws; a.out = c; a.G = fp->G; a.Cj = fp->Cj; a.Rs = fp->Rs; a.Kmod = fp->Kmod;
    a.E = fp->E; a.rot = fp->rot; a.counters = fp->counters;
    a.dbg = std::getenv("NSDGT_DBG") ? std::atoi(std::getenv("NSDGT_DBG")) : 0;
    a.W = W; a.L = fp->L; a.c = fp->c; a.N = fp->N; a.nA = fp->nA; a.nB = fp->nB;
    a.GS = fp->GS; a.ngroups = fp->ngroups;
    cudaAccessPolicyWindow apw{};
    apw.base_ptr = ws;
    apw.num_bytes = fast_workspace_bytes(fp, W);
    apw.hitRatio = 1.0f;
    apw.hitProp = cudaAccessPropertyPersisting;
    apw.missProp = cudaAccessPropertyStreaming;
    // TMA descriptor of the output c viewed as W*M rows x 2N floats (box: 128 B x 256 rows)
    CUtensorMap cmap;
    std::memset(&cmap, 0, sizeof cmap);
    a.tma = fp->ncol == 16 && std::getenv("NSDGT_TMA") != nullptr;
    a.discard = std::getenv("NSDGT_DISCARD") != nullptr;
    if (a.tma) {
        static PFN_encodeTiled encode = nullptr;
        if (!encode) {
            cudaDriverEntryPointQueryResult q;
            if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q) != cudaSuccess ||
                !encode)
                return DGT_ECUDA;
        }
        cuuint64_t gdim[2] = {(cuuint64_t)2 * fp->N, (cuuint64_t)W * fp->MM};
        cuuint64_t gstr[1] = {(cuuint64_t)2 * fp->N * sizeof(float)};
        cuuint32_t box[2] = {32, 256};
        cuuint32_t est[2] = {1, 1};
        if (encode(&cmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, c, gdim, gstr, box, est, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return DGT_ECUDA;
    }
    fp->launch(a, cmap, fp->GS * fp->ngroups, fp->smem, st, fp->persist ? &apw : nullptr);
    return DGT_OK;
}

}  // namespace nsdgt
