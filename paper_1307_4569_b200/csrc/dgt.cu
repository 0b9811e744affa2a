// dgt.cu -- plan, window preparation, the Zak/factorisation kernels and the C ABI.
//
// The method:
//   Algorithm 1 of PAPER.md:852-900 reduces the nonseparable lattice (a, M, lambda)
//   to a separable one by the chirp P_{s1} (time shear) or by a length-L FFT and the
//   chirp P_{-s0} (frequency shear, with the Fourier-domain trick PAPER.md:902-919).
//   The separable DGT with a full-length window is the factorisation algorithm whose
//   cost is Eq. (rect-flops): Zak gather + d-point DFTs, p x q
//   products against the window factorisation, d-point DFTs, M-point FFTs.  The final
//   phase and index remap of Alg. 1 (lines 9-15 / 25-31) is fused into the store.
//
// Kernel A (zak_kernel):   one CTA = (signal w, residue block r0..r0+RB, l).  Gathers
//   f~(x(r,k,l,s)) with the chirp multiplied on load, DFT_d over s, products with the
//   plan's window factors, DFT_d over nu, and writes the intermediate C[w][j'][kappa][n'].
// Kernel B (out_kernel):   one CTA = (signal w, tile of consecutive n).  Reads the
//   columns C(., n), FFT over j, then the Alg. 1 phase + remap, and stores c[w][m][n].
#include <cuda_runtime.h>
#include <cufft.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <set>
#include <string>
#include <vector>

#include <cooperative_groups.h>
#include <nvtx3/nvToolsExt.h>

#include "../../include/nsdgt.h"
#include "cplx.cuh"
#include "fft_smem.cuh"
#include "planner.hpp"
#include "fast_kernels.cuh"

namespace nsdgt {

static thread_local std::string g_last_error;
static thread_local int64_t g_last_lmin = 0;

static int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

#define CUDA_TRY(expr)                                                                      \
    do {                                                                                    \
        cudaError_t _e = (expr);                                                            \
        if (_e != cudaSuccess)                                                              \
            return fail(_e == cudaErrorMemoryAllocation ? DGT_ENOMEM : DGT_ECUDA,           \
                        std::string(#expr) + ": " + cudaGetErrorString(_e));                \
    } while (0)

#define CUFFT_TRY(expr)                                                                     \
    do {                                                                                    \
        cufftResult _r = (expr);                                                            \
        if (_r != CUFFT_SUCCESS)                                                            \
            return fail(_r == CUFFT_ALLOC_FAILED ? DGT_ENOMEM : DGT_ECUFFT,                 \
                        std::string(#expr) + ": cufft status " + std::to_string((int)_r));  \
    } while (0)

// ---------------------------------------------------------------------------------
// plan-time device kernels (fp64 arithmetic, cast once to the working precision)
// ---------------------------------------------------------------------------------

// P_sigma(x) = exp(i pi r / L), r = (sigma * x^2 * (L+1)) mod 2L  (
// reading Z4: every factor reduced mod 2L first, exact in 128-bit integers).
__device__ __forceinline__ double2 chirp_val(int64_t sigma, int64_t x, int64_t L) {
    const unsigned __int128 twoL = (unsigned __int128)(2 * L);
    const unsigned __int128 sg = (unsigned __int128)(((sigma % (2 * L)) + 2 * L) % (2 * L));
    const unsigned __int128 xx = ((unsigned __int128)x * (unsigned __int128)x) % twoL;
    const unsigned __int128 lp = (unsigned __int128)((L + 1) % (2 * L));
    const unsigned __int128 r = (sg * xx % twoL) * lp % twoL;
    double s, c;
    sincospi((double)(int64_t)r / (double)L, &s, &c);
    return make_double2(c, s);
}

template <typename T>
__global__ void k_chirp_table(cx<T>* out, int64_t sigma, int64_t L) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < L; x += (int64_t)gridDim.x * blockDim.x) {
        double2 v = chirp_val(sigma, x, L);
        out[x] = mk<T>((T)v.x, (T)v.y);
    }
}

// out[s] = P_sigma(K s), s < n (the chirp's factor R of ZakArgs::chR)
template <typename T>
__global__ void k_chirp_stride(cx<T>* out, int64_t sigma, int64_t L, int64_t K, int64_t n) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
        const double2 v = chirp_val(sigma, (K * s) % (2 * L), L);
        out[s] = mk<T>((T)v.x, (T)v.y);
    }
}

// gt = P_sigma * g  (fp64), g given in precision Tin
template <typename Tin>
__global__ void k_window_time(double2* gt, const cx<Tin>* g, int64_t sigma, int64_t L) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < L; x += (int64_t)gridDim.x * blockDim.x) {
        double2 gv = make_double2((double)g[x].x, (double)g[x].y);
        double2 v = sigma ? cmul(chirp_val(sigma, x, L), gv) : gv;
        gt[x] = v;
    }
}

// after the fp64 FFT: ghat = P_{-s0} * FFT(P_{s1} g) / L   (Alg. 1 line 22)
__global__ void k_window_freq_post(double2* gh, int64_t sigma, int64_t L) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < L; x += (int64_t)gridDim.x * blockDim.x) {
        double2 v = cmul(chirp_val(sigma, x, L), gh[x]);
        gh[x] = make_double2(v.x / (double)L, v.y / (double)L);
    }
}

// Window factorisation: for r<c, u<q, k<p, nu<d
//   Gamma_r(k,u;nu) = sum_{s<d} g~(x(r,k,u,s)) exp(-2 pi i s nu / d),
//   x(r,k,u,s) = r + c ((k q + p u + s p q) mod (L/c)),
// stored as G[((r*q + u)*p + k)*d + nu] = conj(Gamma)/d.  Direct sum in fp64 with exact
// integer reduction of s*nu mod d (plan time only).
template <typename T>
__global__ void k_window_factor(cx<T>* G, const double2* gt, int64_t L, int64_t c, int64_t d, int64_t p,
                                int64_t q) {
    const int64_t total = c * q * p * d;
    const int64_t Lc = L / c;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t nu = i % d;
        const int64_t k = (i / d) % p;
        const int64_t u = (i / (d * p)) % q;
        const int64_t r = i / (d * p * q);
        double sr = 0.0, si = 0.0;
        int64_t e = 0;  // s*nu mod d
        for (int64_t s = 0; s < d; ++s) {
            const int64_t x = r + c * ((k * q + p * u + s * p * q) % Lc);
            double sn, cs;
            sincospi(-2.0 * (double)e / (double)d, &sn, &cs);
            const double2 gv = gt[x];
            sr += gv.x * cs - gv.y * sn;
            si += gv.x * sn + gv.y * cs;
            e += nu;
            if (e >= d) e -= d;
        }
        G[i] = mk<T>((T)(sr / (double)d), (T)(-si / (double)d));
    }
}

template <typename T>
__global__ void k_twiddles(cx<T>* tw, int64_t n) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        double s, c;
        sincospi(-2.0 * (double)k / (double)n, &s, &c);
        tw[k] = mk<T>((T)c, (T)s);
    }
}

// W_n^k for k < count (a prefix of the length-n table)
template <typename T>
__global__ void k_twiddles_prefix(cx<T>* tw, int64_t n, int64_t count) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < count; k += (int64_t)gridDim.x * blockDim.x) {
        double s, c;
        sincospi(-2.0 * (double)k / (double)n, &s, &c);
        tw[k] = mk<T>((T)c, (T)s);
    }
}

// T-branch post tables (Alg. 1 lines 8-12): E(n) = exp(i pi (C1 n^2 mod 2N)/N) and the
// row rotation rot(n) = ceil(s1 a n / b) mod M (the printed ((-s1 n a + m b) mod L) div b
// equals (m - rot(n)) mod M; reading Z5).
template <typename T>
__global__ void k_post_time(cx<T>* E, int* rot, int64_t N, int64_t C1, int64_t s1, int64_t a, int64_t b,
                            int64_t M) {
    for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < N; n += (int64_t)gridDim.x * blockDim.x) {
        const unsigned __int128 twoN = 2 * N;
        const int64_t e = (int64_t)(((unsigned __int128)C1 * (((unsigned __int128)n * n) % twoN)) % twoN);
        double s, c;
        sincospi((double)e / (double)N, &s, &c);
        E[n] = mk<T>((T)c, (T)s);
        const __int128 x = (__int128)s1 * a * n;
        rot[n] = (int)(((x + b - 1) / b) % M);
    }
}

// F-branch phase table ptab[e] = exp(i pi e / N), e < 2N.
template <typename T>
__global__ void k_phase_table(cx<T>* P, int64_t N) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < 2 * N; e += (int64_t)gridDim.x * blockDim.x) {
        double s, c;
        sincospi((double)e / (double)N, &s, &c);
        P[e] = mk<T>((T)c, (T)s);
    }
}

template <typename T>
__global__ void k_cast_to(cx<T>* out, const double2* in, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = mk<T>((T)in[i].x, (T)in[i].y);
}

// ---------------------------------------------------------------------------------
// execute-time kernels (generic path)
// ---------------------------------------------------------------------------------

// F-branch front end: out = P_pre(x) * f(x) (promotes real input), written complex.
template <typename T>
__global__ void k_prechirp(cx<T>* out, const void* f, int real_in, const cx<T>* __restrict__ chirp, int64_t L,
                           int64_t total) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        cx<T> v;
        if (real_in) v = mk<T>(((const T*)f)[i], T(0));
        else v = ((const cx<T>*)f)[i];
        if (chirp) v = cmul(v, chirp[i % L]);
        out[i] = v;
    }
}

#ifdef NSDGT_KTRACE
// experiment builds only (tools/ktrace.py): %globaltimer at phase boundaries of block (0, 0)
__device__ unsigned long long g_ktrace[64];
#define KTRACE(k)                                                                               \
    do {                                                                                        \
        if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {                           \
            unsigned long long t_;                                                              \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                              \
            g_ktrace[k] = t_;                                                                   \
        }                                                                                       \
    } while (0)
#else
#define KTRACE(k) do { } while (0)
#endif

// Launch with the programmatic-serialisation attribute (PDL; cplx.cuh pdl_wait / pdl_trigger):
// the kernel's launch and prologue overlap its predecessor's tail.  NSDGT_PDL_OFF: plain launch.
static bool pdl_enabled() {
    static const bool on = std::getenv("NSDGT_PDL_OFF") == nullptr;
    return on;
}
template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// The same with a thread-block cluster of cx CTAs along x.
template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl_cluster(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                      unsigned cx, Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    at[1].id = cudaLaunchAttributeClusterDimension;
    at[1].val.clusterDim.x = cx;
    at[1].val.clusterDim.y = 1;
    at[1].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

struct ZakArgs {
    const void* f;     // [W][L] complex (or real) input of the inner separable DGT
    int real_in;
    const void* chirp;  // [L] multiplier applied on load (nullable)
    const void* G;      // window factors [c][q][p][d]
    void* C;            // intermediate [W][iM][q][d]
    int64_t L, c, d, p, q, iM;
    int RB;
    int allu;           // p = 1: products and DFT_d of all q values of u in one pass (smem 2 q RB d)
    unsigned char* gscr;   // non-null: per-CTA buffers in global memory (d too large for shared)
    int64_t gstride;       // bytes per CTA in gscr
    Radices rd;
    const void* tw;     // twiddles of length d
    int cnj;            // zak_ct only: intermediate stored [W][n][iM] (n = kappa + q n', j fastest)
    // zak_ct only (chR non-null): the load chirp factorised on the gather's lattice x = x0 + K s
    // (K = c q, x0 = r + c l, L = K d): P(x0 + K s) = P(x0) W_d^{-sigD x0 s} R(s), R(s) = P(K s),
    // sigD = sigma (L + 1) mod d.  The gather multiplies R(s) (a d-entry table instead of the
    // length-L one), and the W_d modulation is the index shift m0 = -sigD x0 (mod d) of the
    // Zak DFT's output, applied with P(x0) where the products read it.
    const void* chR;
    int sigD;
};

template <typename T>
__global__ void __launch_bounds__(256) zak_kernel(ZakArgs A) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    using C = cx<T>;
    pdl_trigger();
    pdl_wait();
    const int64_t d = A.d, p = A.p, q = A.q, c = A.c, L = A.L;
    const int RB = A.RB;
    const int nrb = (int)((c + RB - 1) / RB);
    const int rblk = blockIdx.x % nrb;
    const int l = blockIdx.x / nrb;
    const int64_t w = blockIdx.y;
    const int64_t r0 = (int64_t)rblk * RB;
    const int nr = (int)((c - r0) < RB ? (c - r0) : RB);
    unsigned char* sbase = A.gscr ? A.gscr + ((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * A.gstride : smem_raw;
    C* bufA = (C*)sbase;                    // RB*p*d
    C* bufB = bufA + (size_t)RB * p * d;    // RB*p*d (>= RB*d)
    C* bufY = bufB + (size_t)RB * p * d;    // RB*d
    const C* __restrict__ tw = (const C*)A.tw;
    const C* __restrict__ chirp = (const C*)A.chirp;
    const int64_t Lc = L / c;

    // 1. gather f~(x(r,k,l,s)), x = r + c((k q + p l + s p q) mod (L/c)), rr fastest.
    //    32-bit index arithmetic within a signal (the host checks L < 2^31).
    const int ng = nr * (int)p * (int)d;
    const int di = (int)d, pi = (int)p, qi = (int)q, ci = (int)c, Lci = (int)Lc;
    const int base_kq = pi * l;                     // p l
    const T* fr = (const T*)A.f + w * L;            // real input
    const C* fc = (const C*)A.f + w * L;
    for (int i = threadIdx.x; i < ng; i += blockDim.x) {
        const int rr = i % nr;
        const int ks = i / nr;  // k*d + s
        const int s = ks % di, k = ks / di;
        int z = k * qi + base_kq + s * pi * qi;     // < p q (d + 1): fits
        z %= Lci;
        const int x = (int)r0 + rr + ci * z;
        C v;
        if (A.real_in) v = mk<T>(fr[x], T(0));
        else v = fc[x];
        if (chirp) v = cmul(v, chirp[x]);
        bufA[(rr * pi + k) * di + s] = v;
    }
    __syncthreads();
    if (A.allu) {
        // p = 1, all u at once: DFT_d of the nr gathered columns, the q nr products, one
        // batched DFT_d of q nr sequences, one scatter (3 barrier-separated phases of q x
        // the work instead of q rounds of products + DFT + scatter).  Buffers: two regions of
        // q RB d; Phi lives in the first nr d of one of them.
        C* R1 = bufA;
        C* R2 = bufA + (size_t)qi * RB * d;
        C* phi = fft_smem<T>(R1, R2, A.rd, nr, di, tw);
        C* Yb = (phi == R1) ? R2 : R1;
        const C* __restrict__ G = (const C*)A.G;
        const int nrd = nr * di;
        for (int i = threadIdx.x; i < qi * nrd; i += blockDim.x) {
            const int u = i / nrd, rem = i - u * nrd;
            const int rr = rem / di, nu = rem - rr * di;
            Yb[i] = cmul(phi[rem], G[(((int)r0 + rr) * qi + u) * di + nu]);
        }
        __syncthreads();
        C* Y = fft_smem<T>(Yb, phi, A.rd, qi * nr, di, tw);
        C* Cw = (C*)A.C + w * A.iM * q * d;
        const int jbase = (int)(r0 + c * ((l * p) % q));
        for (int i = threadIdx.x; i < qi * nrd; i += blockDim.x) {
            const int u = i / nrd, rem = i - u * nrd;
            const int rr = rem / di, np = rem - rr * di;
            const int kappa = ((l - u) % qi + qi) % qi;
            int tau = di - np - (l < u ? 1 : 0);       // (-n' - [l < u]) mod d
            if (tau >= di) tau -= di;
            if (tau < 0) tau += di;
            Cw[((jbase + rr) * qi + kappa) * di + np] = Y[(u * nr + rr) * di + tau];
        }
        return;
    }
    // 2. DFT_d over s for nr*p sequences
    C* phi = fft_smem<T>(bufA, bufB, A.rd, nr * (int)p, (int)d, tw);
    C* free0 = (phi == bufA) ? bufB : bufA;
    const C* __restrict__ G = (const C*)A.G;
    C* Cout = (C*)A.C;
    const int64_t jp = (l * p) % q;  // j' = r + c*((l p) mod q)
    for (int u = 0; u < q; ++u) {
        // 3. Y(nu) = sum_k Phi_r(k,l;nu) * conj(Gamma_r(k,u;nu))/d
        for (int64_t i = threadIdx.x; i < (int64_t)nr * d; i += blockDim.x) {
            const int rr = (int)(i / d);
            const int64_t nu = i % d;
            const C* gk = G + (((r0 + rr) * q + u) * p) * d + nu;
            C acc = cmul(phi[(rr * p) * d + nu], gk[0]);
            for (int64_t k = 1; k < p; ++k) acc = acc + cmul(phi[(rr * p + k) * d + nu], gk[k * d]);
            free0[rr * d + nu] = acc;
        }
        __syncthreads();
        // 4. DFT_d over nu
        C* Y = fft_smem<T>(free0, bufY, A.rd, nr, (int)d, tw);
        // 5. scatter T_r(l,u;tau) to n = (l - u - q tau) mod N:
        //    kappa = (l-u) mod q, n' = (-tau - [l<u]) mod d, C[w][j'][kappa][n']
        const int kappa = (int)(((l - u) % q + q) % q);
        const int off = (l < u) ? 1 : 0;
        C* Cw = Cout + w * A.iM * q * d;
        const int jbase = (int)(r0 + c * jp);
        for (int i = threadIdx.x; i < nr * di; i += blockDim.x) {
            const int rr = i / di;
            const int np = i - rr * di;                // destination n'
            int tau = di - np - off;                   // (-n' - off) mod d
            if (tau >= di) tau -= di;
            if (tau < 0) tau += di;
            Cw[((jbase + rr) * qi + kappa) * di + np] = Y[rr * di + tau];
        }
        __syncthreads();
    }
}

// All-u Zak kernel with compile-time inner length D, q = Q and RBC columns per CTA (config 4:
// D = 180, Q = 4, RBC = 4 for c128).  Same phases as zak_kernel's all-u mode (gather with
// the chirp on load, DFT_D of the RBC columns, the Q RBC window products, one DFT_D of Q RBC
// sequences, scatter), but every index divides by a constant, each thread issues all its
// global loads of a phase before using them, and p = 1 makes the gather index
// z = l + Q s < L/c (no reduction).
// Row order of zak_ct's RBC-column loops: rows (stride D in shared memory) are visited in
// aligned blocks of 8 with the upper half of the columns shifted by 2 rows, so one shared-memory
// wavefront (4 x 16-byte or 8 x 8-byte columns, 2 rows) hits distinct banks -- D e / 16 B is
// 4 mod 8 for d = 180, which made column c and c + RBC/2 collide.  A permutation within each
// block (ragged last block unchanged); the global side still moves RBC consecutive elements.
template <int D, int RBC, int E>
__device__ __forceinline__ int zrow(int g, int rr, int G) {
    if constexpr (RBC * E == 64 && D % 8 == 4)
        return (g | 7) < G ? ((g & ~7) | ((g + 2 * (rr / (RBC / 2))) & 7)) : g;
    else
        return g;
}

template <typename T, int D, int Q, int RBC, int NT = 256>
__global__ void __launch_bounds__(NT, 512 / NT) zak_ct_kernel(ZakArgs A) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    using C = cx<T>;
    constexpr int NG = (RBC * D + NT - 1) / NT, NP = (Q * RBC * D + NT - 1) / NT;
    const int c = (int)A.c;
    const int nrb = c / RBC;
    const int rblk = blockIdx.x % nrb, l = blockIdx.x / nrb;
    const int64_t w = blockIdx.y;
    const int r0 = rblk * RBC;
    // d = 720 (one column per CTA, config 2), experiment builds: the window factors loaded
    // first (a plan table: before the PDL wait) -- slower, the gather's loads queue behind them
#ifndef NSDGT_ZCT_EG   // window factors before the gather: measured slower (33.0 vs 31.8 us, config 2)
#define NSDGT_ZCT_EG 0
#endif
    constexpr bool EG = D == 720 && NSDGT_ZCT_EG;
    C gv[NP];
    KTRACE(0);
    pdl_trigger();
    if constexpr (EG) {
        const C* __restrict__ G = (const C*)A.G;
#pragma unroll
        for (int it = 0; it < NP; ++it) {
            const int i = threadIdx.x + it * NT;
            if (i < Q * RBC * D) {
                const int u = i / (RBC * D), rem = i % (RBC * D);
                gv[it] = __ldg(G + ((r0 + rem / D) * Q + u) * D + rem % D);
            }
        }
    }
    pdl_wait();
    C* R1 = (C*)smem_raw;
    C* R2 = R1 + Q * RBC * D;
    const C* __restrict__ tw = (const C*)A.tw;
    const C* __restrict__ chirp = (const C*)A.chirp;
    const int tid = threadIdx.x;
    {
        // gather f~(r0 + rr + c (l + Q s)), rr fastest (RBC consecutive residues per row s)
        const C* fc = (const C*)A.f + w * A.L;
        const T* fr = (const T*)A.f + w * A.L;
        C v[NG];
#pragma unroll
        for (int it = 0; it < NG; ++it) {
            const int i = tid + it * NT;
            if (i < RBC * D) {
                const int rr = i % RBC, s = zrow<D, RBC, sizeof(C)>(i / RBC, rr, D);
                const int x = r0 + rr + c * (l + Q * s);
                v[it] = A.real_in ? mk<T>(fr[x], T(0)) : fc[x];
            }
        }
        if (A.chR) {
            const C* __restrict__ R = (const C*)A.chR;
#pragma unroll
            for (int it = 0; it < NG; ++it) {
                const int i = tid + it * NT;
                if (i < RBC * D) {
                    const int rr = i % RBC, s = zrow<D, RBC, sizeof(C)>(i / RBC, rr, D);
                    v[it] = cmul(v[it], __ldg(R + s));
                }
            }
        } else if (chirp) {
#pragma unroll
            for (int it = 0; it < NG; ++it) {
                const int i = tid + it * NT;
                if (i < RBC * D) {
                    const int rr = i % RBC, s = zrow<D, RBC, sizeof(C)>(i / RBC, rr, D);
                    v[it] = cmul(v[it], __ldg(chirp + r0 + rr + c * (l + Q * s)));
                }
            }
        }
#pragma unroll
        for (int it = 0; it < NG; ++it) {
            const int i = tid + it * NT;
            if (i < RBC * D) R1[(i % RBC) * D + zrow<D, RBC, sizeof(C)>(i / RBC, i % RBC, D)] = v[it];
        }
    }
    __syncthreads();
    KTRACE(1);
    C* phi = fft_ct<T, D>(R1, R2, RBC, tw);     // Phi in the first RBC D of R1 or R2
    KTRACE(2);
    C* Yb = phi == R1 ? R2 : R1;
    {
        const C* __restrict__ G = (const C*)A.G;
        if constexpr (!EG) {
#pragma unroll
            for (int it = 0; it < NP; ++it) {
                const int i = tid + it * NT;
                if (i < Q * RBC * D) {
                    const int u = i / (RBC * D), rem = i % (RBC * D);
                    gv[it] = __ldg(G + ((r0 + rem / D) * Q + u) * D + rem % D);
                }
            }
        }
        if (A.chR) {
            // Phi(nu) = P(x0) U((nu + m0) mod D), U the DFT of f R (see ZakArgs::chR)
#pragma unroll
            for (int it = 0; it < NP; ++it) {
                const int i = tid + it * NT;
                if (i < Q * RBC * D) {
                    const int rem = i % (RBC * D), rr = rem / D, nu = rem % D;
                    const int x0 = r0 + rr + c * l;
                    int m0 = D - (int)(((long long)A.sigD * x0) % D);
                    if (m0 >= D) m0 -= D;
                    int nn = nu + m0;
                    if (nn >= D) nn -= D;
                    const C P0 = __ldg(chirp + x0);
                    Yb[i] = cmul(cmul(phi[rr * D + nn], P0), gv[it]);
                }
            }
        } else {
#pragma unroll
            for (int it = 0; it < NP; ++it) {
                const int i = tid + it * NT;
                if (i < Q * RBC * D) Yb[i] = cmul(phi[i % (RBC * D)], gv[it]);
            }
        }
    }
    __syncthreads();
    KTRACE(3);
    C* Y = fft_ct<T, D>(Yb, phi, Q * RBC, tw);   // Phi is dead: its buffer is the scratch
    KTRACE(4);
    C* Cw = (C*)A.C + w * A.iM * Q * D;
    const int jbase = r0 + c * (l % Q);
    if (A.cnj) {
        // [n][j] layout: rr fastest, RBC consecutive j per (kappa, n') (RBC * e = 64 B runs)
        const int iM = (int)A.iM;
#pragma unroll
        for (int it = 0; it < NP; ++it) {
            const int i = tid + it * NT;
            if (i < Q * RBC * D) {
                const int rr = i % RBC, g = zrow<D, RBC, sizeof(C)>(i / RBC, rr, Q * D);
                const int u = g / D, np = g % D;
                const int kappa = (l - u + Q) % Q;
                int tau = D - np - (l < u ? 1 : 0);
                if (tau >= D) tau -= D;
                Cw[(int64_t)(kappa + Q * np) * iM + jbase + rr] = Y[(u * RBC + rr) * D + tau];
            }
        }
        return;
    }
#pragma unroll
    for (int it = 0; it < NP; ++it) {
        const int i = tid + it * NT;
        if (i < Q * RBC * D) {
            const int u = i / (RBC * D), rem = i % (RBC * D);
            const int rr = rem / D, np = rem % D;
            const int kappa = (l - u + Q) % Q;
            int tau = D - np - (l < u ? 1 : 0);    // (-n' - [l < u]) mod D
            if (tau >= D) tau -= D;
            Cw[((jbase + rr) * Q + kappa) * D + np] = Y[(u * RBC + rr) * D + tau];
        }
    }
#ifdef NSDGT_KTRACE
    __syncthreads();
#endif
    KTRACE(5);
}

#include "zak_rr.cuh"

struct OutArgs {
    const void* C;  // [W][iM][q][d]
    void* out;      // [W][M][N]
    int64_t iM, iN, q, d;
    int NT;         // columns per CTA: T-branch consecutive inner n; F-branch (grouped) n = kappa + q (n'0 + i)
    unsigned char* gscr;   // non-null: per-CTA buffers in global memory (iM too large for shared)
    int64_t gstride;
    int grouped;    // 1: CTA x = (kappa, block of NT consecutive n'), contiguous loads
    Radices rd;
    const void* tw;  // twiddles of length iM
    int cnj;         // out_f4096 only: intermediate stored [W][n][iM] (see ZakArgs::cnj)
    int branch;
    // T-branch
    const void* E;
    const int* rot;
    int64_t M, N;
    // F-branch
    const void* ptab;
    int64_t L, b, Nr, ar, s1, C1, C2, C3, C4, C5, C6;
    int64_t sar;                   // (-s1 a_r) mod L
    unsigned int D1, D5, DX;       // 256 C1 mod 2N, 256 C5 mod 2N, 256 sar mod L (k -> k - 256)
    unsigned int invb;             // floor((2^32 - 1) / b)
    unsigned long long inv2N, invL;   // Barrett constants floor(2^64 / 2N), floor(2^64 / L)
};

// x mod m for x < 2^64, 2 <= m < 2^32 (Barrett: inv = floor((2^64 - 1) / m); the quotient
// estimate is at most 2 short)
__device__ __forceinline__ unsigned int bmod(unsigned long long x, unsigned int m, unsigned long long inv) {
    const unsigned long long qe = __umul64hi(x, inv);
    unsigned long long r = x - qe * m;
    if (r >= m) r -= m;
    if (r >= m) r -= m;
    return (unsigned int)r;
}

// F-branch output remap (Alg. 1 lines 24-31): c[kt][mt] = E(k,m) c_r[(-k) mod N_r][m]; the
// inner channel is the FFT output index kc = (-k) mod N_r, the inner time index m = n.
//   sq = (C1 k + C2 m) mod 2N,  e = (C3 sq^2 - m (C4 m + C5 k)) mod 2N,
//   mt = sq mod N,  kt = ((-s1 a_r k + C6 m) mod L) div b
// The k-dependent residues come from the plan's per-channel table, the m-dependent ones
// are per-column constants; every reduction is exact (Barrett, 64-bit products).
struct FbCol {
    unsigned int mD, mA, mC4, mT;
};
__device__ __forceinline__ FbCol fb_col(const OutArgs& A, unsigned long long m) {
    const unsigned int twoN = (unsigned int)(2 * A.N), Lu = (unsigned int)A.L;
    FbCol c;
    c.mD = bmod(m, twoN, A.inv2N);
    c.mA = bmod((unsigned long long)A.C2 * c.mD, twoN, A.inv2N);
    c.mC4 = bmod((unsigned long long)A.C4 * c.mD, twoN, A.inv2N);
    c.mT = bmod((unsigned long long)(A.C6 % A.L) * (m % A.L), Lu, A.invL);
    return c;
}
__device__ __forceinline__ unsigned int submod(unsigned int x, unsigned int dlt, unsigned int m) {
    return x >= dlt ? x - dlt : x + m - dlt;
}
// The residues of one column along kc, kc + 256, kc + 512, ... (k = N_r - kc decreases by
// 256 per step): sq = (C1 k + C2 m) mod 2N, uu = (C4 m + C5 k) mod 2N, t2 = m uu mod 2N and
// xx = (-s1 a_r k + C6 m) mod L are affine in k, so each step is a subtraction mod 2N / L
// (the deltas D1 = 256 C1, D5 = 256 C5, DX = 256 (-s1 a_r) are plan constants); only the
// C3 sq^2 term (0 for config 4) needs a product per coefficient.
template <typename C>
struct FbIter {
    unsigned int sq, uu, t2, xx, dt2;
    C ph, dph;   // C3 = 0: the phase exp(i pi e / N), e = -t2, advances by a factor per step
};
template <typename C>
__device__ __forceinline__ FbIter<C> fb_iter(const OutArgs& A, const FbCol& cc, unsigned long long k) {
    const unsigned int twoN = (unsigned int)(2 * A.N), Lu = (unsigned int)A.L;
    FbIter<C> it;
    it.sq = bmod((unsigned long long)A.C1 * k, twoN, A.inv2N) + cc.mA;
    if (it.sq >= twoN) it.sq -= twoN;
    it.uu = cc.mC4 + bmod((unsigned long long)A.C5 * k, twoN, A.inv2N);
    if (it.uu >= twoN) it.uu -= twoN;
    it.t2 = bmod((unsigned long long)cc.mD * it.uu, twoN, A.inv2N);
    it.xx = (A.sar ? bmod((unsigned long long)A.sar * k, Lu, A.invL) : 0u) + cc.mT;
    if (it.xx >= Lu) it.xx -= Lu;
    it.dt2 = bmod((unsigned long long)cc.mD * A.D5, twoN, A.inv2N);
    if (!A.C3) {
        const C* P = (const C*)A.ptab;
        it.ph = __ldg(P + (it.t2 ? twoN - it.t2 : 0u));
        it.dph = __ldg(P + it.dt2);
    }
    return it;
}
template <typename C>
__device__ __forceinline__ void fb_step(const OutArgs& A, FbIter<C>& it) {
    const unsigned int twoN = (unsigned int)(2 * A.N);
    it.sq = submod(it.sq, A.D1, twoN);
    it.uu = submod(it.uu, A.D5, twoN);
    it.t2 = submod(it.t2, it.dt2, twoN);
    it.xx = submod(it.xx, A.DX, (unsigned int)A.L);
    if (!A.C3) it.ph = cmul(it.ph, it.dph);
}
template <typename C>
__device__ __forceinline__ void fb_dest(const OutArgs& A, const FbIter<C>& it, size_t* dst, C* phase) {
    const unsigned int twoN = (unsigned int)(2 * A.N), Nn = (unsigned int)A.N;
    C ph;
    if (A.C3) {
        const unsigned int s2 = bmod((unsigned long long)it.sq * it.sq, twoN, A.inv2N);
        const unsigned int t1 = bmod((unsigned long long)A.C3 * s2, twoN, A.inv2N);
        ph = __ldg((const C*)A.ptab + submod(t1, it.t2, twoN));
    } else {
        ph = it.ph;
    }
    const unsigned int mt = it.sq >= Nn ? it.sq - Nn : it.sq;
    // kt = xx div b (32-bit Barrett, two corrections)
    const unsigned int bu = (unsigned int)A.b;
    unsigned int kt = __umulhi(it.xx, A.invb);
    unsigned int r = it.xx - kt * bu;
    if (r >= bu) { r -= bu; ++kt; }
    if (r >= bu) ++kt;
    *dst = (size_t)kt * Nn + mt;
    *phase = ph;
}
template <typename C>
__device__ __forceinline__ void fb_put(const OutArgs& A, C* out, const FbIter<C>& it, C val) {
    size_t dst;
    C ph;
    fb_dest(A, it, &dst, &ph);
    out[dst] = cmul(ph, val);
}
// column m, coefficients kc = kc0 + 256 i, i < cnt (kc0 < 256; CNT > 0: compile-time count,
// fully unrolled so get(i) may index registers)
template <int CNT, typename C, class Get>
__device__ __forceinline__ void fb_column(const OutArgs& A, C* out, unsigned long long m, unsigned int kc0, int cnt,
                                          Get&& get) {
    const FbCol cc = fb_col(A, m);
    const int n = CNT > 0 ? CNT : cnt;
    if (n <= 0) return;
    // k = N_r - kc for kc > 0, k = 0 for kc = 0 (then the sequence restarts at N_r - 256)
    FbIter<C> it = fb_iter<C>(A, cc, kc0 ? (unsigned long long)A.Nr - kc0 : 0ull);
#pragma unroll
    for (int i = 0; i < (CNT > 0 ? CNT : 1 << 30); ++i) {
        if (CNT <= 0 && i >= n) break;
        if (i == 1 && kc0 == 0) it = fb_iter<C>(A, cc, (unsigned long long)A.Nr - 256u);
        else if (i > 0) fb_step(A, it);
        fb_put(A, out, it, get(i));
    }
}

// fb_column's iteration, handing each coefficient's destination and phase to put(i, dst, ph)
template <int CNT, typename C, class Put>
__device__ __forceinline__ void fb_column_dest(const OutArgs& A, unsigned long long m, unsigned int kc0, Put&& put) {
    const FbCol cc = fb_col(A, m);
    FbIter<C> it = fb_iter<C>(A, cc, kc0 ? (unsigned long long)A.Nr - kc0 : 0ull);
#pragma unroll
    for (int i = 0; i < CNT; ++i) {
        if (i == 1 && kc0 == 0) it = fb_iter<C>(A, cc, (unsigned long long)A.Nr - 256u);
        else if (i > 0) fb_step(A, it);
        size_t dst;
        C ph;
        fb_dest(A, it, &dst, &ph);
        put(i, dst, ph);
    }
}

// IMCT > 0: compile-time inner channel count (its DFT by fft_ct; config 2: 200)
template <typename T, int IMCT = 0>
__global__ void __launch_bounds__(256) out_kernel(OutArgs A) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    using C = cx<T>;
    pdl_trigger();
    const int64_t iM = IMCT ? IMCT : A.iM, iN = A.iN, q = A.q, d = A.d;
    const int NT = A.NT;
    const int iMi = (int)iM, qi = (int)q, di = (int)d;
    // column cl of this CTA is inner n = nb + ns * cl: T-branch nb = x NT, ns = 1 (consecutive
    // n, coalesced stores); F-branch grouped: x = kappa + q * blk, nb = kappa + q NT blk,
    // ns = q, so C(j, n) = [j][kappa][n'] is contiguous over cl (the F-branch stores are
    // scattered by the remap anyway)
    int64_t nb, ns;
    int nt;
    if (A.grouped) {
        const int kap = (int)(blockIdx.x % q), blk = (int)(blockIdx.x / q);
        nb = kap + q * (int64_t)blk * NT;
        ns = q;
        nt = (int)((d - (int64_t)blk * NT) < NT ? (d - (int64_t)blk * NT) : NT);
    } else {
        nb = (int64_t)blockIdx.x * NT;
        ns = 1;
        nt = (int)((iN - nb) < NT ? (iN - nb) : NT);
    }
    const int64_t w = blockIdx.y;
    // T-branch with blockDim = 256 and nt | 256 (this tile's column count): thread t's output
    // column is always nb + t mod nt, so its E(n) and rot(n) (plan tables) are loaded once,
    // before the PDL wait
    KTRACE(10);
    C Et = mk<T>(T(1), T(0));
    int rott = 0;
#ifndef NSDGT_OUT_COLFIX   // experiment builds: 0 reads E(n), rot(n) per element (config 2: 33.6 vs 31.8 us)
#define NSDGT_OUT_COLFIX 1
#endif
    const bool colfix = NSDGT_OUT_COLFIX && A.branch != DGT_BRANCH_FREQ && nt > 0 && 256 % nt == 0;
    if (colfix) {
        const int n = (int)nb + (int)(threadIdx.x % nt);
        Et = __ldg((const C*)A.E + n);
        rott = __ldg(A.rot + n);
    }
    pdl_wait();
    unsigned char* sbase = A.gscr ? A.gscr + ((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * A.gstride : smem_raw;
    C* bufA = (C*)sbase;
    C* bufB = bufA + (size_t)NT * iM;
    const C* __restrict__ Cin = (const C*)A.C + w * iM * iN;
    // load columns: C(j, n) stored at [j][n mod q][n div q] (32-bit indices within a signal);
    // eight independent loads in flight per thread
    if (IMCT > 0 && (nt == 16 || nt == 20) && qi == 4 && ns == 1 && (nb & 3) == 0) {
        // config 2 (M' = 200, q = 4, nt consecutive columns = 4 kappa x nt/4 n'): element
        // i = (j, kappa, n'') with n'' fastest, so nt/4 lanes read contiguous bytes of row
        // (j, kappa) (the generic loop's lanes each touch another row)
        const int nq0 = (int)nb >> 2, NQ = nt >> 2;
        constexpr int U = (20 * (IMCT > 0 ? IMCT : 1) + 255) / 256;
        C v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = threadIdx.x + 256 * u;
            if (i < nt * iMi) {
                const int t = i / NQ, nn = i - t * NQ, kap = t & 3, j = t >> 2;
                v[u] = Cin[(j * 4 + kap) * di + nq0 + nn];
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = threadIdx.x + 256 * u;
            if (i < nt * iMi) {
                const int t = i / NQ, nn = i - t * NQ;
                bufA[(4 * nn + (t & 3)) * iMi + (t >> 2)] = v[u];   // column cl = 4 n'' + kappa
            }
        }
    } else {
        const int total = nt * iMi, nbi = (int)nb, nsi = (int)ns;
        constexpr int U = IMCT > 0 ? 16 : 8;   // config 2 (NT = 16, M' = 200): all loads in one round
        for (int i0 = threadIdx.x; i0 < total; i0 += U * blockDim.x) {
            C v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int i = i0 + u * blockDim.x;
                if (i < total) {
                    const int cl = i % nt, j = i / nt;
                    const int n = nbi + nsi * cl;
                    const int nq = n / qi;
                    v[u] = Cin[(j * qi + (n - nq * qi)) * di + nq];
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int i = i0 + u * blockDim.x;
                if (i < total) bufA[(i % nt) * iMi + i / nt] = v[u];
            }
        }
    }
    __syncthreads();
    KTRACE(11);
    C* X;
    if constexpr (IMCT > 0) X = fft_ct<T, IMCT>(bufA, bufB, nt, (const C*)A.tw);
    else X = fft_smem<T>(bufA, bufB, A.rd, nt, (int)iM, (const C*)A.tw);
    KTRACE(12);
    if (A.branch != DGT_BRANCH_FREQ) {
        // c[w][(m - rot(n)) mod M][n] = E(n) * X(m, n)   (Alg. 1 lines 9-12)
        C* out = (C*)A.out + w * A.M * A.N;
        const C* E = (const C*)A.E;
        const int Mi = (int)A.M, Ni = (int)A.N;
        for (int i = threadIdx.x; i < nt * iMi; i += blockDim.x) {
            const int cl = i % nt;
            const int mo = i / nt;
            const int n = (int)nb + cl;
            int m = mo + (colfix ? rott : A.rot[n]);
            if (m >= Mi) m -= Mi;
            out[mo * Ni + n] = cmul(colfix ? Et : E[n], X[cl * iMi + m]);
        }
#ifdef NSDGT_KTRACE
        __syncthreads();
#endif
        KTRACE(13);
    } else {
        C* out = (C*)A.out + w * A.M * A.N;
        for (int cl = 0; cl < nt; ++cl) {
            const C* Xc = X + cl * iMi;
            const int kc0 = threadIdx.x;   // blockDim.x == 256
            fb_column<0>(A, out, (unsigned long long)(nb + ns * cl), (unsigned int)kc0, (iMi - kc0 + 255) / 256,
                      [&](int i) { return Xc[kc0 + 256 * i]; });
        }
    }
}

// F-branch output kernel for N_r = iM = 4096 = 16^3 (config 4): one CTA of 256 threads per
// inner column m.  Three register radix-16 passes with two shared-memory exchanges in one
// padded buffer (16 x 272 elements) instead of three Stockham ping-pong passes over two
// full-column buffers: 70 KB (c128) per CTA, so 3 CTAs share an SM; the 16 loads of pass 1
// come straight from the intermediate C[w][j][kappa][n'] (j = t + 256 r).
//   pass 1 (lane t):         Y(t, k1)  = W_4096^{t k1} sum_r x(t + 256 r) W_16^{r k1}
//   pass 2 (lane k1, t1):    Z(k1, t1, k2) = W_256^{t1 k2} sum_t2 Y(t1 + 16 t2, k1) W_16^{t2 k2}
//   pass 3 (lane k1, k2):    X(k1 + 16 k2 + 256 k3) = sum_t1 Z(k1, t1, k2) W_16^{t1 k3}
// v[k] *= W_4096^{s k}, k = 1..15, from one table load (W^s), three squarings and eleven
// products (at most six roundings per twiddle; fifteen scattered loads per lane was the
// kernel's largest L1 cost)
template <typename C>
__device__ __forceinline__ void twiddle15(C* v, const C* __restrict__ tw, int s) {
    const C w1 = __ldg(tw + (s & 4095));
    const C w2 = cmul(w1, w1), w4 = cmul(w2, w2), w8 = cmul(w4, w4);   // squarings: one load
    const C w3 = cmul(w1, w2), w5 = cmul(w1, w4), w6 = cmul(w2, w4), w7 = cmul(w3, w4);
    v[1] = cmul(v[1], w1); v[2] = cmul(v[2], w2); v[3] = cmul(v[3], w3); v[4] = cmul(v[4], w4);
    v[5] = cmul(v[5], w5); v[6] = cmul(v[6], w6); v[7] = cmul(v[7], w7); v[8] = cmul(v[8], w8);
    v[9] = cmul(v[9], cmul(w1, w8)); v[10] = cmul(v[10], cmul(w2, w8)); v[11] = cmul(v[11], cmul(w3, w8));
    v[12] = cmul(v[12], cmul(w4, w8)); v[13] = cmul(v[13], cmul(w5, w8)); v[14] = cmul(v[14], cmul(w6, w8));
    v[15] = cmul(v[15], cmul(w7, w8));
}

// CL (config 4, clusters of 3 CTAs): the three inner columns m = 3 kt + i fill output row kt,
// column i the positions mt = i (mod 3) (checked at plan time, k_cl_check).  Each CTA stages
// E(k, m) X(kc) at slot mt / 3 of its shared memory; after a cluster barrier CTA i copies row
// positions [4096 i, 4096 i + 4096) out of the three CTAs' shared memory (distributed shared
// memory) with contiguous 16-byte stores -- instead of each column's 16-byte stores at a
// 48-byte stride.
template <typename T, int MINB, bool CL = false>
__global__ void __launch_bounds__(256, MINB) out_f4096_kernel(OutArgs A) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    using C = cx<T>;
    pdl_trigger();
    pdl_wait();
    C* S = (C*)smem_raw;
    const int tid = threadIdx.x;
    const int m = blockIdx.x;              // inner column
    const int64_t w = blockIdx.y;
    const int qi = (int)A.q, di = (int)A.d;
    const C* __restrict__ src = (const C*)A.C + w * A.iM * A.iN +
                                (A.cnj ? (int64_t)m * A.iM : (int64_t)((m % qi) * di + m / qi));
    const C* __restrict__ tw = (const C*)A.tw;
    const int ld = A.cnj ? 1 : qi * di;    // stride of C over j
    C v[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = src[(tid + 256 * r) * ld];
    dft16<T>(v);
    twiddle15(v, tw, tid);
#pragma unroll
    for (int k = 0; k < 16; ++k) S[k * 256 + tid] = v[k];
    __syncthreads();
    const int hi = tid >> 4, lo = tid & 15;   // pass 2: (k1, t1); pass 3: (k1, k2)
#pragma unroll
    for (int t2 = 0; t2 < 16; ++t2) v[t2] = S[hi * 256 + lo + 16 * t2];
    __syncthreads();
    dft16<T>(v);
    twiddle15(v, tw, 16 * lo);
#pragma unroll
    for (int k = 0; k < 16; ++k) S[hi * 272 + 17 * k + lo] = v[k];
    __syncthreads();
#pragma unroll
    for (int t1 = 0; t1 < 16; ++t1) v[t1] = S[hi * 272 + 17 * lo + t1];
    dft16<T>(v);
    C* out = (C*)A.out + w * A.M * A.N;
    if constexpr (CL) {
        namespace cg = cooperative_groups;
        cg::cluster_group cl = cg::this_cluster();
        const int kt = m / 3;
        const size_t rowb = (size_t)kt * (size_t)A.N;
        __syncthreads();   // every pass-3 read of S is done
        fb_column_dest<16, C>(A, (unsigned long long)m, (unsigned int)(hi + 16 * lo),
                              [&](int i, size_t dst, C ph) { S[(dst - rowb) / 3] = cmul(ph, v[i]); });
        cl.sync();
        const int r = (int)cl.block_rank();
        C y[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const int mt = 4096 * r + tid + 256 * j;
            const C* rs = cl.map_shared_rank(S, mt % 3);
            y[j] = rs[mt / 3];
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) out[rowb + 4096 * r + tid + 256 * j] = y[j];
        cl.sync();   // no CTA leaves while another reads its shared memory
    } else {
        fb_column<16>(A, out, (unsigned long long)m, (unsigned int)(hi + 16 * lo), 16, [&](int i) { return v[i]; });
    }
}
constexpr size_t kOutF4096Elems = 16 * 272;

// Plan time: does config 4's cluster variant apply -- for every inner column m and channel
// kc, the destination row is m / 3 and the position is m (mod 3), within 3 x 4096?
template <typename T>
__global__ void k_cl_check(OutArgs A, int* bad) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= A.iN * A.iM) return;
    const int m = (int)(i / A.iM), kc = (int)(i % A.iM);
    const FbCol cc = fb_col(A, (unsigned long long)m);
    const FbIter<cx<T>> it = fb_iter<cx<T>>(A, cc, kc ? (unsigned long long)A.Nr - kc : 0ull);
    size_t dst;
    cx<T> ph;
    fb_dest(A, it, &dst, &ph);
    const size_t row = dst / (size_t)A.N, mt = dst % (size_t)A.N;
    if (row != (size_t)(m / 3) || mt % 3 != (size_t)(m % 3) || mt >= 3 * 4096) atomicExch(bad, 1);
}

#include "tiny.cuh"

// ---------------------------------------------------------------------------------
// synthesis (the inverse DGT with the plan's window as the synthesis window gamma; SURVEY
// NEXT-1): f = sum_{m,n} c(m,n) M_{b(m+w(n))} T_{an} gamma, the inversion formula of
// PAPER.md:171-175 (pass the canonical dual S^{-1} g to invert).  It is the adjoint of the
// forward pipeline, so the kernels run the forward steps backwards with every linear map
// replaced by its adjoint: permutations by their inverses, multipliers by their conjugates,
// the forward DFTs by unnormalised inverse DFTs, computed as conj(DFT(conj(.))) on the same
// Stockham engine (the conjugations are folded into the loads and stores).
// ---------------------------------------------------------------------------------

// Adjoint of out_kernel: c[w][M][N] -> C[w][j][kappa][n'].  Same CTA tiling as out_kernel.
//   T-branch: X'(m', n) = conj(E(n)) c[(m' - rot(n)) mod M][n];  F-branch: X'(kc, m) =
//   conj(E(k,m)) c[kt][mt] (the Alg. 1 remap read backwards);  then C'(j, n) = sum_m' X'(m', n)
//   exp(+2 pi i j m' / iM).
template <typename T, int IMCT = 0>   // IMCT = 200: the compile-time DFT over m (config 2)
__global__ void __launch_bounds__(256) out_adj_kernel(OutArgs A) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    using C = cx<T>;
    pdl_trigger();
    pdl_wait();
    const int64_t iM = A.iM, iN = A.iN, q = A.q, d = A.d;
    const int NT = A.NT;
    const int iMi = (int)iM, qi = (int)q, di = (int)d;
    int64_t nb, ns;
    int nt;
    if (A.grouped) {
        const int kap = (int)(blockIdx.x % q), blk = (int)(blockIdx.x / q);
        nb = kap + q * (int64_t)blk * NT;
        ns = q;
        nt = (int)((d - (int64_t)blk * NT) < NT ? (d - (int64_t)blk * NT) : NT);
    } else {
        nb = (int64_t)blockIdx.x * NT;
        ns = 1;
        nt = (int)((iN - nb) < NT ? (iN - nb) : NT);
    }
    const int64_t w = blockIdx.y;
    unsigned char* sbase = A.gscr ? A.gscr + ((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * A.gstride : smem_raw;
    C* bufA = (C*)sbase;
    C* bufB = bufA + (size_t)NT * iM;
    const C* cin = (const C*)A.out + w * A.M * A.N;   // the coefficients (input here)
    // bufA = conj(X'), the input of the forward engine
    if (A.branch != DGT_BRANCH_FREQ) {
        const C* E = (const C*)A.E;
        const int Mi = (int)A.M, Ni = (int)A.N;
        for (int i = threadIdx.x; i < nt * iMi; i += blockDim.x) {
            const int cl = i % nt, mo = i / nt;
            const int n = (int)nb + cl;
            int m = mo + A.rot[n];
            if (m >= Mi) m -= Mi;
            // c[mo][n] = E(n) X(m, n)  =>  conj(X'(m, n)) = E(n) conj(c[mo][n])
            const C v = cin[(size_t)mo * Ni + n];
            bufA[cl * iMi + m] = cmul(E[n], mk<T>(v.x, -v.y));
        }
    } else {
        const unsigned int Nn = (unsigned int)A.N;
        for (int cl = 0; cl < nt; ++cl) {
            const FbCol cc = fb_col(A, (unsigned long long)(nb + ns * cl));
            const unsigned int kc0 = threadIdx.x;   // blockDim.x == 256
            const int cnt = (iMi - (int)kc0 + 255) / 256;
            if (cnt <= 0) continue;
            FbIter<C> it = fb_iter<C>(A, cc, kc0 ? (unsigned long long)A.Nr - kc0 : 0ull);
            for (int i = 0; i < cnt; ++i) {
                if (i == 1 && kc0 == 0) it = fb_iter<C>(A, cc, (unsigned long long)A.Nr - 256u);
                else if (i > 0) fb_step(A, it);
                const unsigned int twoN = 2 * Nn;
                C ph;
                if (A.C3) {
                    const unsigned int s2 = bmod((unsigned long long)it.sq * it.sq, twoN, A.inv2N);
                    const unsigned int t1 = bmod((unsigned long long)A.C3 * s2, twoN, A.inv2N);
                    ph = __ldg((const C*)A.ptab + submod(t1, it.t2, twoN));
                } else {
                    ph = it.ph;
                }
                const unsigned int mt = it.sq >= Nn ? it.sq - Nn : it.sq;
                const unsigned int bu = (unsigned int)A.b;
                unsigned int kt = __umulhi(it.xx, A.invb);
                unsigned int r = it.xx - kt * bu;
                if (r >= bu) { r -= bu; ++kt; }
                if (r >= bu) ++kt;
                const C v = cin[(size_t)kt * Nn + mt];
                bufA[cl * iMi + kc0 + 256 * i] = cmul(ph, mk<T>(v.x, -v.y));
            }
        }
    }
    __syncthreads();
    C* X;
    if constexpr (IMCT > 0) X = fft_ct<T, IMCT>(bufA, bufB, nt, (const C*)A.tw);
    else X = fft_smem<T>(bufA, bufB, A.rd, nt, iMi, (const C*)A.tw);
    // C'(j, n) = conj(X(j)), stored at [j][n mod q][n div q]
    C* Cw = (C*)A.C + w * iM * iN;
    if (IMCT > 0 && (nt == 16 || nt == 20) && qi == 4 && ns == 1 && (nb & 3) == 0) {
        // config 2: element i = (j, kappa, n'') with n'' fastest -- nt/4 lanes store contiguous
        // bytes of row (j, kappa) (the generic loop's lanes each hit another row)
        const int nq0 = (int)nb >> 2, NQ = nt >> 2;
        for (int i = threadIdx.x; i < nt * iMi; i += blockDim.x) {
            const int t = i / NQ, nn = i - t * NQ, kap = t & 3, j = t >> 2;
            const C v = X[(4 * nn + kap) * iMi + j];
            Cw[(j * 4 + kap) * di + nq0 + nn] = mk<T>(v.x, -v.y);
        }
        return;
    }
    for (int i = threadIdx.x; i < nt * iMi; i += blockDim.x) {
        const int cl = i % nt, j = i / nt;
        const int n = (int)(nb + ns * cl);
        const int nq = n / qi;
        const C v = X[cl * iMi + j];
        Cw[(j * qi + (n - nq * qi)) * di + nq] = mk<T>(v.x, -v.y);
    }
}

// Adjoints of the config-4 kernels (same CTA shapes and passes, run backwards).
// F-branch remap gather for column m: put(i, E(k,m) conj(c[kt][mt])) for kc = kc0 + 256 i
// (the conjugated X' = conj(E) c of the adjoint remap), residues advanced as in fb_column.
template <int CNT, typename C, class Put>
__device__ __forceinline__ void fb_gather(const OutArgs& A, const C* cin, unsigned long long m, unsigned int kc0,
                                          Put&& put) {
    const FbCol cc = fb_col(A, m);
    const unsigned int Nn = (unsigned int)A.N, twoN = 2 * Nn, bu = (unsigned int)A.b;
    FbIter<C> it = fb_iter<C>(A, cc, kc0 ? (unsigned long long)A.Nr - kc0 : 0ull);
#pragma unroll
    for (int i = 0; i < CNT; ++i) {
        if (i == 1 && kc0 == 0) it = fb_iter<C>(A, cc, (unsigned long long)A.Nr - 256u);
        else if (i > 0) fb_step(A, it);
        C ph;
        if (A.C3) {
            const unsigned int s2 = bmod((unsigned long long)it.sq * it.sq, twoN, A.inv2N);
            const unsigned int t1 = bmod((unsigned long long)A.C3 * s2, twoN, A.inv2N);
            ph = __ldg((const C*)A.ptab + submod(t1, it.t2, twoN));
        } else {
            ph = it.ph;
        }
        const unsigned int mt = it.sq >= Nn ? it.sq - Nn : it.sq;
        unsigned int kt = __umulhi(it.xx, A.invb);
        unsigned int r = it.xx - kt * bu;
        if (r >= bu) { r -= bu; ++kt; }
        if (r >= bu) ++kt;
        const C v = cin[(size_t)kt * Nn + mt];
        put(i, cmul(ph, mk<decltype(v.x)>(v.x, -v.y)));
    }
}

// Adjoint of out_f4096_kernel: c -> C[w][j][kappa][n'] for N_r = iM = 4096.  Thread t gathers
// conj(X'(t + 256 r)) (the pass-1 input layout), the three radix-16 passes run as in the
// forward kernel, and pass 3's outputs X(j) give C'(j) = conj(X(j)).
template <typename T, int MINB>
__global__ void __launch_bounds__(256, MINB) out_f4096_adj_kernel(OutArgs A) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    using C = cx<T>;
    pdl_trigger();
    pdl_wait();
    C* S = (C*)smem_raw;
    const int tid = threadIdx.x;
    const int m = blockIdx.x;
    const int64_t w = blockIdx.y;
    const int qi = (int)A.q, di = (int)A.d;
    const C* __restrict__ tw = (const C*)A.tw;
    const C* cin = (const C*)A.out + w * A.M * A.N;
    C v[16];
    fb_gather<16>(A, cin, (unsigned long long)m, (unsigned int)tid, [&](int i, C x) { v[i] = x; });
    dft16<T>(v);
    twiddle15(v, tw, tid);
#pragma unroll
    for (int k = 0; k < 16; ++k) S[k * 256 + tid] = v[k];
    __syncthreads();
    const int hi = tid >> 4, lo = tid & 15;
#pragma unroll
    for (int t2 = 0; t2 < 16; ++t2) v[t2] = S[hi * 256 + lo + 16 * t2];
    __syncthreads();
    dft16<T>(v);
    twiddle15(v, tw, 16 * lo);
#pragma unroll
    for (int k = 0; k < 16; ++k) S[hi * 272 + 17 * k + lo] = v[k];
    __syncthreads();
#pragma unroll
    for (int t1 = 0; t1 < 16; ++t1) v[t1] = S[hi * 272 + 17 * lo + t1];
    dft16<T>(v);
    C* dst = (C*)A.C + w * A.iM * A.iN + (A.cnj ? (int64_t)m * A.iM : (int64_t)((m % qi) * di + m / qi));
    const int ld = A.cnj ? 1 : qi * di;
#pragma unroll
    for (int k3 = 0; k3 < 16; ++k3) dst[(hi + 16 * lo + 256 * k3) * ld] = mk<T>(v[k3].x, -v[k3].y);
}

// Adjoint of zak_ct_kernel (d = D, q = Q, RBC columns): gather conj(T'_u(tau)) for all u
// through the inverse scatter map, one DFT_D of Q RBC sequences, conj(Phi')(nu) =
// sum_u Y_u(nu) G_u(nu), one DFT_D of the RBC columns, f(x) = conj(chirp(x) R(s)).
template <typename T, int D, int Q, int RBC, int NT = 256>
__global__ void __launch_bounds__(NT, 512 / NT) zak_ct_adj_kernel(ZakArgs A, void* fout) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    using C = cx<T>;
    pdl_trigger();
    pdl_wait();
    constexpr int NG = (RBC * D + NT - 1) / NT, NP = (Q * RBC * D + NT - 1) / NT;
    const int c = (int)A.c;
    const int nrb = c / RBC;
    const int rblk = blockIdx.x % nrb, l = blockIdx.x / nrb;
    const int64_t w = blockIdx.y;
    const int r0 = rblk * RBC;
    C* R1 = (C*)smem_raw;
    C* R2 = R1 + Q * RBC * D;
    const C* __restrict__ tw = (const C*)A.tw;
    const int tid = threadIdx.x;
    {
        const C* Cw = (const C*)A.C + w * A.iM * Q * D;
        const int jbase = r0 + c * (l % Q);
        const bool cnj = A.cnj != 0;   // [n][j] layout: rr fastest (see zak_ct_kernel)
        const int iM = (int)A.iM;
        C v[NP];
#pragma unroll
        for (int it = 0; it < NP; ++it) {
            const int i = tid + it * NT;
            if (i < Q * RBC * D) {
                const int g = zrow<D, RBC, sizeof(C)>(i / RBC, i % RBC, Q * D);
                const int u = cnj ? g / D : i / (RBC * D), rem = i % (RBC * D);
                const int rr = cnj ? i % RBC : rem / D, np = cnj ? g % D : rem % D;
                const int kappa = (l - u + Q) % Q;
                v[it] = cnj ? Cw[(int64_t)(kappa + Q * np) * iM + jbase + rr]
                            : Cw[((jbase + rr) * Q + kappa) * D + np];
            }
        }
#pragma unroll
        for (int it = 0; it < NP; ++it) {
            const int i = tid + it * NT;
            if (i < Q * RBC * D) {
                const int g = zrow<D, RBC, sizeof(C)>(i / RBC, i % RBC, Q * D);
                const int u = cnj ? g / D : i / (RBC * D), rem = i % (RBC * D);
                const int rr = cnj ? i % RBC : rem / D, np = cnj ? g % D : rem % D;
                int tau = D - np - (l < u ? 1 : 0);
                if (tau >= D) tau -= D;
                R1[(u * RBC + rr) * D + tau] = mk<T>(v[it].x, -v[it].y);
            }
        }
    }
    __syncthreads();
    C* Y = fft_ct<T, D>(R1, R2, Q * RBC, tw);   // in R1 or R2
    C* Acc = Y == R1 ? R2 : R1;
    {
        const C* __restrict__ G = (const C*)A.G;
#pragma unroll
        for (int it = 0; it < NG; ++it) {
            const int i = tid + it * NT;
            if (i < RBC * D) {
                const int rr = i / D, nu = i % D;
                C acc = cmul(Y[rr * D + nu], __ldg(G + ((r0 + rr) * Q) * D + nu));
#pragma unroll
                for (int u = 1; u < Q; ++u)
                    acc = acc + cmul(Y[(u * RBC + rr) * D + nu], __ldg(G + ((r0 + rr) * Q + u) * D + nu));
                Acc[i] = acc;
            }
        }
    }
    __syncthreads();
    C* R = fft_ct<T, D>(Acc, Y, RBC, tw);   // Y is dead: its buffer is the scratch
    const C* __restrict__ chirp = (const C*)A.chirp;
    C* fo = (C*)fout + w * A.L;
#pragma unroll
    for (int it = 0; it < NG; ++it) {
        const int i = tid + it * NT;
        if (i < RBC * D) {
            const int rr = i % RBC, s = zrow<D, RBC, sizeof(C)>(i / RBC, rr, D);   // rr fastest (RBC consecutive residues per row s)
            const int x = r0 + rr + c * (l + Q * s);
            C v = R[rr * D + s];
            if (chirp) v = cmul(v, __ldg(chirp + x));
            fo[x] = mk<T>(v.x, -v.y);
        }
    }
}

// Adjoint of zak_kernel: C[w][j][kappa][n'] -> f~[w][x].  Same CTA tiling (signal, residue
// block, l).  Per u: gather T'(tau) (the scatter read backwards), adjoint DFT_d over tau,
// accumulate Phi'(k; nu) += Y'_u(nu) conj(G(k, u; nu)); then the adjoint DFT_d over nu and the
// write through the (bijective, gcd(p, q) = 1) Zak index map with conj(chirp).  Buffers: the
// conjugated accumulator acc (RB p d), scratch B (RB p d >= RB d), Y (RB d).
template <typename T>
__global__ void __launch_bounds__(256) zak_adj_kernel(ZakArgs A, void* fout) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    using C = cx<T>;
    pdl_trigger();
    pdl_wait();
    const int64_t d = A.d, p = A.p, q = A.q, c = A.c, L = A.L;
    const int RB = A.RB;
    const int nrb = (int)((c + RB - 1) / RB);
    const int rblk = blockIdx.x % nrb;
    const int l = blockIdx.x / nrb;
    const int64_t w = blockIdx.y;
    const int64_t r0 = (int64_t)rblk * RB;
    const int nr = (int)((c - r0) < RB ? (c - r0) : RB);
    unsigned char* sbase = A.gscr ? A.gscr + ((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * A.gstride : smem_raw;
    C* acc = (C*)sbase;                     // RB*p*d: conj(Phi')
    C* bufB = acc + (size_t)RB * p * d;     // RB*p*d
    C* bufY = bufB + (size_t)RB * p * d;    // RB*d
    const C* __restrict__ tw = (const C*)A.tw;
    const C* __restrict__ G = (const C*)A.G;
    const int di = (int)d, pi = (int)p, qi = (int)q, ci = (int)c, Lci = (int)(L / c);
    const C* Cw = (const C*)A.C + w * A.iM * q * d;
    const int jbase = (int)(r0 + c * ((l * p) % q));
    for (int u = 0; u < qi; ++u) {
        const int kappa = ((l - u) % qi + qi) % qi;
        const int off = (l < u) ? 1 : 0;
        // gather conj(T'(tau)), tau = (-n' - off) mod d
        for (int i = threadIdx.x; i < nr * di; i += blockDim.x) {
            const int rr = i / di, np = i - rr * di;
            int tau = di - np - off;
            if (tau >= di) tau -= di;
            if (tau < 0) tau += di;
            const C v = Cw[((jbase + rr) * qi + kappa) * di + np];
            bufB[rr * di + tau] = mk<T>(v.x, -v.y);
        }
        __syncthreads();
        const C* Y = fft_smem<T>(bufB, bufY, A.rd, nr, di, tw);   // Y = conj(Y'_u)
        // conj(Phi'(k; nu)) += Y(nu) G(k, u; nu)
        for (int i = threadIdx.x; i < nr * pi * di; i += blockDim.x) {
            const int rr = i / (pi * di), rem = i - rr * pi * di;
            const int k = rem / di, nu = rem - k * di;
            const C t = cmul(Y[rr * di + nu], G[(((r0 + rr) * q + u) * p + k) * d + nu]);
            acc[i] = u ? acc[i] + t : t;
        }
        __syncthreads();
    }
    // f~'(s) = conj(DFT(conj(Phi')))(s) = conj(R(s))
    const C* R = fft_smem<T>(acc, bufB, A.rd, nr * pi, di, tw);
    const C* __restrict__ chirp = (const C*)A.chirp;
    C* fo = (C*)fout + w * L;
    const int base_kq = pi * l;
    for (int i = threadIdx.x; i < nr * pi * di; i += blockDim.x) {
        const int rr = i % nr;
        const int ks = i / nr;   // k*d + s (rr fastest: consecutive residues, coalesced)
        const int s = ks % di, k = ks / di;
        int z = k * qi + base_kq + s * pi * qi;
        z %= Lci;
        const int x = (int)r0 + rr + ci * z;
        C v = R[(rr * pi + k) * di + s];
        if (chirp) v = cmul(v, chirp[x]);
        fo[x] = mk<T>(v.x, -v.y);   // conj(chirp(x)) f~'(x) = conj(chirp(x) R)
    }
}

// out = conj(pre) * in, elementwise over n elements (pre is L-periodic)
template <typename T>
__global__ void k_conj_chirp(cx<T>* out, const cx<T>* in, const cx<T>* __restrict__ pre, int64_t L, int64_t total) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const cx<T> p = pre[i % L];
        out[i] = cmulc(in[i], p);
    }
}

// ---------------------------------------------------------------------------------
// canonical dual / tight window (Alg. 2 of PAPER.md:951-994 with the separable
// dual by factorisation).  All in fp64, plan time.
//
// The plan's inner separable lattice transforms the window to g~ (T: P_{s1} g) or g^ (F:
// P_{-s0} FFT(P_{s1} g) / L) with factorisation Gamma_r(k, u; nu) = sum_s g~(x(r,k,u,s))
// W_d^{s nu} (p x q per (r, nu)).  With Z the factorisation map (Z* Z = d) the separable frame
// operator is S = M' Z* (H (x) I) Z / d,  H = Gamma Gamma^H (p x p), so
//   dual:  Z gamma~ = H^{-1} Gamma / M',      tight: Z g~_t = H^{-1/2} Gamma / sqrt(M')
// (M' = iM, the inner channel count).  Then gamma~ = Z^{-1}(.) and the shear is undone:
//   T: gamma = conj(P_{s1}) gamma~;   F: gamma = conj(P_{s1}) IFFT_unnorm(conj(P_{-s0}) gamma~) / L
// (S_nonsep = V* S~ V with V = P_{-s0} F P_{s1}, V* V = L; the tight window takes 1/sqrt(L)
// instead of 1/L).
// ---------------------------------------------------------------------------------
constexpr int kDualPMax = 8, kDualQMax = 64;

// one thread per (r, nu); G64[((r q + u) p + k) d + nu] = conj(Gamma)/d  ->  Gd (same layout,
// the factorisation Gamma^d of the result, NOT conjugated)
__global__ void k_dual_factor(double2* Gd, const double2* G64, int64_t c, int64_t d, int p, int q, double scale,
                              int tight, int* status) {
    for (int64_t rv = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; rv < c * d; rv += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = rv / d, nu = rv % d;
        double2 Gm[kDualPMax][kDualQMax];
        for (int k = 0; k < p; ++k)
            for (int u = 0; u < q; ++u) {
                const double2 v = G64[((r * q + u) * p + k) * d + nu];
                Gm[k][u] = make_double2(v.x * (double)d, -v.y * (double)d);   // Gamma
            }
        double2 H[kDualPMax][kDualPMax];
        for (int k = 0; k < p; ++k)
            for (int k2 = 0; k2 < p; ++k2) {
                double sr = 0.0, si = 0.0;
                for (int u = 0; u < q; ++u) {   // Gamma[k][u] conj(Gamma[k2][u])
                    sr += Gm[k][u].x * Gm[k2][u].x + Gm[k][u].y * Gm[k2][u].y;
                    si += Gm[k][u].y * Gm[k2][u].x - Gm[k][u].x * Gm[k2][u].y;
                }
                H[k][k2] = make_double2(sr, si);
            }
        double2 X[kDualPMax][kDualPMax];   // the p x p left factor: H^{-1} or H^{-1/2}
        if (!tight) {
            // Gauss-Jordan on [H | I] with partial pivoting
            for (int k = 0; k < p; ++k)
                for (int k2 = 0; k2 < p; ++k2) X[k][k2] = make_double2(k == k2 ? 1.0 : 0.0, 0.0);
            for (int col = 0; col < p; ++col) {
                int piv = col;
                double best = 0.0;
                for (int k = col; k < p; ++k) {
                    const double m2 = H[k][col].x * H[k][col].x + H[k][col].y * H[k][col].y;
                    if (m2 > best) { best = m2; piv = k; }
                }
                if (best == 0.0) { atomicExch(status, 1); break; }
                for (int k2 = 0; k2 < p; ++k2) {
                    double2 t = H[col][k2]; H[col][k2] = H[piv][k2]; H[piv][k2] = t;
                    t = X[col][k2]; X[col][k2] = X[piv][k2]; X[piv][k2] = t;
                }
                const double2 hv = H[col][col];
                const double den = hv.x * hv.x + hv.y * hv.y;
                const double2 inv = make_double2(hv.x / den, -hv.y / den);
                for (int k2 = 0; k2 < p; ++k2) { H[col][k2] = cmul(H[col][k2], inv); X[col][k2] = cmul(X[col][k2], inv); }
                for (int k = 0; k < p; ++k) {
                    if (k == col) continue;
                    const double2 fct = H[k][col];
                    for (int k2 = 0; k2 < p; ++k2) {
                        H[k][k2] = H[k][k2] - cmul(fct, H[col][k2]);
                        X[k][k2] = X[k][k2] - cmul(fct, X[col][k2]);
                    }
                }
            }
        } else if (p == 1) {
            X[0][0] = make_double2(1.0 / sqrt(H[0][0].x), 0.0);
        } else {
            // p = 2: sqrt(H) = (H + sqrt(det) I) / sqrt(tr + 2 sqrt(det)), then its inverse
            const double det = H[0][0].x * H[1][1].x - (H[0][1].x * H[0][1].x + H[0][1].y * H[0][1].y);
            const double sd = sqrt(det), tnorm = sqrt(H[0][0].x + H[1][1].x + 2.0 * sd);
            const double a00 = (H[0][0].x + sd) / tnorm, a11 = (H[1][1].x + sd) / tnorm;
            const double2 a01 = make_double2(H[0][1].x / tnorm, H[0][1].y / tnorm);
            const double dr = a00 * a11 - (a01.x * a01.x + a01.y * a01.y);   // det(sqrt H) > 0
            X[0][0] = make_double2(a11 / dr, 0.0);
            X[1][1] = make_double2(a00 / dr, 0.0);
            X[0][1] = make_double2(-a01.x / dr, -a01.y / dr);
            X[1][0] = make_double2(-a01.x / dr, a01.y / dr);   // conj(a01)
        }
        for (int k = 0; k < p; ++k)
            for (int u = 0; u < q; ++u) {
                double sr = 0.0, si = 0.0;
                for (int k2 = 0; k2 < p; ++k2) {
                    const double2 t = cmul(X[k][k2], Gm[k2][u]);
                    sr += t.x;
                    si += t.y;
                }
                Gd[((r * q + u) * p + k) * d + nu] = make_double2(sr * scale, si * scale);
            }
    }
}

// gamma~(x(r,k,u,s)) = (1/d) sum_nu Gd_r(k,u;nu) W_d^{-s nu}, then the T-branch un-shear
// conj(P_sigma(x)) (sigma = s1; 0 = none) or, F-branch, conj(P_{-s0}(x)) before the IFFT.
__global__ void k_dual_unfactor(double2* out, const double2* Gd, int64_t L, int64_t c, int64_t d, int64_t p,
                                int64_t q, int64_t sigma) {
    const int64_t Lc = L / c;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < L; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = i % d;
        const int64_t k = (i / d) % p;
        const int64_t u = (i / (d * p)) % q;
        const int64_t r = i / (d * p * q);
        const double2* src = Gd + ((r * q + u) * p + k) * d;
        double sr = 0.0, si = 0.0;
        int64_t e = 0;   // s nu mod d
        for (int64_t nu = 0; nu < d; ++nu) {
            double sn, cs;
            sincospi(2.0 * (double)e / (double)d, &sn, &cs);
            const double2 v = src[nu];
            sr += v.x * cs - v.y * sn;
            si += v.x * sn + v.y * cs;
            e += s;
            if (e >= d) e -= d;
        }
        const int64_t x = r + c * ((k * q + p * u + s * p * q) % Lc);
        double2 v = make_double2(sr / (double)d, si / (double)d);
        if (sigma) v = cmulc(v, chirp_val(sigma, x, L));
        out[x] = v;
    }
}

// F-branch tail: out = conj(P_{s1}(x)) in(x) / L (s1 = 0: the chirp is 1), cast to T
template <typename T>
__global__ void k_dual_finish(cx<T>* out, const double2* in, int64_t L, int64_t sigma, double scale) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < L; x += (int64_t)gridDim.x * blockDim.x) {
        double2 v = in[x];
        if (sigma) v = cmulc(v, chirp_val(sigma, x, L));
        out[x] = mk<T>((T)(v.x * scale), (T)(v.y * scale));
    }
}

// ---------------------------------------------------------------------------------
// shear-OLA (PAPER.md:815-831 overlap-add, 921-949 shear-OLA): the DGT with an
// FIR window (support Lg) of a long signal as DGTs of blocks.  Block b holds f[b Lb, (b+1) Lb)
// zero-extended to Lx >= Lb + Lg + 2a (a legal length); its length-Lx DGT with the window
// zero-extended to Lx has, at local position p (n_local = p mod Nx), exactly the part of
// c(m, b Lb/a + p) that comes from the block's samples -- no wrap-around reaches them, and the
// phases agree because L_min | Lb -- so summing the blocks' coefficients over b gives c.
// ---------------------------------------------------------------------------------
template <typename Tin>
__global__ void k_ola_split(Tin* x, const Tin* f, int64_t L, int64_t Lb, int64_t Lx, int64_t Nb, int64_t total) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t l = i % Lx, wb = i / Lx;
        const int64_t w = wb / Nb, b = wb % Nb;
        Tin v{};
        if (l < Lb) v = f[w * L + b * Lb + l];
        x[i] = v;
    }
}

// c[w][m][n] = sum over blocks b with p = n - b nb (cyclic mod N) in [pmin, pmax] of
// cb[w Nb + b][m][p mod Nx]
template <typename T>
__global__ void k_ola_add(cx<T>* c, const cx<T>* cb, int64_t M, int64_t N, int64_t Nx, int64_t nb, int64_t Nb,
                          int64_t pmin, int64_t pmax, int64_t total) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t n = i % N, m = (i / N) % M, w = i / (N * M);
        cx<T> acc = mk<T>(T(0), T(0));
        // blocks whose window range covers n: b from floor((n - pmin) / nb) downwards
        const int64_t bhi = (n - pmin) >= 0 ? (n - pmin) / nb : -((pmin - n + nb - 1) / nb);
        const int64_t span = (pmax - pmin) / nb + 2;
        for (int64_t db = 0; db < span && db < Nb; ++db) {
            const int64_t b = (((bhi - db) % Nb) + Nb) % Nb;
            int64_t p = ((n - b * nb) % N + N) % N;   // in [0, N)
            if (p > pmax) p -= N;                      // the block's negative positions
            if (p < pmin || p > pmax) continue;
            const int64_t nl = ((p % Nx) + Nx) % Nx;
            acc = acc + cb[((w * Nb + b) * M + m) * Nx + nl];
        }
        c[i] = acc;
    }
}

// Multiwindow DGT, Eq. (mw_phases) of PAPER.md:397-403: with n = nt lambda2 + m (m < lambda2;
// reading Z12: m = n mod lambda2), at = lambda2 a and sigma_m = m s mod b,
//   c[w][k][n] = exp(-2 pi i nt at sigma_m / L) d_m[w][k][nt],
// d_m the separable DGT of f with g_m = M_{sigma_m} T_{m a} g on (at, b).  The phase index
// (nt at mod L) sigma_m mod L is exact in int64 (nt at < L, sigma_m < b <= L < 2^31).
template <typename T>
__global__ void k_mw_interleave(cx<T>* c, const cx<T>* d, const int64_t* sig, int64_t Wc, int64_t M, int64_t N,
                                int64_t l2, int64_t at, int64_t L, int64_t total) {
    const int64_t Nt = N / l2;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t n = i % N, wk = i / N;
        const int64_t m = n % l2, nt = n / l2;
        const int64_t r = (((nt * at) % L) * sig[m]) % L;
        double sn, cs;
        sincospi(-2.0 * (double)r / (double)L, &sn, &cs);
        const cx<T> v = d[(m * Wc * M + wk) * Nt + nt];
        const T pr = (T)cs, pi = (T)sn;
        c[i] = mk<T>(v.x * pr - v.y * pi, v.x * pi + v.y * pr);
    }
}

// ---------------------------------------------------------------------------------
// the plan
// ---------------------------------------------------------------------------------

struct Plan;
static void free_plan(Plan* P);
static constexpr int64_t kMaxChunk = 8192;   // signals per launch pair of the generic path
struct Plan {
    dgt_lattice_info info{};
    int dtype = DGT_C64;
    int flags = 0;
    int device = 0;
    size_t esz = 8;  // complex element size
    // device tables
    void* G = nullptr;       // window factors (L complex)
    double2* gt64 = nullptr; // the Alg. 1 window transform g~ / g^ in fp64 (dual/tight windows)
    void* chirp = nullptr;   // kernel-A load multiplier (L complex) or null
    void* pre = nullptr;     // F-branch pre-FFT chirp (L complex) or null
    void* tw_d = nullptr;    // twiddles length d
    void* tw_m = nullptr;    // twiddles length iM
    void* E = nullptr;       // T-branch column phases (N)
    int* rot = nullptr;      // T-branch rotations (N)
    void* ptab = nullptr;    // F-branch phase table (2N)
    // workspace
    void* Cws = nullptr;     // chunk intermediate
    void* fhat = nullptr;    // F-branch chunk spectra
    int64_t chunk = 1;
    int64_t fb = 1;          // F-branch front batch (signals per cuFFT call)
    int64_t ib = 1;          // F-branch synthesis batch
    size_t ws_bytes = 0;
    std::map<int64_t, cufftHandle> fft_plans;
    // kernel configuration
    Radices rd_d{}, rd_m{};
    int RB = 1, NT = 1;
    size_t smemA = 0, smemB = 0;
    int allu = 0;            // zak_kernel all-u mode (p = 1)
    // shear-OLA (dgt_plan_fir): blocks of Lb samples zero-extended to Lx run
    // through the inner plan; their coefficients are overlap-added
    struct Plan* ola = nullptr;
    int64_t ola_Lb = 0, ola_Nb = 0, ola_Ws = 0, ola_pmin = 0, ola_pmax = 0;
    // multiwindow plan (dgt_plan_multiwindow): lambda2 separable
    // plans on (lambda2 a, M) with the windows g_m, a [lambda2][Wc][M][N / lambda2] buffer of
    // their coefficients and the residues sigma_m = m s mod b (device)
    std::vector<struct Plan*> mw;
    int64_t mw_Wc = 0;
    void* mw_d = nullptr;
    int64_t* mw_sig = nullptr;
    void* ola_x = nullptr;   // [Ws Nb][Lx] blocks (input type)
    void* ola_c = nullptr;   // [Ws Nb][M][Nx] block coefficients
    int gA = 0, gB = 0;      // Zak / output kernels with per-CTA buffers in global scratch
    unsigned char* scrA = nullptr;
    unsigned char* scrB = nullptr;
    // synthesis (dgt_execute_inverse): chunk, zak_adj_kernel smem, workspace (made at plan
    // time by alloc_workspace: C intermediate + F-branch spectra, shared with the forward's)
    int64_t inv_chunk = 1;
    size_t smemAinv = 0;
    void* Cinv = nullptr;
    void* finv = nullptr;
    int inv_alias = 0;       // bit 0: Cinv is Cws, bit 1: finv is fhat (not freed twice)
    int zct = 0;             // zak_kernel compile-time inner length (0 = runtime radices)
    int inv_generic = 0;     // experiment knob (NSDGT_INV_GENERIC, read at plan time): generic synthesis
    int outct = 0;           // out_kernel compile-time inner channel count (0 = runtime radices)
    int zrr = 0;             // forward Zak with zak_rr_kernel (d = 180 = 12 x 15 in registers)
    int front = 0;           // F-branch front end by front_f4096_kernel + zak_rr0_kernel (L = 180 x 4096)
    int outcl = 0;           // config 4: out_f4096 in clusters of 3 CTAs staging whole rows (k_cl_check)
    void* chR = nullptr;     // zak_ct: the chirp's d-entry factor R(s) = P(c q s) (ZakArgs::chR)
    int sigD = 0;
    int tiny = 0;            // whole transform of a signal in one CTA (tiny.cuh)
    unsigned int* tiny_dst = nullptr;   // F-branch output remap table (tiny.cuh)
    void* tiny_ph = nullptr;
    void* tiny_pack = nullptr;          // the one-CTA path's tables in one allocation (TinyArgs)
    TinyArgs tiny_args{};
    size_t tiny_smem = 0;
    Radices rd_L{};
    void* twL = nullptr;     // W_L^e, e < 180 * 256 (front_f4096_kernel)
    int zsmall = 0;          // forward zak_ct with 128-thread CTAs of RB / 2 columns (c128, d = 180)
    int cnj = 0;             // zak_ct -> out_f4096 intermediate in [n][j] layout
    int outk = 0;            // output kernel: 0 generic, 1 out_f4096 (F-branch, iM = 4096)
    int fast = 0;  // specialised path id (0 = generic)
    FastPlan fp{};
    // host pipeline (dgt_execute_host)
    cudaStream_t s_in = nullptr, s_out = nullptr;
    cudaEvent_t ev_in[2] = {nullptr, nullptr}, ev_comp[2] = {nullptr, nullptr}, ev_out[2] = {nullptr, nullptr};
    void* stage_f[2] = {nullptr, nullptr};
    void* stage_c[2] = {nullptr, nullptr};
    int64_t stage_W = 0;
    // profiling (dgt_profile_begin / dgt_profile_end)
    struct ProfRec {
        int kind;
        cudaEvent_t a, b;
        double bytes, flops;
    };
    bool prof = false;
    std::vector<ProfRec> recs;
    std::vector<cudaEvent_t> pool;
    size_t pool_used = 0;
};

enum ProfKind { PK_FRONT = 0, PK_ZAK = 1, PK_OUT = 2, PK_FAST = 3, PK_ZAKCT = 4, PK_OUTF = 5, PK_ZAKADJ = 6,
                PK_OUTADJ = 7, PK_FASTADJ = 8, PK_MW = 9, PK_FRONTF = 10, PK_ZAKRR = 11, PK_TINY = 12, PK_TINYADJ = 13, PK_COUNT = 14 };
static const char* kProfNames[PK_COUNT] = {"front_fft_cufft", "zak_generic", "out_generic", "fused_fast",
                                           "zak_ct", "out_f4096", "zak_adjoint", "out_adjoint",
                                           "fused7a_t_p1", "multiwindow_interleave", "front_f4096", "zak_rr", "tiny", "tiny_adjoint"};

static cudaEvent_t prof_event(Plan* P) {
    if (P->pool_used == P->pool.size()) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        P->pool.push_back(e);
    }
    return P->pool[P->pool_used++];
}
// open a timed region on `st` (returns index or -1 when not profiling)
static int prof_open(Plan* P, cudaStream_t st) {
    if (!P->prof) return -1;
    Plan::ProfRec r{};
    r.a = prof_event(P);
    r.b = prof_event(P);
    cudaEventRecord(r.a, st);
    P->recs.push_back(r);
    return (int)P->recs.size() - 1;
}
static void prof_close(Plan* P, int h, int kind, double bytes, double flops, cudaStream_t st) {
    if (h < 0) return;
    Plan::ProfRec& r = P->recs[h];
    r.kind = kind;
    r.bytes = bytes;
    r.flops = flops;
    cudaEventRecord(r.b, st);
}

static void free_plan(Plan* P) {
    if (!P) return;
    if (P->ola) free_plan(P->ola);
    for (Plan* Q : P->mw) free_plan(Q);
    if (P->mw_d) cudaFree(P->mw_d);
    if (P->mw_sig) cudaFree(P->mw_sig);
    if (P->ola_x) cudaFree(P->ola_x);
    if (P->ola_c) cudaFree(P->ola_c);
    if (P->inv_alias & 1) P->Cinv = nullptr;
    if (P->inv_alias & 2) P->finv = nullptr;
    void* ptrs[] = {P->G, P->chirp, P->pre, P->tw_d, P->tw_m, P->E, P->rot, P->ptab, P->Cws, P->fhat,
                    P->stage_f[0], P->stage_f[1], P->stage_c[0], P->stage_c[1], P->Cinv, P->finv, P->gt64,
                    P->scrA, P->scrB, P->twL, P->tiny_dst, P->tiny_ph, P->tiny_pack, P->chR};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    free_fast(&P->fp);
    for (auto& kv : P->fft_plans) cufftDestroy(kv.second);
    for (cudaEvent_t e : P->pool) cudaEventDestroy(e);
    for (int i = 0; i < 2; ++i) {
        if (P->ev_in[i]) cudaEventDestroy(P->ev_in[i]);
        if (P->ev_comp[i]) cudaEventDestroy(P->ev_comp[i]);
        if (P->ev_out[i]) cudaEventDestroy(P->ev_out[i]);
    }
    if (P->s_in) cudaStreamDestroy(P->s_in);
    if (P->s_out) cudaStreamDestroy(P->s_out);
    delete P;
}

static int grid_for(int64_t n, int block = 256) {
    int64_t g = (n + block - 1) / block;
    return (int)std::max<int64_t>(1, std::min<int64_t>(g, 148 * 64));
}

static int get_fft_plan(Plan* P, int64_t batch, cudaStream_t st, cufftHandle* out) {
    auto it = P->fft_plans.find(batch);
    if (it == P->fft_plans.end()) {
        cufftHandle h;
        long long n = P->info.L;
        size_t wsz = 0;
        CUFFT_TRY(cufftCreate(&h));
        CUFFT_TRY(cufftMakePlanMany64(h, 1, &n, nullptr, 1, n, nullptr, 1, n,
                                      P->dtype == DGT_C64 ? CUFFT_C2C : CUFFT_Z2Z, (long long)batch, &wsz));
        P->fft_plans[batch] = h;
        it = P->fft_plans.find(batch);
    }
    CUFFT_TRY(cufftSetStream(it->second, st));
    *out = it->second;
    return DGT_OK;
}

// Length-L FFTs of nb signals (in -> out, may alias) with the plans made at plan time: one
// call when a plan for this batch exists (the front / synthesis batch), else nb calls of the
// batch-1 plan -- so dgt_execute never creates a cuFFT plan (no allocation in execute).
static int exec_fft(Plan* P, const void* in, void* out, int64_t nb, int dir, cudaStream_t st) {
    const size_t per = (size_t)P->info.L * P->esz;
    auto run = [&](cufftHandle h, const void* a, void* b) -> cufftResult {
        cufftSetStream(h, st);
        return P->dtype == DGT_C64 ? cufftExecC2C(h, (cufftComplex*)a, (cufftComplex*)b, dir)
                                   : cufftExecZ2Z(h, (cufftDoubleComplex*)a, (cufftDoubleComplex*)b, dir);
    };
    // the largest planned batch <= the signals left, repeatedly (plans exist for the front and
    // synthesis batches and every power of two below them)
    int64_t done = 0;
    while (done < nb) {
        auto it = P->fft_plans.upper_bound(nb - done);
        if (it == P->fft_plans.begin()) {   // no plan at all (not expected): make the batch-1 plan
            cufftHandle h1;
            int rc = get_fft_plan(P, 1, st, &h1);
            if (rc) return rc;
            continue;
        }
        --it;
        CUFFT_TRY(run(it->second, (const char*)in + done * per, (char*)out + done * per));
        done += it->first;
    }
    return DGT_OK;
}

static OutArgs make_out_args(const Plan* P, void* Cbuf, void* c);

template <typename T>
static int build_tables(Plan* P, const void* g_in, bool g_host, cudaStream_t st) {
    using C = cx<T>;
    const dgt_lattice_info& I = P->info;
    const int64_t L = I.L;
    // window in the caller's precision -> device
    C* g_dev = nullptr;
    CUDA_TRY(cudaMalloc(&g_dev, sizeof(C) * L));
    CUDA_TRY(cudaMemcpyAsync(g_dev, g_in, sizeof(C) * L, g_host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, st));
    double2* gt = nullptr;
    CUDA_TRY(cudaMalloc(&gt, sizeof(double2) * L));
    if (I.branch != DGT_BRANCH_FREQ) {
        // Alg. 1 line 4: g~ = pchirp(L, s1) g
        k_window_time<T><<<grid_for(L), 256, 0, st>>>(gt, g_dev, I.s1, L);
    } else {
        // Alg. 1 lines 4, 22: g^ = pchirp(L,-s0) fft(pchirp(L,s1) g) / L, in fp64
        k_window_time<T><<<grid_for(L), 256, 0, st>>>(gt, g_dev, I.s1, L);
        cufftHandle h;
        CUFFT_TRY(cufftPlan1d(&h, (int)L, CUFFT_Z2Z, 1));
        CUFFT_TRY(cufftSetStream(h, st));
        CUFFT_TRY(cufftExecZ2Z(h, (cufftDoubleComplex*)gt, (cufftDoubleComplex*)gt, CUFFT_FORWARD));
        k_window_freq_post<<<grid_for(L), 256, 0, st>>>(gt, -I.s0, L);
        CUDA_TRY(cudaStreamSynchronize(st));
        cufftDestroy(h);
    }
    CUDA_TRY(cudaMalloc(&P->G, sizeof(C) * L));
    k_window_factor<T><<<grid_for(L), 256, 0, st>>>((C*)P->G, gt, L, I.c, I.d, I.p, I.q);
    // chirp multiplied on kernel-A load: T-branch P_{s1}, F-branch P_{-s0}
    if (I.chirp_sigma % (2 * L) != 0) {
        CUDA_TRY(cudaMalloc(&P->chirp, sizeof(C) * L));
        k_chirp_table<T><<<grid_for(L), 256, 0, st>>>((C*)P->chirp, I.chirp_sigma, L);
    }
    // zak_ct (p = 1, compile-time d): the chirp factorised on the gather lattice (ZakArgs::chR);
    // NSDGT_CHR_OFF keeps the length-L table on the load
    if (P->chirp && P->zct && I.p == 1 && !std::getenv("NSDGT_CHR_OFF")) {
        CUDA_TRY(cudaMalloc(&P->chR, sizeof(C) * I.d));
        k_chirp_stride<T><<<grid_for(I.d), 256, 0, st>>>((C*)P->chR, I.chirp_sigma, L, I.c * I.q, I.d);
        const int64_t D = I.d;
        const int64_t sg = ((I.chirp_sigma % (2 * L)) + 2 * L) % (2 * L);
        P->sigD = (int)(((sg % D) * ((L + 1) % D)) % D);
    }
    if (I.branch == DGT_BRANCH_FREQ && I.pre_sigma % (2 * L) != 0) {
        CUDA_TRY(cudaMalloc(&P->pre, sizeof(C) * L));
        k_chirp_table<T><<<grid_for(L), 256, 0, st>>>((C*)P->pre, I.pre_sigma, L);
    }
    CUDA_TRY(cudaMalloc(&P->tw_d, sizeof(C) * I.d));
    k_twiddles<T><<<grid_for(I.d), 256, 0, st>>>((C*)P->tw_d, I.d);
    CUDA_TRY(cudaMalloc(&P->tw_m, sizeof(C) * I.iM));
    k_twiddles<T><<<grid_for(I.iM), 256, 0, st>>>((C*)P->tw_m, I.iM);
    if (P->tiny && I.branch == DGT_BRANCH_FREQ) {   // W_L for the one-CTA path's DFT_L
        CUDA_TRY(cudaMalloc(&P->twL, sizeof(C) * L));
        k_twiddles<T><<<grid_for(L), 256, 0, st>>>((C*)P->twL, L);
    }
    if (P->front) {
        CUDA_TRY(cudaMalloc(&P->twL, sizeof(C) * 180 * 256));
        k_twiddles_prefix<T><<<grid_for(180 * 256), 256, 0, st>>>((C*)P->twL, I.L, 180 * 256);
    }
    if (I.branch != DGT_BRANCH_FREQ) {
        CUDA_TRY(cudaMalloc(&P->E, sizeof(C) * I.N));
        CUDA_TRY(cudaMalloc(&P->rot, sizeof(int) * I.N));
        k_post_time<T><<<grid_for(I.N), 256, 0, st>>>((C*)P->E, P->rot, I.N, I.C1, I.s1, I.a, I.b, I.M);
    } else {
        CUDA_TRY(cudaMalloc(&P->ptab, sizeof(C) * 2 * I.N));
        k_phase_table<T><<<grid_for(2 * I.N), 256, 0, st>>>((C*)P->ptab, I.N);
    }
    // experiment (NSDGT_OUTCL=1): out_f4096 in clusters of 3 CTAs staging whole output rows in
    // distributed shared memory -- parity-tested, measured slower (0.64 against 0.44 ms per 16
    // signals: two cluster barriers and 64 KB of DSMEM reads per CTA), off by default
    if (P->outk == 2 && P->cnj && I.iN % 3 == 0 && I.N == 3 * 4096 && I.iM == 4096 && std::getenv("NSDGT_OUTCL")) {
        int* bad = nullptr;
        CUDA_TRY(cudaMalloc(&bad, sizeof(int)));
        CUDA_TRY(cudaMemsetAsync(bad, 0, sizeof(int), st));
        const OutArgs B = make_out_args(P, nullptr, nullptr);
        const int64_t n = I.iN * I.iM;
        k_cl_check<T><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(B, bad);
        int hb = 1;
        CUDA_TRY(cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaStreamSynchronize(st));
        cudaFree(bad);
        P->outcl = hb == 0 ? 1 : 0;
        if (P->outcl)
            CUDA_TRY(cudaFuncSetAttribute(out_f4096_kernel<T, 2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)(kOutF4096Elems * sizeof(C))));
    }
    if (P->tiny && I.branch == DGT_BRANCH_FREQ) {   // the one-CTA path's output remap table
        const int64_t n = I.iM * I.iN;
        CUDA_TRY(cudaMalloc(&P->tiny_dst, sizeof(unsigned int) * n));
        CUDA_TRY(cudaMalloc(&P->tiny_ph, sizeof(C) * n));
        const OutArgs B = make_out_args(P, nullptr, nullptr);
        k_tiny_remap<T><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(B, P->tiny_dst, (C*)P->tiny_ph, (int)I.iM, (int)I.iN);
    }
    if (P->tiny) {
        // every table the one-CTA kernel reads, copied into one allocation: after the L2 flush
        // of a latency measurement each separate allocation costs its own cold page walk
        const bool freq = I.branch == DGT_BRANCH_FREQ;
        const int64_t LQ = I.iM * I.iN;
        struct Part { const void* src; size_t bytes; const void** dst; };
        TinyArgs& TA = P->tiny_args;
        std::vector<Part> parts = {{P->G, sizeof(C) * L, &TA.G}, {P->chirp, P->chirp ? sizeof(C) * L : 0, &TA.chirp},
                                   {P->twL, freq ? sizeof(C) * L : 0, &TA.twL}, {P->tw_d, sizeof(C) * I.d, &TA.twd},
                                   {P->tw_m, sizeof(C) * I.iM, &TA.twm}, {P->tiny_ph, freq ? sizeof(C) * LQ : 0, &TA.oph},
                                   {P->tiny_dst, freq ? sizeof(unsigned int) * LQ : 0, &TA.odst},
                                   {P->pre, P->pre ? sizeof(C) * L : 0, &TA.pre}};
        size_t tot = 0;
        for (auto& pt : parts) tot += (pt.bytes + 255) / 256 * 256;
        CUDA_TRY(cudaMalloc(&P->tiny_pack, tot));
        size_t off = 0;
        for (auto& pt : parts) {
            if (!pt.bytes) { *pt.dst = nullptr; continue; }
            CUDA_TRY(cudaMemcpyAsync((char*)P->tiny_pack + off, pt.src, pt.bytes, cudaMemcpyDeviceToDevice, st));
            *pt.dst = (char*)P->tiny_pack + off;
            off += (pt.bytes + 255) / 256 * 256;
        }
    }
    CUDA_TRY(cudaGetLastError());
    int rc = build_fast<T>(&P->fp, P->info, gt, P->E, (P->flags & DGT_FORCE_GENERIC) != 0, st);
    if (rc) return rc;
    P->fast = P->fp.kind;
    CUDA_TRY(cudaStreamSynchronize(st));
    cudaFree(g_dev);
    P->gt64 = gt;   // kept for dgt_window_dual
    return DGT_OK;
}

// Arguments of the output kernels (forward and adjoint): intermediate C, coefficients c, the
// Alg. 1 constants reduced mod 2N / L and the F-branch remap's per-step deltas.
static OutArgs make_out_args(const Plan* P, void* Cbuf, void* c) {
    const dgt_lattice_info& I = P->info;
    OutArgs B{};
    B.C = Cbuf; B.out = c; B.iM = I.iM; B.iN = I.iN; B.q = I.q; B.d = I.d; B.NT = P->NT;
    B.rd = P->rd_m; B.tw = P->tw_m; B.branch = (int)I.branch; B.cnj = P->cnj;
    B.gscr = P->gB ? P->scrB : nullptr; B.gstride = (int64_t)P->smemB;
    B.grouped = I.branch == DGT_BRANCH_FREQ ? 1 : 0;
    B.E = P->E; B.rot = P->rot; B.M = I.M; B.N = I.N;
    B.ptab = P->ptab; B.L = I.L; B.b = I.b; B.Nr = I.N_r; B.ar = I.a_r; B.s1 = I.s1;
    const int64_t twoN = 2 * I.N;
    auto nm = [](int64_t v, int64_t m) { return ((v % m) + m) % m; };
    B.C1 = nm(I.C1, twoN); B.C2 = nm(I.C2, twoN); B.C3 = nm(I.C3, twoN); B.C4 = nm(I.C4, twoN);
    B.C5 = nm(I.C5, twoN); B.C6 = nm(I.C6, I.L);
    B.sar = (((-(I.s1 % I.L)) * (I.a_r % I.L)) % I.L + I.L) % I.L;
    B.D1 = (unsigned int)((256 * B.C1) % twoN);
    B.D5 = (unsigned int)((256 * B.C5) % twoN);
    B.DX = (unsigned int)(((__int128)256 * B.sar) % I.L);
    B.invb = (unsigned int)(0xffffffffull / (unsigned long long)I.b);
    B.inv2N = ~0ull / (unsigned long long)twoN;
    B.invL = ~0ull / (unsigned long long)I.L;
    return B;
}

// F-branch front end for nb signals (Alg. 1 line 23): f^ = fft(pchirp(L, s1) f),
// unnormalised, into P->fhat (sized for P->fb signals); P_{-s0} is applied on the Zak load.
// One batched cuFFT call per front batch (config 4: 16 us per signal at batch 16 against
// 36 us one signal at a time).
template <typename T>
static int launch_front(Plan* P, const void* f, int64_t nb, cudaStream_t st) {
    using C = cx<T>;
    const dgt_lattice_info& I = P->info;
    const bool real_in = (P->flags & DGT_REAL_INPUT) != 0;
    const double e = (double)sizeof(C), ein = real_in ? e / 2 : e, L = (double)I.L;
    const int ph = prof_open(P, st);
    if (P->front) {
        FrontArgs FA{};
        FA.f = f; FA.real_in = real_in ? 1 : 0; FA.pre = P->pre; FA.H = P->fhat;
        FA.tw = P->tw_m; FA.twL = P->twL; FA.L = I.L;
        CUDA_TRY(launch_pdl(front_f4096_kernel<T, kFrontMinB, kFrontRes>, dim3(180 / kFrontRes, (unsigned)nb),
                            dim3(256 * kFrontRes), front_smem(sizeof(C)), st, FA));
        // a length-4096 DFT of 180 residues per signal (the DFT_180 runs in zak_rr0_kernel)
        prof_close(P, ph, PK_FRONTF, nb * L * ein, nb * 5.0 * L * 12.0, st);
        CUDA_TRY(cudaGetLastError());
        return DGT_OK;
    }
    const void* fin = f;
    if (real_in || P->pre) {
        k_prechirp<T><<<grid_for(nb * I.L), 256, 0, st>>>((C*)P->fhat, f, real_in ? 1 : 0, (const C*)P->pre, I.L,
                                                          nb * I.L);
        fin = P->fhat;
    }
    int rc = exec_fft(P, fin, P->fhat, nb, CUFFT_FORWARD, st);
    if (rc) return rc;
    // Table 1 "Freq. shear": one length-L FFT of f per signal (4 L log2 L)
    prof_close(P, ph, PK_FRONT, nb * L * ein, nb * 4.0 * L * std::log2(L), st);
    CUDA_TRY(cudaGetLastError());
    return DGT_OK;
}

template <typename T>
static int launch_chunk(Plan* P, const void* f, void* c, int64_t Wc, cudaStream_t st, const void* spectra) {
    using C = cx<T>;
    const dgt_lattice_info& I = P->info;
    const bool real_in = (P->flags & DGT_REAL_INPUT) != 0;
    const void* src = f;
    int real_src = real_in ? 1 : 0;
    const double e = (double)sizeof(C), ein = real_in ? e / 2 : e;
    const double L = (double)I.L, MN = (double)I.M * (double)I.N;
    const double lg_d = std::log2((double)I.d), lg_m = std::log2((double)I.iM);
    if (I.branch == DGT_BRANCH_FREQ) {
        src = spectra;   // f^ of these signals (launch_front)
        real_src = 0;
    }
    // Eq. (rect-flops): 8Lq + 4L log2 d + 4MN log2 d + 4MN log2 M, plus 6MN for the phase
    const double fl_zak = Wc * (8.0 * L * I.q / I.p + 4.0 * L * lg_d + 4.0 * MN * lg_d);
    const double fl_out = Wc * (4.0 * MN * lg_m + 6.0 * MN);
    const double by_in = (I.branch == DGT_BRANCH_FREQ ? 0.0 : Wc * L * ein) + L * e;  // f (T) + window factors
    const double by_out = Wc * MN * e;
    if (P->fast) {
        const int ph = prof_open(P, st);
        int rc = launch_fast<T>(&P->fp, src, real_src, P->Cws, c, Wc, st);
        if (rc) return rc;
        prof_close(P, ph, PK_FAST, by_in + by_out, fl_zak + fl_out, st);
        CUDA_TRY(cudaGetLastError());
        return DGT_OK;
    }
    ZakArgs A{};
    A.f = src; A.real_in = real_src; A.chirp = P->chirp; A.G = P->G; A.C = P->Cws;
    A.chR = P->chR; A.sigD = P->sigD;
    A.L = I.L; A.c = I.c; A.d = I.d; A.p = I.p; A.q = I.q; A.iM = I.iM;
    A.RB = P->RB; A.rd = P->rd_d; A.tw = P->tw_d; A.allu = P->allu; A.cnj = P->cnj;
    A.gscr = P->gA ? P->scrA : nullptr; A.gstride = (int64_t)std::max(P->smemA, P->smemAinv);
    const int nrb = (int)((I.c + P->RB - 1) / P->RB);
    int ph = prof_open(P, st);
    cudaError_t le;
    if (P->front)
        le = launch_pdl(zak_rr0_kernel<T, 8, kZrr0MinB>, dim3((unsigned)(I.c / 8 * I.q), (unsigned)Wc), dim3(128),
                        zrr_smem<T>(), st, A);
    else if (P->zrr)
        le = launch_pdl(zak_rr_kernel<T, 8, kZrrMinB>, dim3((unsigned)(I.c / 8 * I.q), (unsigned)Wc), dim3(128),
                        zrr_smem<T>(), st, A);
    else if (P->zsmall && sizeof(C) == 16)
        le = launch_pdl(zak_ct_kernel<T, 180, 4, 2, 128>, dim3(2 * nrb * (unsigned)I.q, (unsigned)Wc), dim3(128),
                        P->smemA / 2, st, A);
    else if (P->zct == 180 && sizeof(C) == 16)
        le = launch_pdl(zak_ct_kernel<T, 180, 4, 4>, dim3(nrb * (unsigned)I.q, (unsigned)Wc), dim3(256), P->smemA, st, A);
    else if (P->zct == 180)
        le = launch_pdl(zak_ct_kernel<T, 180, 4, 8>, dim3(nrb * (unsigned)I.q, (unsigned)Wc), dim3(256), P->smemA, st, A);
    else if (P->zct == 720)
        le = launch_pdl(zak_ct_kernel<T, 720, 4, 1>, dim3(nrb * (unsigned)I.q, (unsigned)Wc), dim3(256), P->smemA, st, A);
    else
        le = launch_pdl(zak_kernel<T>, dim3(nrb * (unsigned)I.q, (unsigned)Wc), dim3(256), P->gA ? 0 : P->smemA, st, A);
    CUDA_TRY(le);
    prof_close(P, ph, (P->zrr || P->front) ? PK_ZAKRR : P->zct ? PK_ZAKCT : PK_ZAK, by_in, fl_zak, st);
    const OutArgs B = make_out_args(P, P->Cws, c);
    const int ntiles = B.grouped ? (int)(I.q * ((I.d + P->NT - 1) / P->NT)) : (int)((I.iN + P->NT - 1) / P->NT);
    ph = prof_open(P, st);
    if (P->outk == 1)
        le = launch_pdl(out_f4096_kernel<T, 3>, dim3((unsigned)I.iN, (unsigned)Wc), dim3(256), kOutF4096Elems * sizeof(C),
                        st, B);
    else if (P->outk == 2 && P->outcl)
        le = launch_pdl_cluster(out_f4096_kernel<T, 2, true>, dim3((unsigned)I.iN, (unsigned)Wc), dim3(256),
                                kOutF4096Elems * sizeof(C), st, 3u, B);
    else if (P->outk == 2)
        le = launch_pdl(out_f4096_kernel<T, 2>, dim3((unsigned)I.iN, (unsigned)Wc), dim3(256), kOutF4096Elems * sizeof(C),
                        st, B);
    else if (P->outct == 200)
        le = launch_pdl(out_kernel<T, 200>, dim3(ntiles, (unsigned)Wc), dim3(256), P->smemB, st, B);
    else
        le = launch_pdl(out_kernel<T>, dim3(ntiles, (unsigned)Wc), dim3(256), P->gB ? 0 : P->smemB, st, B);
    CUDA_TRY(le);
    prof_close(P, ph, P->outk ? PK_OUTF : PK_OUT, by_out, fl_out, st);
    CUDA_TRY(cudaGetLastError());
    return DGT_OK;
}

// The constant-memory twiddles W_180, W_720 of fft_ct / dft_pq (same values for every plan;
// long-double cos/sin of exact residues on the host, rounded once).  __constant__ memory is per
// device: uploaded once per device (a mutex-guarded set of devices; a failed upload is retried
// by the next plan instead of poisoning it).  Used by the compile-time Zak kernels, zak_rr* and
// the one-CTA path's compile-time variant.
static bool upload_const_twiddles() {
    static std::mutex tw_mu;
    static std::set<int> tw_done;
    std::lock_guard<std::mutex> lk(tw_mu);
    auto fill = [](auto& dsym, auto& fsym, int n) {
        std::vector<double2> d(n);
        std::vector<float2> f(n);
        for (int k = 0; k < n; ++k) {
            const long double th = -2.0L * 3.141592653589793238462643383279502884L * (long double)k / (long double)n;
            d[k] = make_double2((double)cosl(th), (double)sinl(th));
            f[k] = make_float2((float)d[k].x, (float)d[k].y);
        }
        return cudaMemcpyToSymbol(dsym, d.data(), sizeof(double2) * n) == cudaSuccess &&
               cudaMemcpyToSymbol(fsym, f.data(), sizeof(float2) * n) == cudaSuccess;
    };
    int dev = -1;
    cudaGetDevice(&dev);
    if (tw_done.count(dev)) return true;
    if (!fill(c_tw180d, c_tw180f, 180) || !fill(c_tw720d, c_tw720f, 720)) return false;
    tw_done.insert(dev);
    return true;
}

template <typename T>
static int configure(Plan* P, int64_t max_chunk) {
    const dgt_lattice_info& I = P->info;
    const size_t e = sizeof(cx<T>);
    int dev = 0;
    CUDA_TRY(cudaGetDevice(&dev));
    int smem_optin = 0, l2 = 0;
    CUDA_TRY(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    CUDA_TRY(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev));
    const size_t budget = std::min<size_t>((size_t)smem_optin, 200 * 1024);
    if (I.d > (1 << 30) || I.iM > (1 << 30)) return fail(DGT_EUNSUPPORTED, "inner length too large");
    // the generic kernels index within one signal in 32-bit arithmetic
    if (I.L >= ((int64_t)1 << 31) || I.M * I.N >= ((int64_t)1 << 31) || 2 * I.N >= ((int64_t)1 << 31))
        return fail(DGT_EUNSUPPORTED, "signal too long for 32-bit in-signal indexing");
    P->rd_d = make_radices((int)I.d);
    P->rd_m = make_radices((int)I.iM);
    if (P->rd_d.nst > kMaxStages || P->rd_m.nst > kMaxStages) return fail(DGT_EUNSUPPORTED, "too many FFT stages");
    // kernel A: residues per CTA for >= 32-byte gathers, within the smem budget
    auto smemA = [&](int rb) { return (size_t)rb * (2 * I.p + 1) * I.d * e; };
    int rb = (int)std::min<int64_t>(I.c, std::max<int64_t>(1, 64 / (int64_t)e));
    // few residue classes (small c, e.g. config 2: c = 50): fewer residues per CTA so that one
    // signal still spreads over >= 2 CTAs per SM
    while (rb > 1 && ((I.c + rb - 1) / rb) * I.q < 2 * 148) --rb;
    while (rb > 1 && smemA(rb) > budget) --rb;
    // d too large for shared memory: the Zak kernels keep their buffers in a per-CTA global
    // scratch (L2-resident; correct, slower)
    P->gA = smemA(rb) > budget ? 1 : 0;
    P->RB = rb;
    P->smemA = smemA(rb);
    // p = 1: all-u mode when two regions of q RB d fit (config 4: 92 KB, 2 CTAs per SM)
    const size_t smem_allu = (size_t)2 * I.q * rb * I.d * e;
    if (I.p == 1 && smem_allu <= budget && !std::getenv("NSDGT_ZAK_PERU")) {
        P->allu = 1;
        P->smemA = std::max(P->smemA, smem_allu);
    }
    auto smemB = [&](int nt) { return (size_t)2 * nt * I.iM * e; };
    int nt = (int)std::min<int64_t>(I.iN, 16);
    // long columns: keep >= 2 CTAs per SM (config 4: 2 x 4096 x 16 B per column, NT = 4 left
    // one CTA of 8 warps per SM, latency-bound on its loads)
    while (nt > 1 && smemB(nt) > budget / 2 && smemB(nt) > 48 * 1024) --nt;
    if (const char* ev = std::getenv("NSDGT_OUT_NT")) nt = std::max(1, std::atoi(ev));   // experiment
    while (nt > 1 && smemB(nt) > budget) --nt;
    P->gB = smemB(nt) > budget ? 1 : 0;   // likewise for the output kernels
    P->NT = nt;
    P->smemB = smemB(nt);
    CUDA_TRY(cudaFuncSetAttribute(zak_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, P->gA ? 0 : (int)P->smemA));
    // compile-time Zak kernels (p = 1, q = 4, all-u mode): d = 180 with RB = 64 / e columns
    // (config 4), d = 720 with one column per CTA (config 2)
    P->zct = 0;
    // DGT_FORCE_GENERIC: the runtime-radix chunk kernels only (no compile-time, register-resident,
    // one-CTA or fused kernel)
    const bool forced = (P->flags & DGT_FORCE_GENERIC) != 0;
    if (P->allu && I.q == 4 && I.c % P->RB == 0 && !std::getenv("NSDGT_ZAK_RT") && !forced) {
        if (I.d == 180 && P->RB == (int)(64 / e)) P->zct = 180;
        if (I.d == 720 && P->RB == 1) P->zct = 720;
        // c128 forward: 128-thread CTAs of RB / 2 columns (32-byte rows), 4 CTAs per SM -- finer
        // barriers than 2 CTAs of 8 warps (config 4: 0.497 -> 0.474 ms per 16 signals); the
        // adjoint measured slower that way (0.492 -> 0.527) and keeps RB
        P->zsmall = (P->zct == 180 && e == 16 && !std::getenv("NSDGT_ZCT_BIG")) ? 1 : 0;
        // register-resident DFT_180 passes (zak_rr.cuh), 8 residues per 128-thread CTA;
        // NSDGT_ZAK_CT keeps zak_ct (A/B experiment)
        P->zrr = (P->zct == 180 && I.c % 8 == 0 && !std::getenv("NSDGT_ZAK_CT")) ? 1 : 0;
        // frequency shear with L = 180 x 4096 = d x (c q): the length-L FFT as front_f4096_kernel
        // (4096-point DFTs of the 180 residues) + one DFT_180 pass pair inside the Zak kernel
        // (NSDGT_FRONT_CUFFT keeps cuFFT, A/B experiment)
        P->front = (P->zrr && I.branch == DGT_BRANCH_FREQ && I.L == 180 * 4096 && I.c * I.q == 4096 &&
                    !std::getenv("NSDGT_FRONT_CUFFT")) ? 1 : 0;
    }
    if (P->zct) {
        if (!upload_const_twiddles()) return fail(DGT_ECUDA, "constant twiddle upload");
        CUDA_TRY(cudaFuncSetAttribute(zak_ct_kernel<T, 180, 4, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P->smemA));
        CUDA_TRY(cudaFuncSetAttribute(zak_ct_kernel<T, 180, 4, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P->smemA));
        CUDA_TRY(cudaFuncSetAttribute(zak_ct_kernel<T, 720, 4, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P->smemA));
        CUDA_TRY(cudaFuncSetAttribute(zak_ct_kernel<T, 180, 4, 2, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P->smemA / 2));
        CUDA_TRY(cudaFuncSetAttribute(zak_rr_kernel<T, 8, kZrrMinB>, cudaFuncAttributeMaxDynamicSharedMemorySize, zrr_smem<T>()));
        CUDA_TRY(cudaFuncSetAttribute(zak_rr0_kernel<T, 8, kZrr0MinB>, cudaFuncAttributeMaxDynamicSharedMemorySize, zrr_smem<T>()));
        CUDA_TRY(cudaFuncSetAttribute(front_f4096_kernel<T, kFrontMinB, kFrontRes>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, front_smem((int)e)));
        CUDA_TRY(cudaFuncSetAttribute(front_f4096_kernel<T, kFrontMinB, kFrontRes, true>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, front_smem((int)e)));
        CUDA_TRY(cudaFuncSetAttribute(zak_rr0_adj_kernel<T, 8, kZrr0MinB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      zrr_smem<T>()));
    }
    CUDA_TRY(cudaFuncSetAttribute(out_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, P->gB ? 0 : (int)P->smemB));
    // compile-time output DFT for M' = 200 (config 2, time shear)
    P->outct = (I.branch != DGT_BRANCH_FREQ && I.iM == 200 && !P->gB && !std::getenv("NSDGT_OUT_GENERIC") && !forced) ? 200 : 0;
    if (P->outct) CUDA_TRY(cudaFuncSetAttribute(out_kernel<T, 200>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P->smemB));
    // out_f4096: 2 CTAs per SM for c128 (128 registers, measured faster than 3 CTAs at 80
    // registers with spills), 3 for c64
    P->outk = (I.branch == DGT_BRANCH_FREQ && I.iM == 4096 && !std::getenv("NSDGT_OUT_GENERIC") && !forced) ? (e == 16 ? 2 : 1) : 0;
    if (P->outk && std::getenv("NSDGT_OUTF_MINB")) P->outk = std::atoi(std::getenv("NSDGT_OUTF_MINB")) == 2 ? 2 : 1;   // experiment
    // zak_ct (d = 180) feeding out_f4096: the intermediate is stored [n][j] so the output
    // kernel's column loads are contiguous (NSDGT_CNJ_OFF: the generic [j][kappa][n'] layout)
    P->cnj = (P->outk && P->zct == 180 && !std::getenv("NSDGT_CNJ_OFF")) ? 1 : 0;
    CUDA_TRY(cudaFuncSetAttribute(out_f4096_kernel<T, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(kOutF4096Elems * e)));
    CUDA_TRY(cudaFuncSetAttribute(out_f4096_kernel<T, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(kOutF4096Elems * e)));
    // short signals: the whole transform of a signal in one CTA when its tables and buffers fit
    // 160 KB of shared memory (config 1); NSDGT_TINY_OFF keeps the chunked kernels
    {
        const bool freq = I.branch == DGT_BRANCH_FREQ;
        const int64_t te = tiny_elems(I.L, I.q, I.p, I.d, I.iM, freq);
        const Radices rl = make_radices((int)std::min<int64_t>(I.L, 1 << 30));
        P->tiny = (!std::getenv("NSDGT_TINY_OFF") && !forced && te * (int64_t)e <= 160 * 1024 && I.iM * I.iN == I.L / I.p * I.q &&
                   I.iM == I.c * I.q && rl.nst <= kMaxStages) ? 1 : 0;
        if (P->tiny) {
            P->rd_L = rl;
            P->tiny_smem = (size_t)te * e;
            CUDA_TRY(cudaFuncSetAttribute(tiny_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P->tiny_smem));
            CUDA_TRY(cudaFuncSetAttribute(tiny_adj_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P->tiny_smem));
            // config 1's shape as a compile-time variant (NSDGT_TINY_RT keeps the runtime one)
            if (I.L == 240 && I.c == 5 && I.d == 8 && I.p == 2 && I.q == 3 && freq && !std::getenv("NSDGT_TINY_RT")) {
                if (!upload_const_twiddles()) return fail(DGT_ECUDA, "constant twiddle upload");   // dft_pq's W_15
                P->tiny = 2;
                CUDA_TRY(cudaFuncSetAttribute(tiny_kernel<T, 240, 5, 8, 2, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)P->tiny_smem));
                CUDA_TRY(cudaFuncSetAttribute(tiny_adj_kernel<T, 240, 5, 8, 2, 3>,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P->tiny_smem));
            }
        }
    }
    P->inv_generic = std::getenv("NSDGT_INV_GENERIC") ? 1 : 0;
    // synthesis kernels (the adjoints of zak_kernel / out_kernel)
    P->smemAinv = (size_t)P->RB * (2 * I.p + 1) * I.d * e;
    CUDA_TRY(cudaFuncSetAttribute(zak_adj_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, P->gA ? 0 : (int)P->smemAinv));
    CUDA_TRY(cudaFuncSetAttribute(out_adj_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, P->gB ? 0 : (int)P->smemB));
    if (P->outct == 200)
        CUDA_TRY(cudaFuncSetAttribute(out_adj_kernel<T, 200>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P->smemB));
    if (P->zct) {
        CUDA_TRY(cudaFuncSetAttribute(zak_ct_adj_kernel<T, 180, 4, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P->smemA));
        CUDA_TRY(cudaFuncSetAttribute(zak_ct_adj_kernel<T, 180, 4, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P->smemA));
        CUDA_TRY(cudaFuncSetAttribute(zak_ct_adj_kernel<T, 720, 4, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P->smemA));
    }
    CUDA_TRY(cudaFuncSetAttribute(out_f4096_adj_kernel<T, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(kOutF4096Elems * e)));
    CUDA_TRY(cudaFuncSetAttribute(out_f4096_adj_kernel<T, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(kOutF4096Elems * e)));
    // chunk: signals per launch pair.  Up to ~1 GiB of intermediate: the launches then span
    // many waves (config 4: 1.88 ms at 1 signal per launch, the L2-resident size; 1.49 ms at
    // 16).  The kernels are compute- or latency-bound, so the intermediate's trip through HBM
    // costs less than the launch tails.  NSDGT_CHUNK_L2 restores the L2-sized chunk (experiment).
    const size_t per_sig = (size_t)I.iM * I.iN * e;
    int64_t ch = std::max<int64_t>(1, (int64_t)((size_t)(l2 > 0 ? l2 : (64 << 20)) * 2 / 5 / per_sig));
    if (!std::getenv("NSDGT_CHUNK_L2")) ch = std::max<int64_t>(ch, (int64_t)((1ull << 30) / per_sig));
    // the chunk is gridDim.y of the zak / out kernels and their adjoints (<= 65535); 8192
    // signals of any lattice fill the GPU many times over, so tiny signals do not size a
    // ~1 GiB workspace and cuFFT batches of 10^5 at plan time
    ch = std::min<int64_t>(ch, kMaxChunk);
    if (max_chunk > 65535) return fail(DGT_EINVAL, "max_chunk > 65535 (grid y limit of the chunk kernels)");
    P->inv_chunk = max_chunk > 0 ? max_chunk : ch;
    if (max_chunk > 0) ch = max_chunk;
    P->chunk = ch;
    return DGT_OK;
}

static int alloc_workspace(Plan* P, int64_t Wc) {
    const dgt_lattice_info& I = P->info;
    if (P->Cws) return DGT_OK;
    // global per-CTA scratch of the Zak / output kernels when their buffers exceed shared memory
    const int64_t wmax = std::max<int64_t>(Wc, P->inv_chunk);
    if (P->gA) {
        const int64_t ctas = ((I.c + P->RB - 1) / P->RB) * I.q * wmax;
        CUDA_TRY(cudaMalloc(&P->scrA, (size_t)ctas * std::max(P->smemA, P->smemAinv)));
    }
    if (P->gB) {
        const int64_t tiles = (I.branch == DGT_BRANCH_FREQ ? I.q * ((I.d + P->NT - 1) / P->NT) : (I.iN + P->NT - 1) / P->NT);
        CUDA_TRY(cudaMalloc(&P->scrB, (size_t)tiles * wmax * P->smemB));
    }
    size_t need = P->fast ? fast_workspace_bytes(&P->fp, Wc) : (size_t)Wc * I.iM * I.iN * P->esz;
    CUDA_TRY(cudaMalloc(&P->Cws, need));
    P->ws_bytes = need;
    if (I.branch == DGT_BRANCH_FREQ && !P->fast) {
        // front batch: a multiple of the chunk holding ~192 MB of spectra (at least one chunk)
        const size_t per = (size_t)I.L * P->esz;
        const int64_t want = std::max<int64_t>(1, (int64_t)((192ull << 20) / per));
        P->fb = std::max<int64_t>(1, want / Wc) * Wc;
        CUDA_TRY(cudaMalloc(&P->fhat, (size_t)P->fb * per));
        P->ws_bytes += (size_t)P->fb * per;
        // the cuFFT plans execute uses: the front and synthesis batches and the powers of two
        // below them (ragged batches run as a few batched calls; no plan is made in execute)
        P->ib = std::max<int64_t>(1, want / P->inv_chunk) * P->inv_chunk;
        std::vector<int64_t> sizes = {P->fb, P->ib};
        for (int64_t b = 1; b < std::max(P->fb, P->ib); b *= 2) sizes.push_back(b);
        for (int64_t b : sizes) {
            cufftHandle h;
            int rc = get_fft_plan(P, b, nullptr, &h);
            if (rc) return rc;
        }
    }
    // synthesis workspace (dgt_execute_inverse), also made here so that no execute entry point
    // allocates: the forward chunk intermediate and spectra serve it when they have its size
    // (one plan never runs two executes at once -- include/nsdgt.h), else its own buffers
    if (!P->fast || P->inv_generic) {
        const size_t inv_need = (size_t)P->inv_chunk * I.iM * I.iN * P->esz;
        if (!P->fast && P->inv_chunk <= Wc) {
            P->Cinv = P->Cws;
            P->inv_alias |= 1;
        } else {
            CUDA_TRY(cudaMalloc(&P->Cinv, inv_need));
            P->ws_bytes += inv_need;
        }
        if (I.branch == DGT_BRANCH_FREQ) {
            if (P->fhat && P->ib <= P->fb) {
                P->finv = P->fhat;
                P->inv_alias |= 2;
            } else {
                CUDA_TRY(cudaMalloc(&P->finv, (size_t)P->ib * I.L * P->esz));
                P->ws_bytes += (size_t)P->ib * I.L * P->esz;
            }
        }
    }
    return DGT_OK;
}

// Synthesis of Wc signals: c (device, Wc x M x N) -> f (device, Wc x L complex).
template <typename T>
static int launch_inverse_chunk(Plan* P, const void* c, void* f, int64_t Wc, cudaStream_t st, void* spectra) {
    using C = cx<T>;
    const dgt_lattice_info& I = P->info;
    const double e = (double)sizeof(C), L = (double)I.L, MN = (double)I.M * (double)I.N;
    const OutArgs B = make_out_args(P, P->Cinv, const_cast<void*>(c));
    const int ntiles = B.grouped ? (int)(I.q * ((I.d + P->NT - 1) / P->NT)) : (int)((I.iN + P->NT - 1) / P->NT);
    int ph = prof_open(P, st);
    if (P->outk == 2)
        CUDA_TRY(launch_pdl(out_f4096_adj_kernel<T, 2>, dim3((unsigned)I.iN, (unsigned)Wc), dim3(256),
                            kOutF4096Elems * sizeof(C), st, B));
    else if (P->outk == 1)
        CUDA_TRY(launch_pdl(out_f4096_adj_kernel<T, 3>, dim3((unsigned)I.iN, (unsigned)Wc), dim3(256),
                            kOutF4096Elems * sizeof(C), st, B));
    else
        CUDA_TRY(P->outct == 200 ? launch_pdl(out_adj_kernel<T, 200>, dim3(ntiles, (unsigned)Wc), dim3(256), P->smemB, st, B)
                                 : launch_pdl(out_adj_kernel<T>, dim3(ntiles, (unsigned)Wc), dim3(256), P->gB ? 0 : P->smemB, st, B));
    prof_close(P, ph, PK_OUTADJ, Wc * MN * e, Wc * (4.0 * MN * std::log2((double)I.iM) + 6.0 * MN), st);
    ZakArgs A{};
    A.f = nullptr; A.real_in = 0; A.chirp = P->chirp; A.G = P->G; A.C = P->Cinv;
    A.L = I.L; A.c = I.c; A.d = I.d; A.p = I.p; A.q = I.q; A.iM = I.iM;
    A.RB = P->RB; A.rd = P->rd_d; A.tw = P->tw_d; A.allu = 0; A.cnj = P->cnj;
    A.gscr = P->gA ? P->scrA : nullptr; A.gstride = (int64_t)std::max(P->smemA, P->smemAinv);
    const int nrb = (int)((I.c + P->RB - 1) / P->RB);
    const bool freq = I.branch == DGT_BRANCH_FREQ;
    void* zout = freq ? spectra : f;
    const double lg_d = std::log2((double)I.d);
    ph = prof_open(P, st);
    if (P->front)   // config 4: the register-resident adjoint, h(r, x) for front_f4096<..., ADJ>
        CUDA_TRY(launch_pdl(zak_rr0_adj_kernel<T, 8, kZrr0MinB>, dim3((unsigned)(I.c / 8 * I.q), (unsigned)Wc),
                            dim3(128), zrr_smem<T>(), st, A, zout));
    else if (P->zct == 180 && sizeof(C) == 16)
        CUDA_TRY(launch_pdl(zak_ct_adj_kernel<T, 180, 4, 4>, dim3(nrb * (unsigned)I.q, (unsigned)Wc), dim3(256), P->smemA,
                            st, A, zout));
    else if (P->zct == 180)
        CUDA_TRY(launch_pdl(zak_ct_adj_kernel<T, 180, 4, 8>, dim3(nrb * (unsigned)I.q, (unsigned)Wc), dim3(256), P->smemA,
                            st, A, zout));
    else if (P->zct == 720)
        CUDA_TRY(launch_pdl(zak_ct_adj_kernel<T, 720, 4, 1>, dim3(nrb * (unsigned)I.q, (unsigned)Wc), dim3(256), P->smemA,
                            st, A, zout));
    else
        CUDA_TRY(launch_pdl(zak_adj_kernel<T>, dim3(nrb * (unsigned)I.q, (unsigned)Wc), dim3(256),
                            P->gA ? 0 : P->smemAinv, st, A, zout));
    prof_close(P, ph, PK_ZAKADJ, Wc * L * e + L * e, Wc * (8.0 * L * I.q / I.p + 4.0 * L * lg_d + 4.0 * MN * lg_d), st);
    CUDA_TRY(cudaGetLastError());
    return DGT_OK;
}

// F-branch synthesis tail for nb signals: the adjoint of f^ = fft(pchirp(L, s1) f) -- one
// batched unnormalised inverse FFT of the spectra (P->finv), then conj(pchirp(L, s1)).
template <typename T>
static int launch_inverse_tail(Plan* P, void* f, int64_t nb, cudaStream_t st) {
    using C = cx<T>;
    const dgt_lattice_info& I = P->info;
    const double e = (double)sizeof(C), L = (double)I.L;
    const int ph = prof_open(P, st);
    if (P->front) {   // the adjoint of front_f4096 (4096-point DFTs per residue, stride-180 writes)
        FrontArgs FA{};
        FA.f = P->finv; FA.real_in = 0; FA.pre = P->pre; FA.H = f; FA.tw = P->tw_m; FA.twL = P->twL; FA.L = I.L;
        CUDA_TRY(launch_pdl(front_f4096_kernel<T, kFrontMinB, kFrontRes, true>, dim3(180 / kFrontRes, (unsigned)nb),
                            dim3(256 * kFrontRes), front_smem(sizeof(C)), st, FA));
        prof_close(P, ph, PK_FRONTF, nb * L * e, nb * 5.0 * L * 12.0, st);
        CUDA_TRY(cudaGetLastError());
        return DGT_OK;
    }
    void* dst = P->pre ? P->finv : f;
    int rc = exec_fft(P, P->finv, dst, nb, CUFFT_INVERSE, st);
    if (rc) return rc;
    if (P->pre)
        k_conj_chirp<T><<<grid_for(nb * I.L), 256, 0, st>>>((C*)f, (const C*)P->finv, (const C*)P->pre, I.L, nb * I.L);
    prof_close(P, ph, PK_FRONT, nb * L * e, nb * 4.0 * L * std::log2(L), st);
    CUDA_TRY(cudaGetLastError());
    return DGT_OK;
}

// Synthesis on the one-CTA path (tiny.cuh, tiny_adj_kernel): one CTA per signal.
template <typename T>
static int launch_tiny_adj(Plan* P, const void* c, void* f, int64_t W, cudaStream_t st) {
    const dgt_lattice_info& I = P->info;
    TinyArgs TA = P->tiny_args;
    TA.f = nullptr; TA.real_in = 0;
    TA.rdL = P->rd_L; TA.rdd = P->rd_d; TA.rdm = P->rd_m;
    TA.L = (int)I.L; TA.c = (int)I.c; TA.d = (int)I.d; TA.p = (int)I.p; TA.q = (int)I.q;
    TA.iM = (int)I.iM; TA.iN = (int)I.iN;
    TA.B = make_out_args(P, nullptr, nullptr);
    const double e = (double)P->esz, L = (double)I.L, MN = (double)I.M * (double)I.N;
    const double fl = W * ((I.branch == DGT_BRANCH_FREQ ? 4.0 * L * std::log2(L) : 0.0) + 8.0 * L * I.q / I.p +
                           4.0 * L * std::log2((double)I.d) + 4.0 * MN * std::log2((double)I.d) +
                           4.0 * MN * std::log2((double)I.iM) + 6.0 * MN);
    const int ph = prof_open(P, st);
    for (int64_t w0 = 0; w0 < W; w0 += 65535 * 1024) {
        const int64_t wc = std::min<int64_t>(65535 * 1024, W - w0);
        const void* cc = (const char*)c + (size_t)w0 * I.M * I.N * P->esz;
        void* fc = (char*)f + (size_t)w0 * I.L * P->esz;
        if (P->tiny == 2)
            CUDA_TRY(launch_pdl(tiny_adj_kernel<T, 240, 5, 8, 2, 3>, dim3((unsigned)wc), dim3(256), P->tiny_smem, st, TA,
                                cc, fc));
        else
            CUDA_TRY(launch_pdl(tiny_adj_kernel<T>, dim3((unsigned)wc), dim3(256), P->tiny_smem, st, TA, cc, fc));
    }
    prof_close(P, ph, PK_TINYADJ, W * (L + MN) * e + L * e, fl, st);
    CUDA_TRY(cudaGetLastError());
    return DGT_OK;
}

static int execute_inverse(Plan* P, const void* c, void* f, int64_t W, cudaStream_t st) {
    const dgt_lattice_info& I = P->info;
    if (P->tiny && !P->fast)
        return P->dtype == DGT_C64 ? launch_tiny_adj<float>(P, c, f, W, st) : launch_tiny_adj<double>(P, c, f, W, st);
    if (P->fast && !P->inv_generic) {
        // fused synthesis (fused7_adj.cuh) on the forward ring
        const int ph = prof_open(P, st);
        const int64_t chunk = fast_chunk(&P->fp);
        for (int64_t w0 = 0; w0 < W; w0 += chunk) {
            const int64_t wc = std::min<int64_t>(chunk, W - w0);
            int rc = launch_fast_adj(&P->fp, (const char*)c + (size_t)w0 * I.M * I.N * 8,
                                     P->Cws, (char*)f + (size_t)w0 * I.L * 8, wc, st);
            if (rc) return rc;
        }
        const double L = (double)I.L, MN = (double)I.M * (double)I.N;
        prof_close(P, ph, PK_FASTADJ, W * (L + MN) * 8.0 + L * 8.0,
                   W * (8.0 * L * I.q + 4.0 * L * std::log2((double)I.d) + 4.0 * MN * std::log2((double)I.d) +
                        4.0 * MN * std::log2((double)I.iM) + 6.0 * MN), st);
        CUDA_TRY(cudaGetLastError());
        return DGT_OK;
    }
    const bool freq = I.branch == DGT_BRANCH_FREQ;
    // frequency shear: spectra of a batch of ib signals (a multiple of the chunk, ~192 MB) are
    // collected and inverse-transformed by one batched cuFFT call
    const int64_t ib = freq ? P->ib : W;
    if (!P->Cinv || (freq && !P->finv)) return fail(DGT_EINVAL, "synthesis workspace missing (made at plan time)");
    for (int64_t b0 = 0; b0 < W; b0 += ib) {
        const int64_t nb = std::min<int64_t>(ib, W - b0);
        for (int64_t w0 = b0; w0 < b0 + nb; w0 += P->inv_chunk) {
            const int64_t wc = std::min<int64_t>(P->inv_chunk, b0 + nb - w0);
            const void* cc = (const char*)c + (size_t)w0 * I.M * I.N * P->esz;
            void* fc = (char*)f + (size_t)w0 * I.L * P->esz;
            void* sp = freq ? (void*)((char*)P->finv + (size_t)(w0 - b0) * I.L * P->esz) : nullptr;
            int rc = P->dtype == DGT_C64 ? launch_inverse_chunk<float>(P, cc, fc, wc, st, sp)
                                         : launch_inverse_chunk<double>(P, cc, fc, wc, st, sp);
            if (rc) return rc;
        }
        if (freq) {
            void* fb = (char*)f + (size_t)b0 * I.L * P->esz;
            int rc = P->dtype == DGT_C64 ? launch_inverse_tail<float>(P, fb, nb, st) : launch_inverse_tail<double>(P, fb, nb, st);
            if (rc) return rc;
        }
    }
    return DGT_OK;
}

static int execute(Plan* P, const void* f, void* c, int64_t W, cudaStream_t st);

static int execute_ola(Plan* P, const void* f, void* c, int64_t W, cudaStream_t st) {
    const dgt_lattice_info& I = P->info;
    Plan* Q = P->ola;
    const int64_t Lx = Q->info.L, Nx = Q->info.N, Nb = P->ola_Nb, nb = P->ola_Lb / I.a;
    const bool real_in = (P->flags & DGT_REAL_INPUT) != 0;
    const size_t ein = real_in ? P->esz / 2 : P->esz;
    for (int64_t w0 = 0; w0 < W; w0 += P->ola_Ws) {
        const int64_t ws = std::min<int64_t>(P->ola_Ws, W - w0);
        const char* fw = (const char*)f + (size_t)w0 * I.L * ein;
        const int64_t tx = ws * Nb * Lx;
        if (P->dtype == DGT_C64) {
            if (real_in) k_ola_split<float><<<grid_for(tx), 256, 0, st>>>((float*)P->ola_x, (const float*)fw, I.L, P->ola_Lb, Lx, Nb, tx);
            else k_ola_split<float2><<<grid_for(tx), 256, 0, st>>>((float2*)P->ola_x, (const float2*)fw, I.L, P->ola_Lb, Lx, Nb, tx);
        } else {
            if (real_in) k_ola_split<double><<<grid_for(tx), 256, 0, st>>>((double*)P->ola_x, (const double*)fw, I.L, P->ola_Lb, Lx, Nb, tx);
            else k_ola_split<double2><<<grid_for(tx), 256, 0, st>>>((double2*)P->ola_x, (const double2*)fw, I.L, P->ola_Lb, Lx, Nb, tx);
        }
        int rc = execute(Q, P->ola_x, P->ola_c, ws * Nb, st);
        if (rc) return rc;
        const int64_t tc = ws * I.M * I.N;
        char* cw = (char*)c + (size_t)w0 * I.M * I.N * P->esz;
        if (P->dtype == DGT_C64)
            k_ola_add<float><<<grid_for(tc), 256, 0, st>>>((float2*)cw, (const float2*)P->ola_c, I.M, I.N, Nx, nb, Nb,
                                                           P->ola_pmin, P->ola_pmax, tc);
        else
            k_ola_add<double><<<grid_for(tc), 256, 0, st>>>((double2*)cw, (const double2*)P->ola_c, I.M, I.N, Nx, nb, Nb,
                                                            P->ola_pmin, P->ola_pmax, tc);
        CUDA_TRY(cudaGetLastError());
    }
    return DGT_OK;
}

static int execute(Plan* P, const void* f, void* c, int64_t W, cudaStream_t st);

// multiwindow: per chunk of Wc signals, the lambda2 separable transforms into mw_d, then the
// phase / interleave kernel into c
static int execute_mw(Plan* P, const void* f, void* c, int64_t W, cudaStream_t st) {
    const dgt_lattice_info& I = P->info;
    const int64_t l2 = (int64_t)P->mw.size(), Nt = I.N / l2;
    const size_t ein = (P->flags & DGT_REAL_INPUT) ? P->esz / 2 : P->esz;
    for (int64_t w0 = 0; w0 < W; w0 += P->mw_Wc) {
        const int64_t wc = std::min<int64_t>(P->mw_Wc, W - w0);
        const char* fw = (const char*)f + (size_t)w0 * I.L * ein;
        for (int64_t m = 0; m < l2; ++m) {
            char* dm = (char*)P->mw_d + (size_t)m * P->mw_Wc * I.M * Nt * P->esz;
            int rc = execute(P->mw[m], fw, dm, wc, st);
            if (rc) return rc;
        }
        const int64_t tot = wc * I.M * I.N;
        char* cw = (char*)c + (size_t)w0 * I.M * I.N * P->esz;
        const int ph = prof_open(P, st);
        if (P->dtype == DGT_C64)
            k_mw_interleave<float><<<grid_for(tot), 256, 0, st>>>((float2*)cw, (const float2*)P->mw_d, P->mw_sig,
                                                                  P->mw_Wc, I.M, I.N, l2, l2 * I.a, I.L, tot);
        else
            k_mw_interleave<double><<<grid_for(tot), 256, 0, st>>>((double2*)cw, (const double2*)P->mw_d, P->mw_sig,
                                                                   P->mw_Wc, I.M, I.N, l2, l2 * I.a, I.L, tot);
        prof_close(P, ph, PK_MW, 2.0 * tot * P->esz, 6.0 * tot, st);
        CUDA_TRY(cudaGetLastError());
    }
    return DGT_OK;
}

// One CTA per signal, the whole transform in shared memory (tiny.cuh).
template <typename T>
static int launch_tiny(Plan* P, const void* f, void* c, int64_t W, cudaStream_t st) {
    const dgt_lattice_info& I = P->info;
    TinyArgs TA = P->tiny_args;   // table pointers into P->tiny_pack (build_tables)
    TA.f = f; TA.real_in = (P->flags & DGT_REAL_INPUT) ? 1 : 0;
    TA.rdL = P->rd_L; TA.rdd = P->rd_d; TA.rdm = P->rd_m;
    TA.L = (int)I.L; TA.c = (int)I.c; TA.d = (int)I.d; TA.p = (int)I.p; TA.q = (int)I.q;
    TA.iM = (int)I.iM; TA.iN = (int)I.iN;
    TA.B = make_out_args(P, nullptr, c);
    const double e = (double)P->esz, ein = (P->flags & DGT_REAL_INPUT) ? e / 2 : e;
    const double L = (double)I.L, MN = (double)I.M * (double)I.N;
    const double lg_d = std::log2((double)I.d), lg_m = std::log2((double)I.iM);
    const double fl = W * ((I.branch == DGT_BRANCH_FREQ ? 4.0 * L * std::log2(L) : 0.0) + 8.0 * L * I.q / I.p +
                           4.0 * L * lg_d + 4.0 * MN * lg_d + 4.0 * MN * lg_m + 6.0 * MN);
    const int ph = prof_open(P, st);
    for (int64_t w0 = 0; w0 < W; w0 += 65535 * 1024) {
        const int64_t wc = std::min<int64_t>(65535 * 1024, W - w0);
        TinyArgs Tw = TA;
        Tw.f = (const char*)f + (size_t)w0 * I.L * (size_t)ein;
        Tw.B.out = (char*)c + (size_t)w0 * I.M * I.N * P->esz;
        if (P->tiny == 2)
            CUDA_TRY(launch_pdl(tiny_kernel<T, 240, 5, 8, 2, 3>, dim3((unsigned)wc), dim3(256), P->tiny_smem, st, Tw));
        else
            CUDA_TRY(launch_pdl(tiny_kernel<T>, dim3((unsigned)wc), dim3(256), P->tiny_smem, st, Tw));
    }
    prof_close(P, ph, PK_TINY, W * (L * ein + MN * e) + L * e, fl, st);
    CUDA_TRY(cudaGetLastError());
    return DGT_OK;
}

static int execute(Plan* P, const void* f, void* c, int64_t W, cudaStream_t st) {
    const dgt_lattice_info& I = P->info;
    if (P->ola) return execute_ola(P, f, c, W, st);
    if (!P->mw.empty()) return execute_mw(P, f, c, W, st);
    if (P->tiny && !P->fast)
        return P->dtype == DGT_C64 ? launch_tiny<float>(P, f, c, W, st) : launch_tiny<double>(P, f, c, W, st);
    const size_t ein = (P->flags & DGT_REAL_INPUT) ? P->esz / 2 : P->esz;
    if (I.branch == DGT_BRANCH_FREQ && !P->fast) {
        // front batches of P->fb signals (a multiple of the chunk), then the chunks of each
        for (int64_t b0 = 0; b0 < W; b0 += P->fb) {
            const int64_t nb = std::min<int64_t>(P->fb, W - b0);
            const void* fb = (const char*)f + (size_t)b0 * I.L * ein;
            int rc = P->dtype == DGT_C64 ? launch_front<float>(P, fb, nb, st) : launch_front<double>(P, fb, nb, st);
            if (rc) return rc;
            for (int64_t w0 = b0; w0 < b0 + nb; w0 += P->chunk) {
                const int64_t wc = std::min<int64_t>(P->chunk, b0 + nb - w0);
                const void* sp = (const char*)P->fhat + (size_t)(w0 - b0) * I.L * P->esz;
                void* cc = (char*)c + (size_t)w0 * I.M * I.N * P->esz;
                rc = P->dtype == DGT_C64 ? launch_chunk<float>(P, nullptr, cc, wc, st, sp)
                                         : launch_chunk<double>(P, nullptr, cc, wc, st, sp);
                if (rc) return rc;
            }
        }
        return DGT_OK;
    }
    for (int64_t w0 = 0; w0 < W; w0 += P->chunk) {
        const int64_t wc = std::min<int64_t>(P->chunk, W - w0);
        const void* fc = (const char*)f + (size_t)w0 * I.L * ein;
        void* cc = (char*)c + (size_t)w0 * I.M * I.N * P->esz;
        int rc = P->dtype == DGT_C64 ? launch_chunk<float>(P, fc, cc, wc, st, nullptr)
                                     : launch_chunk<double>(P, fc, cc, wc, st, nullptr);
        if (rc) return rc;
    }
    return DGT_OK;
}

}  // namespace nsdgt

using namespace nsdgt;

namespace {
// NVTX range around every C-ABI entry point (SURVEY §5 tracing): header-only nvtx3, a no-op
// unless a tool (nsys, ncu --nvtx) is attached
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

extern "C" {

const char* dgt_version(void) { return "nsdgt 0.1 (sm_100a)"; }

const char* dgt_strerror(int status) {
    switch (status) {
        case DGT_OK: return "ok";
        case DGT_EINVAL: return "invalid argument";
        case DGT_ENUMERIC: return "the window does not generate a frame on this lattice";
        case DGT_EILLEGAL_LENGTH: return "illegal transform length (L must be a multiple of L_min)";
        case DGT_ECUDA: return "CUDA runtime error";
        case DGT_ECUFFT: return "cuFFT error";
        case DGT_ENOMEM: return "out of memory";
        case DGT_EUNSUPPORTED: return "unsupported inner transform size";
        default: return "unknown status";
    }
}

const char* dgt_last_error(void) { return g_last_error.c_str(); }
int64_t dgt_last_lmin(void) { return g_last_lmin; }

int dgt_lattice_plan(int64_t L, int64_t a, int64_t M, int64_t l1, int64_t l2, int flags, int force_shear,
                     int64_t s0, int64_t s1, dgt_lattice_info* out) {
    std::string err;
    if (!out) return fail(DGT_EINVAL, "null output");
    int rc = plan_lattice(L, a, M, l1, l2, flags, force_shear != 0, s0, s1, out, &err);
    if (rc == DGT_EILLEGAL_LENGTH) g_last_lmin = out->L_min;
    if (rc) return fail(rc, err);
    return DGT_OK;
}

static int alloc_host_staging(Plan* P);

// The plan of dgt_plan; staging = make the host-buffer staging of dgt_execute_host (inner plans
// of the shear-OLA and multiwindow plans are only executed on device buffers and skip it).
static int make_plan(dgt_plan_t* out, int64_t L, int64_t a, int64_t M, int64_t l1, int64_t l2, const void* g, int dtype,
                     int flags, int64_t max_chunk, int force_shear, int64_t s0, int64_t s1, void* cuda_stream,
                     bool staging) {
    if (!out || !g) return fail(DGT_EINVAL, "null pointer");
    *out = nullptr;
    if (dtype != DGT_C64 && dtype != DGT_C128) return fail(DGT_EINVAL, "bad dtype");
    if (flags & ~(DGT_REAL_INPUT | DGT_G_ON_HOST | DGT_SHEAR_PAPER | DGT_FORCE_GENERIC))
        return fail(DGT_EINVAL, "bad flags");
    if (max_chunk < 0) return fail(DGT_EINVAL, "max_chunk < 0");
    Plan* P = new Plan();
    std::string err;
    int rc = plan_lattice(L, a, M, l1, l2, flags, force_shear != 0, s0, s1, &P->info, &err);
    if (rc) {
        if (rc == DGT_EILLEGAL_LENGTH) g_last_lmin = P->info.L_min;
        delete P;
        return fail(rc, err);
    }
    P->dtype = dtype;
    P->flags = flags;
    P->esz = dtype == DGT_C64 ? 8 : 16;
    cudaStream_t st = (cudaStream_t)cuda_stream;
    cudaGetDevice(&P->device);
    rc = dtype == DGT_C64 ? configure<float>(P, max_chunk) : configure<double>(P, max_chunk);
    if (!rc) rc = dtype == DGT_C64 ? build_tables<float>(P, g, (flags & DGT_G_ON_HOST) != 0, st)
                                   : build_tables<double>(P, g, (flags & DGT_G_ON_HOST) != 0, st);
    if (!rc && P->fast) {
        P->chunk = max_chunk > 0 ? max_chunk : fast_chunk(&P->fp);
    }
    if (!rc) rc = alloc_workspace(P, P->chunk);
    if (!rc && staging) rc = alloc_host_staging(P);
    if (rc) {
        free_plan(P);
        return rc;
    }
    P->info.chunk = P->chunk;
    P->info.workspace_bytes = (int64_t)P->ws_bytes;
    // 2 fused persistent kernel, 4 config-4 front path (front_f4096 + zak_rr0), 8 one-CTA path
    P->info.kernel_path = P->fast ? P->fast : (P->tiny ? 8 : (P->front ? 4 : 0));
    *out = (dgt_plan_t)P;
    return DGT_OK;
}

int dgt_plan(dgt_plan_t* out, int64_t L, int64_t a, int64_t M, int64_t l1, int64_t l2, const void* g, int dtype,
             int flags, int64_t max_chunk, int force_shear, int64_t s0, int64_t s1, void* cuda_stream) {
    NvtxRange nvtx_range("dgt_plan");
    return make_plan(out, L, a, M, l1, l2, g, dtype, flags, max_chunk, force_shear, s0, s1, cuda_stream, true);
}

int dgt_plan_fir(dgt_plan_t* out, int64_t L, int64_t a, int64_t M, int64_t l1, int64_t l2, const void* g, int64_t Lg,
                 int64_t Lb, int dtype, int flags, void* cuda_stream) {
    NvtxRange nvtx_range("dgt_plan_fir");
    if (!out || !g) return fail(DGT_EINVAL, "null pointer");
    *out = nullptr;
    if (dtype != DGT_C64 && dtype != DGT_C128) return fail(DGT_EINVAL, "bad dtype");
    if (flags & ~(DGT_REAL_INPUT | DGT_G_ON_HOST | DGT_SHEAR_PAPER | DGT_FORCE_GENERIC))
        return fail(DGT_EINVAL, "bad flags");
    dgt_lattice_info info{};
    std::string err;
    int rc = plan_lattice(L, a, M, l1, l2, flags, false, 0, 0, &info, &err);
    if (rc) {
        if (rc == DGT_EILLEGAL_LENGTH) g_last_lmin = info.L_min;
        return fail(rc, err);
    }
    if (Lg < 1 || Lg > L) return fail(DGT_EINVAL, "window length Lg must be in [1, L]");
    const int64_t Lmin = info.L_min;
    const size_t esz = dtype == DGT_C64 ? 8 : 16;
    // the window on the host, FIR layout: entries [0, ceil(Lg/2)) are times 0.., the rest
    // times -floor(Lg/2)..-1
    std::vector<unsigned char> gh(esz * Lg);
    if (flags & DGT_G_ON_HOST) std::memcpy(gh.data(), g, esz * Lg);
    else CUDA_TRY(cudaMemcpy(gh.data(), g, esz * Lg, cudaMemcpyDeviceToHost));
    const int64_t hr = (Lg + 1) / 2, hl = Lg / 2;   // times [-hl, hr)
    // automatic block length (throughput): the smallest multiple of L_min dividing L that is
    // >= max(16 Lg, 2^18) -- overhead rho = (Lg + Lb)/Lb <= 1.07 and blocks long enough to fill
    // the GPU (measured: Lb = 2^18 5.5 ms against 11.4 ms at Lb = 4 Lg, L = 2^22, Lg = 1024);
    // else the whole signal.  Streaming callers pass a short Lb for a short delay.
    if (Lb == 0) {
        Lb = L;
        const int64_t want = std::max<int64_t>(16 * Lg, (int64_t)1 << 18);
        for (int64_t k = 1; k * Lmin <= L; ++k)
            if (L % (k * Lmin) == 0 && k * Lmin >= want) { Lb = k * Lmin; break; }
    }
    if (Lb <= 0 || Lb % Lmin || L % Lb) return fail(DGT_EINVAL, "Lb must be a multiple of L_min dividing L");
    // Lx: the smallest multiple of L_min >= Lb + Lg + 2a whose quotient by L_min is 7-smooth
    // (the inner DFT lengths d and M' then factor into the register radices; a large prime
    // factor would take the O(R^2) generic butterfly)
    auto smooth = [](int64_t v) {
        for (int64_t pr : {2, 3, 5, 7})
            while (v % pr == 0) v /= pr;
        return v == 1;
    };
    int64_t kx = (Lb + Lg + 2 * a + Lmin - 1) / Lmin;
    while (!smooth(kx)) ++kx;
    const int64_t Lx = kx * Lmin;
    const bool blocks = Lx < L;
    const int64_t Lin = blocks ? Lx : L;
    // the window zero-extended to the inner length
    std::vector<unsigned char> gx(esz * Lin, 0);
    for (int64_t i = 0; i < Lg; ++i) {
        const int64_t t = i < hr ? i : i - Lg;             // time of entry i
        const int64_t x = ((t % Lin) + Lin) % Lin;
        std::memcpy(gx.data() + esz * x, gh.data() + esz * i, esz);
    }
    dgt_plan_t inner = nullptr;
    rc = make_plan(&inner, Lin, a, M, l1, l2, gx.data(), dtype, (flags & ~DGT_G_ON_HOST) | DGT_G_ON_HOST, 0, 0, 0, 0,
                   cuda_stream, !(Lx < L));
    if (rc) return rc;
    if (!blocks) {   // the blocks would be as long as the signal: the full-length plan
        *out = inner;
        return DGT_OK;
    }
    Plan* P = new Plan();
    P->info = info;
    P->dtype = dtype;
    P->flags = flags & ~DGT_G_ON_HOST;
    P->esz = esz;
    cudaGetDevice(&P->device);
    P->ola = (Plan*)inner;
    P->ola_Lb = Lb;
    P->ola_Nb = L / Lb;
    // local positions p with nonzero coefficients: a p + hr - 1 >= 0 and a p - hl <= Lb - 1
    P->ola_pmin = -((hr - 1) / a);
    P->ola_pmax = (Lb - 1 + hl) / a;
    // signals per group: the block buffers stay below ~1 GiB
    const size_t ein = (flags & DGT_REAL_INPUT) ? esz / 2 : esz;
    const size_t per_sig = (size_t)P->ola_Nb * ((size_t)Lx * ein + (size_t)M * (Lx / a) * esz);
    P->ola_Ws = std::max<int64_t>(1, (int64_t)((1ull << 30) / per_sig));
    if (cudaMalloc(&P->ola_x, (size_t)P->ola_Ws * P->ola_Nb * Lx * ein) != cudaSuccess ||
        cudaMalloc(&P->ola_c, (size_t)P->ola_Ws * P->ola_Nb * M * (Lx / a) * esz) != cudaSuccess) {
        free_plan(P);
        return fail(DGT_ENOMEM, "shear-OLA block buffers");
    }
    P->chunk = P->ola_Ws;
    P->info.chunk = P->ola_Ws;
    P->info.workspace_bytes = (int64_t)(P->ola_Ws * per_sig) + P->ola->info.workspace_bytes;
    P->info.kernel_path = 16 + P->ola->info.kernel_path;   // 16 + inner path: shear-OLA
    if (int rs = alloc_host_staging(P)) {
        free_plan(P);
        return rs;
    }
    *out = (dgt_plan_t)P;
    return DGT_OK;
}

int dgt_plan_multiwindow(dgt_plan_t* out, int64_t L, int64_t a, int64_t M, int64_t l1, int64_t l2, const void* g,
                         int dtype, int flags, void* cuda_stream) {
    NvtxRange nvtx_range("dgt_plan_multiwindow");
    if (!out || !g) return fail(DGT_EINVAL, "null pointer");
    *out = nullptr;
    if (dtype != DGT_C64 && dtype != DGT_C128) return fail(DGT_EINVAL, "bad dtype");
    if (flags & ~(DGT_REAL_INPUT | DGT_G_ON_HOST | DGT_FORCE_GENERIC)) return fail(DGT_EINVAL, "bad flags");
    dgt_lattice_info info{};
    std::string err;
    int rc = plan_lattice(L, a, M, l1, l2, flags, false, 0, 0, &info, &err);
    if (rc) {
        if (rc == DGT_EILLEGAL_LENGTH) g_last_lmin = info.L_min;
        return fail(rc, err);
    }
    const size_t esz = dtype == DGT_C64 ? 8 : 16;
    const int64_t lam2 = info.lambda2, b = info.b, s = info.s, Nt = info.N / lam2;
    // the window in fp64 on the host
    std::vector<double2> gh(L);
    {
        std::vector<unsigned char> raw(esz * L);
        if (flags & DGT_G_ON_HOST) std::memcpy(raw.data(), g, esz * L);
        else CUDA_TRY(cudaMemcpy(raw.data(), g, esz * L, cudaMemcpyDeviceToHost));
        for (int64_t l = 0; l < L; ++l) {
            if (dtype == DGT_C64) {
                const float2 v = ((const float2*)raw.data())[l];
                gh[l] = make_double2(v.x, v.y);
            } else {
                gh[l] = ((const double2*)raw.data())[l];
            }
        }
    }
    Plan* P = new Plan();
    P->info = info;
    P->dtype = dtype;
    P->flags = flags & ~DGT_G_ON_HOST;
    P->esz = esz;
    cudaGetDevice(&P->device);
    // chunk: the coefficient buffer of the lambda2 inner transforms stays near 256 MB
    P->mw_Wc = std::max<int64_t>(1, std::min<int64_t>(kMaxChunk, (int64_t)((256ull << 20) / ((size_t)M * info.N * esz))));
    std::vector<int64_t> sig(lam2);
    std::vector<unsigned char> gm(esz * L);
    for (int64_t m = 0; m < lam2; ++m) {
        // g_m = M_{sigma_m} T_{m a} g, sigma_m = m s mod b (Prop. mwindec / Eq. mw_phases):
        // g_m(l) = exp(2 pi i (sigma_m l mod L) / L) g((l - m a) mod L), exact integer phase index
        sig[m] = (m * s) % b;
        for (int64_t l = 0; l < L; ++l) {
            const int64_t r = (int64_t)(((__int128)sig[m] * l) % L);
            const long double th = 2.0L * 3.141592653589793238462643383279502884L * (long double)r / (long double)L;
            const double c0 = (double)cosl(th), s0 = (double)sinl(th);
            const double2 v = gh[(((l - m * a) % L) + L) % L];
            const double re = v.x * c0 - v.y * s0, im = v.x * s0 + v.y * c0;
            if (dtype == DGT_C64) ((float2*)gm.data())[l] = make_float2((float)re, (float)im);
            else ((double2*)gm.data())[l] = make_double2(re, im);
        }
        dgt_plan_t inner = nullptr;
        rc = make_plan(&inner, L, lam2 * a, M, 0, 1, gm.data(), dtype, (flags & ~DGT_G_ON_HOST) | DGT_G_ON_HOST,
                       P->mw_Wc, 0, 0, 0, cuda_stream, false);
        if (rc) {
            free_plan(P);
            return rc;
        }
        P->mw.push_back((Plan*)inner);
    }
    if (cudaMalloc(&P->mw_d, (size_t)lam2 * P->mw_Wc * M * Nt * esz) != cudaSuccess ||
        cudaMalloc(&P->mw_sig, sizeof(int64_t) * lam2) != cudaSuccess ||
        cudaMemcpy(P->mw_sig, sig.data(), sizeof(int64_t) * lam2, cudaMemcpyHostToDevice) != cudaSuccess) {
        free_plan(P);
        return fail(DGT_ENOMEM, "multiwindow buffers");
    }
    P->chunk = P->mw_Wc;
    P->info.chunk = P->mw_Wc;
    int64_t ws = (int64_t)lam2 * P->mw_Wc * M * Nt * (int64_t)esz;
    for (Plan* Q : P->mw) ws += Q->info.workspace_bytes;
    P->info.workspace_bytes = ws;
    P->info.kernel_path = 32 + P->mw[0]->info.kernel_path;   // 32 + inner path: multiwindow
    if (int rs = alloc_host_staging(P)) {
        free_plan(P);
        return rs;
    }
    *out = (dgt_plan_t)P;
    return DGT_OK;
}

int dgt_execute(dgt_plan_t plan, const void* f, void* c, int64_t W, void* cuda_stream) {
    NvtxRange nvtx_range("dgt_execute");
    Plan* P = (Plan*)plan;
    if (!P) return fail(DGT_EINVAL, "null plan");
    if (W < 0) return fail(DGT_EINVAL, "W < 0");
    if (W == 0) return DGT_OK;
    if (!f || !c) return fail(DGT_EINVAL, "null pointer");
    const size_t ein = (P->flags & DGT_REAL_INPUT) ? P->esz / 2 : P->esz;
    const char* fb = (const char*)f;
    const char* cb = (const char*)c;
    const size_t fbytes = (size_t)W * P->info.L * ein, cbytes = (size_t)W * P->info.M * P->info.N * P->esz;
    if (fb < cb + cbytes && cb < fb + fbytes) return fail(DGT_EINVAL, "f and c alias");
    return execute(P, f, c, W, (cudaStream_t)cuda_stream);
}

int dgt_execute_inverse(dgt_plan_t plan, const void* c, void* f, int64_t W, void* cuda_stream) {
    NvtxRange nvtx_range("dgt_execute_inverse");
    Plan* P = (Plan*)plan;
    if (!P) return fail(DGT_EINVAL, "null plan");
    if (P->ola) return fail(DGT_EUNSUPPORTED, "synthesis is not implemented for shear-OLA plans");
    if (!P->mw.empty()) return fail(DGT_EUNSUPPORTED, "synthesis is not implemented for multiwindow plans");
    if (W < 0) return fail(DGT_EINVAL, "W < 0");
    if (W == 0) return DGT_OK;
    if (!f || !c) return fail(DGT_EINVAL, "null pointer");
    const char* fb = (const char*)f;
    const char* cb = (const char*)c;
    const size_t fbytes = (size_t)W * P->info.L * P->esz, cbytes = (size_t)W * P->info.M * P->info.N * P->esz;
    if (fb < cb + cbytes && cb < fb + fbytes) return fail(DGT_EINVAL, "f and c alias");
    return execute_inverse(P, c, f, W, (cudaStream_t)cuda_stream);
}

int dgt_window_dual(dgt_plan_t plan, int kind, void* out, int flags, void* cuda_stream) {
    NvtxRange nvtx_range("dgt_window_dual");
    Plan* P = (Plan*)plan;
    if (!P || !out) return fail(DGT_EINVAL, "null pointer");
    if (P->ola) return fail(DGT_EUNSUPPORTED, "dual windows are not implemented for shear-OLA plans");
    if (!P->mw.empty()) return fail(DGT_EUNSUPPORTED, "dual windows are not implemented for multiwindow plans");
    if (kind != 0 && kind != 1) return fail(DGT_EINVAL, "kind must be 0 (dual) or 1 (tight)");
    if (flags & ~DGT_G_ON_HOST) return fail(DGT_EINVAL, "bad flags");
    const dgt_lattice_info& I = P->info;
    if (I.p > kDualPMax || I.q > kDualQMax) return fail(DGT_EUNSUPPORTED, "p or q too large for the dual kernel");
    if (kind == 1 && I.p > 2) return fail(DGT_EUNSUPPORTED, "tight window implemented for p <= 2");
    cudaStream_t st = (cudaStream_t)cuda_stream;
    const int64_t L = I.L;
    double2 *G64 = nullptr, *Gd = nullptr, *buf = nullptr;
    int* status = nullptr;
    int rc = DGT_OK;
    auto cleanup = [&]() {
        cudaFree(G64); cudaFree(Gd); cudaFree(buf); cudaFree(status);
    };
    if (cudaMalloc(&G64, sizeof(double2) * L) != cudaSuccess || cudaMalloc(&Gd, sizeof(double2) * L) != cudaSuccess ||
        cudaMalloc(&buf, sizeof(double2) * L) != cudaSuccess || cudaMalloc(&status, sizeof(int)) != cudaSuccess) {
        cleanup();
        return fail(DGT_ENOMEM, "dual window workspace");
    }
    cudaMemsetAsync(status, 0, sizeof(int), st);
    k_window_factor<double><<<grid_for(L), 256, 0, st>>>(G64, P->gt64, L, I.c, I.d, I.p, I.q);
    const double scale = kind == 0 ? 1.0 / (double)I.iM : 1.0 / std::sqrt((double)I.iM);
    k_dual_factor<<<grid_for(I.c * I.d, 64), 64, 0, st>>>(Gd, G64, I.c, I.d, (int)I.p, (int)I.q, scale, kind, status);
    const bool freq = I.branch == DGT_BRANCH_FREQ;
    // T: conj(P_{s1}) on the unfactored window; F: conj(P_{-s0}) before the inverse FFT
    k_dual_unfactor<<<grid_for(L), 256, 0, st>>>(buf, Gd, L, I.c, I.d, I.p, I.q, freq ? -I.s0 : I.s1);
    double2* res = buf;
    if (freq) {
        cufftHandle h;
        if (cufftPlan1d(&h, (int)L, CUFFT_Z2Z, 1) != CUFFT_SUCCESS) { cleanup(); return fail(DGT_ECUFFT, "dual window FFT plan"); }
        cufftSetStream(h, st);
        const cufftResult fr = cufftExecZ2Z(h, (cufftDoubleComplex*)buf, (cufftDoubleComplex*)G64, CUFFT_INVERSE);
        cudaStreamSynchronize(st);
        cufftDestroy(h);
        if (fr != CUFFT_SUCCESS) { cleanup(); return fail(DGT_ECUFFT, "dual window FFT"); }
        res = G64;
    }
    // cast (and the F-branch conj(P_{s1}) / L) into a device buffer of the plan's dtype
    void* dst = out;
    void* tmp = nullptr;
    if (flags & DGT_G_ON_HOST) {
        if (cudaMalloc(&tmp, P->esz * L) != cudaSuccess) { cleanup(); return fail(DGT_ENOMEM, "dual window output"); }
        dst = tmp;
    }
    const int64_t sig_fin = freq ? I.s1 : 0;
    // V = P_{-s0} F P_{s1} has V* V = L: the dual carries 1/L, the tight window 1/sqrt(L)
    const double sc_fin = freq ? (kind == 0 ? 1.0 / (double)L : 1.0 / std::sqrt((double)L)) : 1.0;
    if (P->dtype == DGT_C64) k_dual_finish<float><<<grid_for(L), 256, 0, st>>>((float2*)dst, res, L, sig_fin, sc_fin);
    else k_dual_finish<double><<<grid_for(L), 256, 0, st>>>((double2*)dst, res, L, sig_fin, sc_fin);
    int hstatus = 0;
    cudaError_t e = cudaMemcpyAsync(&hstatus, status, sizeof(int), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess && tmp) e = cudaMemcpyAsync(out, tmp, P->esz * L, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (tmp) cudaFree(tmp);
    cleanup();
    if (e != cudaSuccess) return fail(DGT_ECUDA, std::string("dual window: ") + cudaGetErrorString(e));
    if (hstatus) return fail(DGT_ENUMERIC, "the window does not generate a frame on this lattice (singular factor)");
    return rc;
}

// Host-buffer staging of dgt_execute_host, made at plan time: two copy streams, events and two
// slots of sw signals (~64 MB of output per slot, at most kMaxChunk signals, a multiple of the
// compute chunk when that is smaller; flat from 32 to 512 MB per slot on config 5: the two copy
// directions overlap each other and the kernels at the PCIe floor).
static int alloc_host_staging(Plan* P) {
    const dgt_lattice_info& I = P->info;
    const size_t ein = (P->flags & DGT_REAL_INPUT) ? P->esz / 2 : P->esz;
    const size_t per_f = (size_t)I.L * ein, per_c = (size_t)I.M * I.N * P->esz;
    int64_t sw = std::max<int64_t>(1, std::min<int64_t>(kMaxChunk, (int64_t)((64ull << 20) / per_c)));
    if (P->chunk < sw) sw = sw / P->chunk * P->chunk;
    CUDA_TRY(cudaStreamCreateWithFlags(&P->s_in, cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamCreateWithFlags(&P->s_out, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
        CUDA_TRY(cudaEventCreateWithFlags(&P->ev_in[i], cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&P->ev_comp[i], cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&P->ev_out[i], cudaEventDisableTiming));
        CUDA_TRY(cudaMalloc(&P->stage_f[i], per_f * sw));
        CUDA_TRY(cudaMalloc(&P->stage_c[i], per_c * sw));
    }
    P->stage_W = sw;
    P->ws_bytes += 2 * (per_f + per_c) * sw;
    return DGT_OK;
}

int dgt_execute_host(dgt_plan_t plan, const void* f_host, void* c_host, int64_t W, void* cuda_stream) {
    NvtxRange nvtx_range("dgt_execute_host");
    Plan* P = (Plan*)plan;
    if (!P) return fail(DGT_EINVAL, "null plan");
    if (W < 0) return fail(DGT_EINVAL, "W < 0");
    if (W == 0) return DGT_OK;
    if (!f_host || !c_host) return fail(DGT_EINVAL, "null pointer");
    if (!P->s_in || P->stage_W < 1) return fail(DGT_EINVAL, "host staging missing (made at plan time)");
    cudaStream_t st = (cudaStream_t)cuda_stream;
    const dgt_lattice_info& I = P->info;
    const size_t ein = (P->flags & DGT_REAL_INPUT) ? P->esz / 2 : P->esz;
    const size_t per_f = (size_t)I.L * ein, per_c = (size_t)I.M * I.N * P->esz;
    const int64_t sw = std::min<int64_t>(P->stage_W, W);
    // Once a copy is enqueued, every return waits for the three streams first: the caller may
    // free or reuse its host buffers as soon as this returns, even on an error.
    bool started = false;
    auto drain = [&](int rc) {
        if (started) {
            cudaStreamSynchronize(P->s_in);
            cudaStreamSynchronize(P->s_out);
            cudaStreamSynchronize(st);
        }
        return rc;
    };
#define HOST_TRY(x)                                                                  \
    do {                                                                             \
        cudaError_t e_ = (x);                                                        \
        if (e_ != cudaSuccess) return drain(fail(DGT_ECUDA, cudaGetErrorString(e_))); \
    } while (0)
    // the caller's stream must be ordered before our copies start
    HOST_TRY(cudaEventRecord(P->ev_out[0], st));
    HOST_TRY(cudaStreamWaitEvent(P->s_in, P->ev_out[0], 0));
    HOST_TRY(cudaEventRecord(P->ev_out[1], st));
    int64_t i = 0;
    for (int64_t w0 = 0; w0 < W; w0 += sw, ++i) {
        const int slot = (int)(i & 1);
        const int64_t wc = std::min<int64_t>(sw, W - w0);
        HOST_TRY(cudaStreamWaitEvent(P->s_in, P->ev_out[slot], 0));
        started = true;
        HOST_TRY(cudaMemcpyAsync(P->stage_f[slot], (const char*)f_host + w0 * per_f, wc * per_f,
                                 cudaMemcpyHostToDevice, P->s_in));
        HOST_TRY(cudaEventRecord(P->ev_in[slot], P->s_in));
        HOST_TRY(cudaStreamWaitEvent(st, P->ev_in[slot], 0));
        int rc = execute(P, P->stage_f[slot], P->stage_c[slot], wc, st);
        if (rc) return drain(rc);
        HOST_TRY(cudaEventRecord(P->ev_comp[slot], st));
        HOST_TRY(cudaStreamWaitEvent(P->s_out, P->ev_comp[slot], 0));
        HOST_TRY(cudaMemcpyAsync((char*)c_host + w0 * per_c, P->stage_c[slot], wc * per_c, cudaMemcpyDeviceToHost,
                                 P->s_out));
        HOST_TRY(cudaEventRecord(P->ev_out[slot], P->s_out));
    }
#undef HOST_TRY
    const cudaError_t e1 = cudaStreamSynchronize(P->s_out), e2 = cudaStreamSynchronize(st);
    cudaStreamSynchronize(P->s_in);
    if (e1 != cudaSuccess || e2 != cudaSuccess) return fail(DGT_ECUDA, cudaGetErrorString(e1 != cudaSuccess ? e1 : e2));
    return DGT_OK;
}

int dgt_destroy(dgt_plan_t plan) {
    free_plan((Plan*)plan);
    return DGT_OK;
}

int dgt_plan_query(dgt_plan_t plan, dgt_lattice_info* info) {
    if (!plan || !info) return fail(DGT_EINVAL, "null pointer");
    *info = ((Plan*)plan)->info;
    return DGT_OK;
}

int dgt_profile_begin(dgt_plan_t plan) {
    Plan* P = (Plan*)plan;
    if (!P) return fail(DGT_EINVAL, "null plan");
    P->prof = true;
    P->recs.clear();
    P->pool_used = 0;
    return DGT_OK;
}

int dgt_profile_end(dgt_plan_t plan, dgt_kernel_stat* stats, int max_stats, int* n_stats) {
    Plan* P = (Plan*)plan;
    if (!P || (!stats && max_stats > 0) || !n_stats) return fail(DGT_EINVAL, "null pointer");
    P->prof = false;
    dgt_kernel_stat acc[PK_COUNT];
    std::memset(acc, 0, sizeof acc);
    for (auto& r : P->recs) {
        CUDA_TRY(cudaEventSynchronize(r.b));
        float ms = 0.f;
        CUDA_TRY(cudaEventElapsedTime(&ms, r.a, r.b));
        acc[r.kind].launches += 1;
        acc[r.kind].ms += ms;
        acc[r.kind].bytes += r.bytes;
        acc[r.kind].flops += r.flops;
    }
    int n = 0;
    for (int k = 0; k < PK_COUNT; ++k) {
        if (!acc[k].launches) continue;
        const char* nm = (k == PK_FAST) ? P->fp.name : kProfNames[k];
        std::snprintf(acc[k].name, sizeof acc[k].name, "%s", nm);
        if (n < max_stats) stats[n] = acc[k];
        ++n;
    }
    *n_stats = n;
    P->recs.clear();
    P->pool_used = 0;
    return DGT_OK;
}

// Debugging aid of -DNSDGT_TRACE builds (tools/v7trace.py; not part of include/nsdgt.h): the
// device buffer of fused7 phase stamps (8 CTAs x 4096 entries) when the plan was made with
// NSDGT_DBG & 16, else null.
void* dgt_debug_trace_log(dgt_plan_t plan) {
    Plan* P = (Plan*)plan;
    return P ? (void*)P->fp.tracelog : nullptr;
}

#ifdef NSDGT_KTRACE
int dgt_debug_ktrace(unsigned long long* out64) {   // experiment builds only
    return cudaMemcpyFromSymbol(out64, g_ktrace, sizeof(unsigned long long) * 64) == cudaSuccess ? 0 : 1;
}
#endif
#ifdef NSDGT_TINY_TRACE
int dgt_debug_tiny_trace(unsigned long long* out16) {   // experiment builds only
    return cudaMemcpyFromSymbol(out16, g_tiny_trace, sizeof(unsigned long long) * 16) == cudaSuccess ? 0 : 1;
}
#endif

int64_t dgt_launches_per_execute(dgt_plan_t plan, int64_t W) {
    Plan* P = (Plan*)plan;
    if (!P || W <= 0) return 0;
    if (P->ola) {   // per group of signals: split + the inner plan's launches + overlap-add
        int64_t n = 0;
        for (int64_t w0 = 0; w0 < W; w0 += P->ola_Ws)
            n += 2 + dgt_launches_per_execute((dgt_plan_t)P->ola, std::min<int64_t>(P->ola_Ws, W - w0) * P->ola_Nb);
        return n;
    }
    if (!P->mw.empty()) {   // per chunk: the lambda2 inner transforms + the interleave kernel
        int64_t n = 0;
        for (int64_t w0 = 0; w0 < W; w0 += P->mw_Wc) {
            const int64_t wc = std::min<int64_t>(P->mw_Wc, W - w0);
            for (Plan* Q : P->mw) n += dgt_launches_per_execute((dgt_plan_t)Q, wc);
            n += 1;
        }
        return n;
    }
    if (P->tiny && !P->fast) return (W + 65535 * 1024 - 1) / (65535 * 1024);
    const int64_t chunks = (W + P->chunk - 1) / P->chunk;
    const int64_t per = P->fast ? fast_launches_per_chunk(&P->fp) + 1 /* counter memset */ : 2;
    int64_t n = chunks * per;
    // F-branch: per front batch front_f4096, or the pre-chirp kernel when needed (the cuFFT
    // call's own kernels are library launches and not counted)
    if (P->info.branch == DGT_BRANCH_FREQ && !P->fast && (P->front || (P->flags & DGT_REAL_INPUT) || P->pre))
        n += (W + P->fb - 1) / P->fb;
    return n;
}

}  // extern "C"
