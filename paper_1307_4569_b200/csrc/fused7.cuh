// fused7.cuh -- the round-1 hot-path kernel for the time-shear / separable branch with
// p = 1, q = 4, d = M in {256, 512}, complex64 (BASELINE configs 3 and 5).  DESIGN.md §4.3.
//
// Notation (Alg. 1 of PAPER.md:852-873, factorisation PAPER.md:790-804):
// x = j + s M (j < M, s < D = d), j = r + c l, n = kappa + q n'.  With the chirp
// factorisation P_sigma(j + sM) = C(j) W_D^{-sh_j s} (R(s) == 1 is required here) and the
// Alg. 1 row rotation rot(n(tau)) = alpha_{l,u} - beta tau (mod M) for n(tau) = (l-u-q tau)
// mod N, the whole T-branch reduces to two batched D-point DFT passes per signal:
//
//   pass A, column j:  F_j(mu) = sum_s f(j + sM) W_D^{s mu}                      (Zak DFT)
//                      for u < q:  x_{j,u}(mu) = F_j((sigma_j - mu) mod D) G'_{j,u}(mu)
//                                  ws[j][kappa][n'] = DFT_D[x_{j,u}](n'),  kappa = (l-u) mod q
//   pass B, column n:  c[m][n] = E(n) sum_j ws[j][n mod q][n div q] W_M^{j m}
//
// sigma_j = (j beta - sh_j) mod D, and the plan-time table
//   G'_{j,u}(mu) = G_{r,u}((j beta - mu) mod D) C(j) W_D^{j alpha_{l,u}} W_D^{-mu e_{l,u}},
//   e_{l,u} = floor((l-u)/q),  G = conj(Gamma)/d  (the window factorisation)
// carries the window, the column chirp C(j), the Alg. 1 row rotation and the output
// index reversal, so ws is already rotated: pass B needs only E(n).  (Derivation:
// DESIGN.md §4.3; every identity is exact, the table is built in fp64.)
//
// Execution: one persistent launch, CTAs of 128 threads (3 per SM for D = 512, 5 for D = 256)
// pull jobs from a global queue.  A job = 8 consecutive columns j of one signal (1 Zak DFT + q product DFTs each),
// B job = 16 consecutive columns n (1 DFT over j each; one 128-byte ring line per row j).
// Dependencies (B(w) after all A(w); A(w) after all B(w - S) because it reuses ring slot
// w mod S) are per-slot monotone counters; every job a CTA waits on was dequeued earlier
// by a resident CTA, so the spin cannot deadlock.
//
// The D-point DFT of an 8-slot tile: D = 16 R1, index x = t + 16 k.  Lane (slot, t) holds
// x(t + 16k), k < R1, loaded straight from global memory (8 columns of a row are 64
// contiguous bytes); it runs a register DFT-R1 over k and multiplies W_D^{t m1}.  One
// shared-memory exchange (in rounds of 16 values of m1 to keep the buffer at 16 KB) gives
// each lane whole sequences over t; a register DFT-16 finishes X(m1 + R1 m2).  All complex
// arithmetic is packed FP32x2 (FADD2/FFMA2/FMUL2): one instruction per complex add, two
// per complex multiply.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "cplx.cuh"
#include "tma.cuh"

namespace nsdgt {
namespace v7 {

// TMA descriptors of the fused kernels' bulk input tiles (TMA variant): f as a 2-D array
// [W D rows][M columns] and the ring as [S M rows][Q D columns], 8-byte elements, boxes of
// 8 columns x 256 rows (64-byte rows of a 32 KB tile, two boxes per tile)
struct Maps {
    CUtensorMap f;
    CUtensorMap ws;
};

// ------------------------------------------------------------------------------------
// packed FP32x2 complex arithmetic
// ------------------------------------------------------------------------------------
typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float2 a) {
    u64 r;
    asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a.x), "f"(a.y));
    return r;
}
__device__ __forceinline__ float2 upk(u64 r) {
    float2 v;
    asm("mov.b64 {%0,%1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r));
    return v;
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) {
    u64 r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk(a)), "l"(pk(b)));
    return upk(r);
}
__device__ __forceinline__ float2 csub(float2 a, float2 b) {
    u64 r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk(a)), "l"(pk(b)));
    return upk(r);
}
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
    u64 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pk(a)), "l"(pk(b)), "l"(pk(c)));
    return upk(r);
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
    u64 r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk(a)), "l"(pk(b)));
    return upk(r);
}
// a + (-i) b
__device__ __forceinline__ float2 cadd_mi(float2 a, float2 b) { return fma2(make_float2(b.y, b.x), make_float2(1.f, -1.f), a); }
// a - (-i) b
__device__ __forceinline__ float2 csub_mi(float2 a, float2 b) { return fma2(make_float2(b.y, b.x), make_float2(-1.f, 1.f), a); }
// d * w  (FMUL2 + FFMA2)
__device__ __forceinline__ float2 cmw(float2 d, float2 w) {
    return fma2(make_float2(-d.y, d.x), make_float2(w.y, w.y), mul2(d, make_float2(w.x, w.x)));
}
// d * (-i)
__device__ __forceinline__ float2 cmi(float2 d) { return make_float2(d.y, -d.x); }

// W_32^k = exp(-2 pi i k / 32), k < 32
__device__ __forceinline__ float2 w32(int k) {
    constexpr float cs[8] = {1.0f, 0.98078528040323044913f, 0.92387953251128675613f, 0.83146961230254523708f,
                             0.70710678118654752440f, 0.55557023301960222474f, 0.38268343236508977173f,
                             0.19509032201612826785f};
    // cos(2 pi k/32) for k in [0,8] via symmetry
    const int q = k >> 3, r = k & 7;
    float c, s;  // cos, sin of 2 pi k / 32
    if (q == 0) { c = cs[r]; s = r ? cs[8 - r] : 0.f; }
    else if (q == 1) { c = r ? -cs[8 - r] : 0.f; s = cs[r]; }
    else if (q == 2) { c = -cs[r]; s = r ? -cs[8 - r] : 0.f; }
    else { c = r ? cs[8 - r] : 0.f; s = -cs[r]; }
    return make_float2(c, -s);
}

// ------------------------------------------------------------------------------------
// register DFTs (forward, natural order in and out; all indices compile-time)
// ------------------------------------------------------------------------------------
__device__ __forceinline__ void dft4(float2& v0, float2& v1, float2& v2, float2& v3) {
    const float2 t0 = cadd(v0, v2), t1 = csub(v0, v2), t2 = cadd(v1, v3), t3 = csub(v1, v3);
    v0 = cadd(t0, t2);
    v2 = csub(t0, t2);
    v1 = cadd_mi(t1, t3);
    v3 = csub_mi(t1, t3);
}

// X[k1 + 4 k2] = sum_{n1} W16^{n1 k1} W4^{n1 k2} sum_{n2} x[n1 + 4 n2] W4^{n2 k1}
__device__ __forceinline__ void dft16(float2* v) {
#pragma unroll
    for (int n1 = 0; n1 < 4; ++n1) dft4(v[n1], v[n1 + 4], v[n1 + 8], v[n1 + 12]);
    // v[n1 + 4 k1] *= W16^{n1 k1} = W32^{2 n1 k1}
    v[5] = cmw(v[5], w32(2));
    v[9] = cmw(v[9], w32(4));
    v[13] = cmw(v[13], w32(6));
    v[6] = cmw(v[6], w32(4));
    v[10] = cmi(v[10]);
    v[14] = cmw(v[14], w32(12));
    v[7] = cmw(v[7], w32(6));
    v[11] = cmw(v[11], w32(12));
    v[15] = cmw(v[15], w32(18));
    float2 y[16];
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) {
        float2 a0 = v[4 * k1], a1 = v[4 * k1 + 1], a2 = v[4 * k1 + 2], a3 = v[4 * k1 + 3];
        dft4(a0, a1, a2, a3);
        y[k1] = a0; y[k1 + 4] = a1; y[k1 + 8] = a2; y[k1 + 12] = a3;
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = y[i];
}

// radix-2 DIT: E = DFT16(even), O = DFT16(odd); X[k] = E + W32^k O, X[k+16] = E - W32^k O
__device__ __forceinline__ void dft32(float2* v) {
    float2 e[16], o[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) { e[i] = v[2 * i]; o[i] = v[2 * i + 1]; }
    dft16(e);
    dft16(o);
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        if (k == 0) { v[0] = cadd(e[0], o[0]); v[16] = csub(e[0], o[0]); }
        else if (k == 8) { v[8] = cadd_mi(e[8], o[8]); v[24] = csub_mi(e[8], o[8]); }
        else {
            const float2 t = cmw(o[k], w32(k));
            v[k] = cadd(e[k], t);
            v[k + 16] = csub(e[k], t);
        }
    }
}

template <int R> __device__ __forceinline__ void dftR(float2* v) {
    if constexpr (R == 16) dft16(v);
    else dft32(v);
}

// ------------------------------------------------------------------------------------
// kernel arguments and job queue
// ------------------------------------------------------------------------------------
struct Args {
    const float2* f;     // [W][L]
    float2* out;         // [W][M][N]
    float2* ws;          // [S][M][Q][D]
    const float4* Gp;    // G' [M][Q][R1/2][16] of float4 (pairs k, k+1)
    const float2* E;     // [N]
    int* ctr;            // [0] job queue, [1..S] doneA per slot, [1+S..2S] doneB per slot
    int W, N, c, Kmod, beta;
    int S, lag, nA, nB;
    int sig0;            // sigma_j = 0 for every column j (the plan checks): wrap-free F gathers
    unsigned long long* log;   // dbg & 16: per-CTA phase timestamps (CTAs < 8, 4096 entries each)
    int dbg;             // experiment knobs (0 in production; results are wrong with all but 16):
                         // 1 no dependency spin, 4 no global stores, 8 no DFT arithmetic,
                         // 16 phase trace (-DNSDGT_TRACE builds), 32 no G' loads (fused8 only),
                         // 64 no c stores, 128 no ring stores, 256 skip B jobs, 512 skip A jobs
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// completion signal: a release reduction (after a CTA barrier it orders every thread's earlier
// stores / discards of the job before the count, like CUTLASS's semaphore arrive) -- no full fence
__device__ __forceinline__ void signal_release(int* p) {
    asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(p) : "memory");
}
__device__ __forceinline__ void spin_until(const int* p, int target) {
    if (ld_acquire(p) >= target) return;
    while (ld_acquire(p) < target) __nanosleep(64);
}
__device__ __forceinline__ float2 ld_cs(const float2* p) { return __ldcs(p); }
// read-only streams that are used once per SM: keep them out of L1
__device__ __forceinline__ float4 ldg_na(const float4* p) {
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
    return r;
}
__device__ __forceinline__ float2 ldg_na2(const float2* p) {
    float2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f32 {%0,%1}, [%2];" : "=f"(r.x), "=f"(r.y) : "l"(p));
    return r;
}
// shared-memory 16-byte load the compiler may not hoist out of loops (the twiddle table is
// loop-invariant; hoisting it costs 32 registers)
__device__ __forceinline__ float4 lds128_nohoist(const float4* p) {
    float4 r;
    const unsigned a = (unsigned)__cvta_generic_to_shared(p);
    asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "r"(a));
    return r;
}
__device__ __forceinline__ float2 ld_cg(const float2* p) { return __ldcg(p); }

// job p -> (isA, w, idx): blocks g = 0, 1, ...: A(g) jobs (g < W) then B(g - lag) jobs (g >= lag).
// 32-bit arithmetic (the host checks W (nA + nB) < 2^31).
__device__ __forceinline__ bool decode(int p, int W, int lag, int nA, int nB, int* isA, int* w, int* idx) {
    const int lagE = lag < W ? lag : W;
    const int seg1 = lagE * nA, seg2 = (W - lagE) * (nA + nB), seg3 = lagE * nB;
    if (p < seg1) { *isA = 1; *w = p / nA; *idx = p - *w * nA; return true; }
    p -= seg1;
    if (p < seg2) {
        const int t = p / (nA + nB), r = p - t * (nA + nB);
        if (r < nA) { *isA = 1; *w = lagE + t; *idx = r; }
        else { *isA = 0; *w = t; *idx = r - nA; }
        return true;
    }
    p -= seg2;
    if (p < seg3) { const int t = p / nB; *isA = 0; *w = W - lagE + t; *idx = p - t * nB; return true; }
    return false;
}

template <int D>
struct Cfg {
    static constexpr int R1 = D / 16;            // stage-1 length (32 or 16)
    static constexpr int NR = R1 / 16;           // exchange rounds = stage-2 sequences per lane (2 or 1)
    static constexpr int Q = 4;
    static constexpr int NS = 8;                 // tile slots (columns or (column, u) pairs)
    static constexpr int NT = 16 * NS;           // 128 threads: 8 slots x 16 lanes
    static constexpr int ACOL = 8;               // columns j per A job (1 Zak tile + 4 product tiles)
    static constexpr int BT = 2;                 // 8-column tiles per B job (16 columns = one ring line)
    static constexpr int XS = 16 * 17 + 2;       // exchange slot stride (rows of 17, 2 mod 16 per slot)
    static constexpr int XR = NS * XS;           // one exchange round, complex (~17.5 KB)
    static constexpr int XE = XR;                // exchange buffer: one round (rounds take turns)
    static constexpr int FS = D + 2;             // F column stride
    static constexpr int FE = ACOL * FS;         // F buffer, complex
    static constexpr int TWS = R1 + 2;           // twiddle-table row stride (rows don't overlap banks)
    static constexpr int TW = 16 * TWS;          // twiddle table W_D^{t m}, t < 16, m < R1
    static constexpr size_t SMEM = (size_t)(XE + FE + TW) * 8;
};

// Exchange buffer (one round of 16 values m1' = m1 mod 16), 8-byte slots, padded instead of
// swizzled so that every access is a lane base plus a compile-time offset:
// slot(s, m1', t) = P(s)*XS + m1'*17 + t, XS = 274 = 2 (mod 16), P(s) = 4 (s & 1) + (s >> 1).
// Every half-warp access of the thread-role maps below hits 16 distinct bank pairs
// (tools/bank_check.py).
__device__ __forceinline__ int xslot(int s) { return (((s & 1) << 2) | (s >> 1)) * (16 * 17 + 2); }

// Stage 1 -> exchange -> stage 2 of an 8-slot D-point DFT tile (128 threads).  The rounds
// share one buffer (a double-buffered variant, 35 KB, measured slower: 3 CTAs x 70 KB leave
// too little L1); the caller puts a barrier between tiles.
//   in:  v[k] = x(t + 16 k) of slot s1, lane t
//   out: emit(r, y) for r < NR, y[m2] = X(16 r + oi + R1 m2) of slot os
// The writer applies the whole twiddle W_D^{t m1} (table row tw = W_D^{t *}, R1 entries).  Per round: write
// 16 values, barrier, read one sequence, barrier (the buffer holds one round).  before_sync
// runs after this thread's first-round writes, after_sync right after the first barrier
// (v is dead then unless NR = 2 -- the second-round values live in v[16..31]).
struct NoMid {
    __device__ void operator()() const {}
};
struct NoBar {
    __device__ void operator()(int) const {}
};
// bar_pre(r) / bar_post(r): every thread, right before / after the exchange barrier of round r
// SYNC0: the buffer X may still be read by the previous tile: a barrier goes right before the
// first-round writes -- after the stage-1 DFT and twiddles, so that warps whose inputs arrived
// early can compute while the others wait (measured neutral against a barrier before the call).
template <int D, bool SYNC0 = false, class Before, class After, class Emit, class Mark, class Mid = NoMid,
          class After0 = NoMid, class BarPre = NoBar, class BarPost = NoBar>
__device__ __forceinline__ void dft_tile(float2* v, const float2* tw, float2* X2, int s1, int t, int os, int oi,
                                         Before&& before_sync, After&& after_sync, Emit&& emit, int dbg, Mark&& mark,
                                         Mid&& mid = Mid(), After0&& after0 = After0(), BarPre&& bar_pre = BarPre(),
                                         BarPost&& bar_post = BarPost()) {
    constexpr int R1 = Cfg<D>::R1, NR = Cfg<D>::NR;
    mark(10);
    if (!(dbg & 8)) dftR<R1>(v);
    mark(11);
    const float4* tw4 = reinterpret_cast<const float4*>(tw);   // twiddle pairs (m, m + 1)
    float2* xw = X2 + xslot(s1) + t;                           // writer: + 17 m1' (+ round buffer)
    const float2* xr = X2 + xslot(os) + 17 * oi;               // reader: + t (+ round buffer)
    // Twiddles: each round's 8 pairs are loaded back to back (32 registers) and then used --
    // loading one pair per use exposed the shared-memory latency (config 5: 5.82 -> 5.63 ms).
    // With two rounds (D = 512) every value is twiddled in place before the first exchange
    // barrier, so the second round only stores (5.61 ms); with one round (D = 256) the
    // twiddles are applied as the values are stored (0.336 against 0.339 ms).
    if constexpr (NR > 1) {
#pragma unroll
        for (int r = 0; r < NR; ++r) {
            float4 w2s[8];
#pragma unroll
            for (int mp = 0; mp < 8; ++mp) w2s[mp] = lds128_nohoist(tw4 + ((16 * r) >> 1) + mp);
#pragma unroll
            for (int m = 0; m < 16; m += 2) {
                if (r || m) v[16 * r + m] = cmw(v[16 * r + m], make_float2(w2s[m >> 1].x, w2s[m >> 1].y));
                v[16 * r + m + 1] = cmw(v[16 * r + m + 1], make_float2(w2s[m >> 1].z, w2s[m >> 1].w));
            }
            asm volatile("" ::: "memory");
        }
    }
    if constexpr (SYNC0 && NR > 1) __syncthreads();
#pragma unroll
    for (int r = 0; r < NR; ++r) {
        if constexpr (NR > 1) {
#pragma unroll
            for (int m = 0; m < 16; ++m) xw[17 * m] = v[16 * r + m];
        } else {
            if constexpr (SYNC0) __syncthreads();
            float4 w2s[8];
#pragma unroll
            for (int mp = 0; mp < 8; ++mp) w2s[mp] = lds128_nohoist(tw4 + ((16 * r) >> 1) + mp);
#pragma unroll
            for (int m = 0; m < 16; m += 2) {
                const float4 w2 = w2s[m >> 1];
                xw[17 * m] = (r || m) ? cmw(v[16 * r + m], make_float2(w2.x, w2.y)) : v[16 * r];
                xw[17 * (m + 1)] = cmw(v[16 * r + m + 1], make_float2(w2.z, w2.w));
            }
            asm volatile("" ::: "memory");
        }
        if (r == 0) before_sync();
        bar_pre(r);
        mark(12);
        __syncthreads();
        bar_post(r);
        if (r == 0) mid();   // every thread's stage-1 inputs of this tile have been consumed
        mark(13);
        float2 y[16];
#pragma unroll
        for (int tt = 0; tt < 16; ++tt) y[tt] = xr[tt];
        if (r + 1 < NR) __syncthreads();   // round r + 1 reuses the buffer
        if (r == NR - 1) after_sync();
        else after0();   // (NR = 2) v[0..15] are dead: the first half of the next tile may load
        if (!(dbg & 8)) dft16(y);
        emit(r, y);
    }
    mark(14);
}

// The same tile with the exchange double-buffered: round k of the kernel (counted across
// tiles by xb, uniform over the CTA) uses buffer k mod 2.  A buffer's previous readers (two
// rounds back) finished before the barrier of the round in between, so a tile needs one
// barrier per round and none at tile boundaries.
template <int D, class Before, class After, class Emit, class Mid>
__device__ __forceinline__ void dft_tile_db(float2* v, const float2* tw, float2* X2, int& xb, int s1, int t, int os,
                                            int oi, Before&& before_sync, After&& after_sync, Emit&& emit, int dbg,
                                            Mid&& mid) {
    constexpr int R1 = Cfg<D>::R1, NR = Cfg<D>::NR;
    if (!(dbg & 8)) dftR<R1>(v);
    const float4* tw4 = reinterpret_cast<const float4*>(tw);
#pragma unroll
    for (int r = 0; r < NR; ++r) {
        float2* XB = X2 + xb * Cfg<D>::XR;
        xb ^= 1;
        float2* xw = XB + xslot(s1) + t;
        const float2* xr = XB + xslot(os) + 17 * oi;
#pragma unroll
        for (int m = 0; m < 16; m += 2) {
            const float4 w2 = lds128_nohoist(tw4 + ((16 * r + m) >> 1));
            const float2 a = (r || m) ? cmw(v[16 * r + m], make_float2(w2.x, w2.y)) : v[16 * r];
            const float2 b = cmw(v[16 * r + m + 1], make_float2(w2.z, w2.w));
            xw[17 * m] = a;
            xw[17 * (m + 1)] = b;
            if ((m & 7) == 6) asm volatile("" ::: "memory");
        }
        if (r == 0) before_sync();
        __syncthreads();
        if (r == 0) mid();
        float2 y[16];
#pragma unroll
        for (int tt = 0; tt < 16; ++tt) y[tt] = xr[tt];
        if (r == NR - 1) after_sync();
        if (!(dbg & 8)) dft16(y);
        emit(r, y);
    }
}

// FULLPF: the whole next tile's inputs are prefetched behind the current tile's stage 2
// (fits the 168-register budget of 3 CTAs/SM; with 4+ CTAs only the first half).
// EARLY (D = 512): the first half of the next tile's inputs is loaded after the first exchange
// round (its registers v[0..15] are dead then), the second half after the last round -- half
// a tile more time in flight than loading both halves at the end.
// CST: the B tiles' coefficients go to global memory by TMA stores: each exchange round's
// 8 columns x 256 rows are written (times E(n)) into one half of the F buffer -- idle in B
// jobs -- as a box [m div R1][m mod R1][column] and stored by one cp.async.bulk.tensor (16 KB)
// that thread 0 issues after the next barrier; before a half is rewritten thread 0 waits for
// the earlier stores' shared-memory reads.  Whole-box stores replace the per-thread 8-byte
// stores that touched 64 bytes of each of four lines per warp instruction.
template <int D, int MINB, bool FULLPF = (MINB <= 3), bool REAL = false, bool EARLY = false, bool CST = false>
__global__ void __launch_bounds__(128, MINB) fused7_kernel(Args A, const __grid_constant__ CUtensorMap cmap) {
    using K = Cfg<D>;
    constexpr int R1 = K::R1, Q = K::Q, M = D, AC = K::ACOL, BT = K::BT;
    constexpr int N = Q * D;       // N = L / a = q d here (the host checks)
    static_assert(!CST || (D == 512 && K::FE >= 2 * 2048), "F buffer holds two 16 KB store boxes (D = 512)");
    extern __shared__ __align__(128) unsigned char smem_tma[];
    float2* X2 = reinterpret_cast<float2*>(smem_tma);
    float2* F = X2 + K::XE;        // F[col * FS + nu], col < ACOL
    float2* twt = F + K::FE;       // twt[t][m] = W_D^{t m}
    __shared__ int jobsm[6];       // next job, 1 if its first tile's inputs were prefetched, its isA, w, idx, slot
    __shared__ int jobdec[6];      // decoded current job: isA (or -1 = done), w, idx, gen, slot
    const int tid = threadIdx.x;
    // thread-role maps (t = stage-1 lane, i = stage-2 lane):
    //   S1 / M1 (Zak tile, B tiles, stage 1 of product tiles): slot s8 = tid & 7, t / i = h8 = tid >> 3
    //   M3 (stage 2 of product tiles): warp w, lane L: slot 4 (w >> 1) + (L >> 3), i = (L & 7) + 8 (w & 1)
    const int s8 = tid & 7, h8 = tid >> 3;
    for (int e = tid; e < 16 * R1; e += K::NT) {
        const int tt = e / R1, m = e % R1;
        double sn, cs;
        sincospi(-2.0 * (double)((tt * m) % D) / (double)D, &sn, &cs);
        twt[tt * K::TWS + m] = make_float2((float)cs, (float)sn);
    }
    const float2* tw = twt + h8 * K::TWS;
#ifdef NSDGT_TRACE
    // phase trace (tools/v7trace.py): thread 0 of CTAs < 8 logs globaltimer stamps
    unsigned long long* lg = (A.dbg & 16) && blockIdx.x < 8 && tid == 0 ? A.log + (size_t)blockIdx.x * 4096 : nullptr;
    int nlog = 0;
    auto mark = [&](int code) {
        if (lg && nlog < 4095) lg[nlog++] = (gtimer() << 8) | (unsigned long long)code;
    };
#else
    auto mark = [](int) {};
#endif
    int* queue = A.ctr;
    int* doneA = A.ctr + 1;
    int* doneB = A.ctr + 1 + A.S;
    const int64_t MQD = (int64_t)M * Q * D;

    // ---- global inputs of a tile -> pre[], values k in [16 b, 16 b + 16) (halves keep a
    // cross-tile prefetch within the register budget) ----
    float2 pre[R1];
    auto load_f = [&](int w, int j0, int b) {   // Zak DFT input: column j0 + s8, rows t + 16 k
        if constexpr (REAL) {   // real samples (4-byte loads, 32 contiguous bytes per row of 8 columns)
            const float* fr = reinterpret_cast<const float*>(A.f) + (int64_t)w * M * D + j0 + s8;
#pragma unroll
            for (int k = 16 * b; k < 16 * b + 16 && k < R1; ++k) pre[k] = make_float2(__ldcs(fr + (int64_t)(h8 + 16 * k) * M), 0.f);
        } else {
            const float2* fw = A.f + (int64_t)w * M * D + j0 + s8;
#pragma unroll
#ifdef NSDGT_XP_NOFR   // experiment builds only: no f / ring loads (results wrong)
            for (int k = 16 * b; k < 16 * b + 16 && k < R1; ++k) pre[k] = make_float2((float)k, (float)(j0 + w));
#else
            for (int k = 16 * b; k < 16 * b + 16 && k < R1; ++k) pre[k] = ldg_na2(fw + (int64_t)(h8 + 16 * k) * M);
#endif
        }
    };
    // G' of product tile h (slot s8 = 4 col + u, lane t).  Layout [j0 / 8][h][kp][t][slot] of
    // float4 (k = 2 kp, 2 kp + 1): a warp reads 512 contiguous bytes.
    auto load_g = [&](int j0, int h, int b) {
        const float4* G4 = A.Gp + ((int64_t)((j0 / AC) * 4 + h) * (R1 / 2)) * 128 + h8 * 8 + s8;
#pragma unroll
        for (int kp = 8 * b; kp < 8 * b + 8 && kp < R1 / 2; ++kp) {
#ifdef NSDGT_XP_NOG   // experiment builds only: no G' loads
            const float4 g = make_float4((float)kp, 1.f, (float)h, 0.5f);
#else
            const float4 g = ldg_na(G4 + kp * 128);
#endif
            pre[2 * kp] = make_float2(g.x, g.y);
            pre[2 * kp + 1] = make_float2(g.z, g.w);
        }
    };
    // pass-B input: ring line (j, line) holds columns n = 16 line + p at position p; tile bt
    // reads positions 8 bt + s8
    auto load_ring = [&](int slot, int line, int bt, int b) {   // slot = w mod S
        const float2* src = A.ws + (int64_t)slot * MQD + (int64_t)h8 * (Q * D) + line * 16 + 8 * bt + s8;
#pragma unroll
#if defined(NSDGT_XP_NOFR) || defined(NSDGT_XP_NORING)   // experiment builds only: no ring loads
        for (int k = 16 * b; k < 16 * b + 16 && k < R1; ++k) pre[k] = make_float2((float)k, (float)(line + slot));
#else
        for (int k = 16 * b; k < 16 * b + 16 && k < R1; ++k) pre[k] = ld_cg(src + (int64_t)(16 * k) * (Q * D));
#endif
    };
    auto load_first = [&](int isA, int w, int idx, int slot, int b) {   // first tile of a job, half b
        if (isA) load_f(w, idx * AC, b);
        else load_ring(slot, idx, 0, b);
    };
    int pnext = -1;
    // Cross-job prefetch.  claim_ready (thread 0, before the last tile's exchange barrier)
    // publishes the next job and whether its inputs may be read now (A: always -- f is
    // read-only; B: its dependency already holds).  prefetch_next (every thread, after that
    // barrier, when pre[] is dead) loads the first half behind the tile's stage 2.
    // (thread 0 decodes the next job once and publishes it: the integer divisions of decode
    // stay out of the 128 threads' prefetch path)
    auto claim_ready = [&]() {
        int isA0, idx0, w0, ready = 0, slot0 = 0;
        if (decode(pnext, A.W, A.lag, A.nA, A.nB, &isA0, &w0, &idx0)) {
            const int gen0 = w0 / A.S;
            slot0 = w0 - gen0 * A.S;
            ready = isA0 || (A.dbg & 1) || ld_acquire(doneA + slot0) >= (gen0 + 1) * A.nA;
            jobsm[2] = isA0; jobsm[3] = w0; jobsm[4] = idx0; jobsm[5] = slot0;
        }
        jobsm[0] = pnext;
        jobsm[1] = ready;
    };
    auto prefetch_next = [&]() {
        if (jobsm[1]) {
            if (!EARLY) load_first(jobsm[2], jobsm[3], jobsm[4], jobsm[5], 0);
            if ((FULLPF || EARLY) && R1 > 16) load_first(jobsm[2], jobsm[3], jobsm[4], jobsm[5], 1);
        }
    };
    auto prefetch_next0 = [&]() {   // EARLY: the first half
        if (jobsm[1]) load_first(jobsm[2], jobsm[3], jobsm[4], jobsm[5], 0);
    };
    // Completion signals are deferred: thread 0 publishes "job done" (fence + counter add)
    // once it is into its next job's first tile, when the job's stores have drained and
    // the fence is cheap -- or before any spin, so it never waits on its own signal.  The
    // loop-top barrier orders every thread's stores (and L2 discards) before that fence.
    int* pend = nullptr;
    auto flush = [&]() {
        if (pend) {
            if (!(A.dbg & 4096)) signal_release(pend);   // (4096: experiment, no completion signals; needs 1)
            pend = nullptr;
        }
    };
    // CST (thread 0): the store box written by the last exchange round, issued after the next
    // barrier -- kept in shared memory (thread 0 alone uses it; registers are at the cap)
    __shared__ int cst_box[5];   // pending, half, x, y, z
    auto cst_issue = [&]() {
        if (CST && cst_box[0]) {
            tma::store_3d(&cmap, F + cst_box[1] * 2048, cst_box[2], cst_box[3], cst_box[4]);
            tma::bulk_commit();
            cst_box[0] = 0;
        }
    };
    if (tid == 0) {
        cst_box[0] = 0;
        if (CST && (tma::saddr(F) & 127)) __trap();   // TMA boxes are 128-byte aligned
        jobsm[0] = atomicAdd(queue, 1);
        jobsm[1] = 0;
    }
    __syncthreads();
    for (;;) {
        // thread 0 decodes the job claimed during the previous job, checks its dependency
        // (spinning if needed) and broadcasts it with the loop-top barrier, which also
        // orders the previous job's stores before its deferred completion signal
        const int pref = jobsm[1];
        if (tid == 0) {
            int isA0, idx0, w0;
            if (decode(jobsm[0], A.W, A.lag, A.nA, A.nB, &isA0, &w0, &idx0)) {
                const int gen0 = w0 / A.S;
                jobdec[0] = isA0; jobdec[1] = w0; jobdec[2] = idx0; jobdec[3] = gen0; jobdec[4] = w0 - gen0 * A.S;
            } else {
                jobdec[0] = -1;
            }
        }
        mark(1);
        __syncthreads();
        if (CST && tid == 0) cst_issue();   // the previous job's last box
        mark(3);
        const int isA = jobdec[0];
        if (isA < 0) break;
        const int w = jobdec[1], idx = jobdec[2];
        const int gen = jobdec[3], slot = jobdec[4];
        float2* wsl = A.ws + (int64_t)slot * MQD;
        if (tid == 0 && !(A.dbg & 1)) {
            const int* cnt = isA ? doneB + slot : (pref ? nullptr : doneA + slot);
            const int target = isA ? gen * A.nB : (gen + 1) * A.nA;   // A: slot free (B(w - S) done); B: all A(w) done
            if (cnt && ld_acquire(cnt) < target) {
                flush();
                spin_until(cnt, target);
            }
        }
        mark(4);
        // B inputs may be read only after the spin.  (A jobs: thread 0's spin precedes its
        // first exchange barrier, hence every ring store.)
        if ((isA && (A.dbg & 512)) || (!isA && (A.dbg & 256))) {   // experiment: skip this job kind
            if (tid == 0) {
                flush();
                pend = (isA ? doneA : doneB) + slot;
                pnext = atomicAdd(queue, 1);
                jobsm[0] = pnext;
                jobsm[1] = 0;
            }
            __syncthreads();
            continue;
        }
        if (!pref) {
            if (!isA) __syncthreads();
            load_first(isA, w, idx, slot, 0);
        }
        if (R1 > 16 && (!FULLPF || !pref)) load_first(isA, w, idx, slot, 1);
        mark(pref ? 6 : 5);
        if (isA) {
            // ---------------- pass A: columns j0 .. j0 + 7 ----------------
            const int j0 = idx * AC;
            // Zak DFT of 8 columns: F_j(nu), nu = 16 r + i + R1 m2, stored at F[col * FS + nu]
            dft_tile<D>(pre, tw, X2, s8, h8, s8, h8,
                        [&] {
                            if (tid == 0) {
                                flush();
                                if (CST) tma::bulk_wait_read0();   // F is rewritten below
                            }
                        },
                        [&] {
                            if (!EARLY) load_g(j0, 0, 0);
                            if ((FULLPF || EARLY) && R1 > 16) load_g(j0, 0, 1);
                        },
                        [&](int r, const float2* y) {
#pragma unroll
                            for (int m2 = 0; m2 < 16; ++m2) {
                                F[s8 * K::FS + 16 * r + h8 + R1 * m2] = y[m2];
                            }
                            // F(D) = F(0): the sigma = 0 gathers below read F(D - t - 16 k) without a wrap
                            if (r == 0 && h8 == 0) F[s8 * K::FS + D] = y[0];
                        }, A.dbg, mark, NoMid(),
                        [&] { if (EARLY) load_g(j0, 0, 0); });
            mark(20);
            __syncthreads();   // F complete; X free
            mark(21);
            // four product tiles: tile h = columns j0 + 2h, j0 + 2h + 1, slot s -> (col = s >> 2, u = s & 3)
            const int wq = tid >> 5, ln = tid & 31;
            const int colM = wq >> 1, uM = ln >> 3, iM = (ln & 7) + 8 * (wq & 1);   // role M3
            const int kap = (j0 / A.c - uM) & (Q - 1);   // kappa = (l - u) mod q: l is the job's (c % 8 == 0)
#pragma unroll 1
            for (int h = 0; h < 4; ++h) {
                const int fcol = 2 * h + (s8 >> 2);   // F column of this stage-1 slot
                const int jS = j0 + fcol;
                const int sig = (jS * (A.beta - A.Kmod)) & (D - 1);   // (j beta - K j) mod D, D a power of 2
                // the next job is claimed in the last tile: claiming it earlier (at this job's
                // start or one tile earlier) measured 50 % / 1.3 % slower -- the later claim
                // keeps B jobs behind their A jobs
                if (h == 3 && tid == 0) pnext = atomicAdd(queue, 1);
                // x(t + 16k) = F((sigma - t - 16k) mod D) G'(t + 16k); G' values k < 16 were
                // prefetched behind the previous tile, the rest are loaded now
                // F index (sigma - t - 16 k) mod D = (e0 - 16 k) mod D, e0 = (sigma - t) mod D: the
                // first (e0 >> 4) + 1 values need no wrap
                const float2* Fc = F + fcol * K::FS;
                if (A.sig0) {
                    // sigma_j = 0 for every column (configs 3 and 5): F((-t - 16 k) mod D) is
                    // F(D - t - 16 k) in [1, D] (F(D) duplicates F(0)): constant offsets
                    const float2* Fb = Fc + (D - h8);
#pragma unroll
                    for (int k = 0; k < 16; ++k) pre[k] = cmw(Fb[-16 * k], pre[k]);
                    if (R1 > 16) {
                        if (!FULLPF) {
                            asm volatile("" ::: "memory");
                            load_g(j0, h, 1);
                        }
#pragma unroll
                        for (int k = 16; k < R1; ++k) pre[k] = cmw(Fb[-16 * k], pre[k]);
                    }
                } else {
                    const int e0 = (sig - h8) & (D - 1);
#pragma unroll
                    for (int k = 0; k < 16; ++k) pre[k] = cmw(Fc[(e0 - 16 * k) & (D - 1)], pre[k]);
                    if (R1 > 16) {
                        if (!FULLPF) {
                            asm volatile("" ::: "memory");
                            load_g(j0, h, 1);
                        }
#pragma unroll
                        for (int k = 16; k < R1; ++k) pre[k] = cmw(Fc[(e0 - 16 * k) & (D - 1)], pre[k]);
                    }
                }
                mark(22);
                // (the barrier for the previous tile's readers of X is inside the tile: SYNC0)
                // ring layout ws[slot][j][n' >> 2][n' & 3][kappa]: one 128-byte line per
                // (j, n' >> 2), holding columns n = 4 n' + kappa in natural order.  A warp of
                // role M3 holds the 4 kappa of one column x 8 consecutive n': every store
                // fills 2 whole lines.
                const int jM = j0 + 2 * h + colM;
                // n' = 16 r + iM + R1 m2: line n' >> 2 = 4 r + (R1 / 4) m2 + (iM >> 2), position 4 (iM & 3) + kappa
                float2* dst = wsl + (int64_t)jM * (Q * D) + (iM >> 2) * 16 + (iM & 3) * 4 + kap;
                dft_tile<D, true>(pre, tw, X2, s8, h8, 4 * colM + uM, iM,
                            [&] { if (h == 3 && tid == 0) claim_ready(); },
                            [&] {
                                if (h < 3) {
                                    if (!EARLY) load_g(j0, h + 1, 0);
                                    if ((FULLPF || EARLY) && R1 > 16) load_g(j0, h + 1, 1);
                                } else {
                                    prefetch_next();
                                }
                            },
                            [&](int r, const float2* y) {
                                if (A.dbg & (4 | 128)) return;
#pragma unroll
                                for (int m2 = 0; m2 < 16; ++m2) dst[(4 * r + (R1 / 4) * m2) * 16] = y[m2];
                            }, A.dbg, mark, NoMid(),
                            [&] {
                                if (EARLY) {
                                    if (h < 3) load_g(j0, h + 1, 0);
                                    else prefetch_next0();
                                }
                            });
            }
            if (tid == 0) pend = doneA + slot;
        } else {
            // ---------------- pass B: columns 16 idx .. 16 idx + 15 (ring line idx) ----------------
#pragma unroll 1
            for (int bt = 0; bt < BT; ++bt) {
                if (bt == BT - 1 && tid == 0) pnext = atomicAdd(queue, 1);
                const int n = idx * 16 + 8 * bt + s8;
                const float2 e = ldg_na2(A.E + n);   // issued here (volatile), used at the emit
                float2* dst = A.out + (int64_t)w * M * N + n;
                if (bt && !FULLPF && R1 > 16) load_ring(slot, idx, bt, 1);   // second half (the first was prefetched)
                // (the barrier for the previous tile's readers of X is inside the tile: SYNC0)
                dft_tile<D, true>(pre, tw, X2, s8, h8, s8, h8,
                            [&] {
                                if (tid == 0) {
                                    flush();
                                    if (bt == BT - 1) claim_ready();
                                }
                            },
                            [&] {
                                if (bt + 1 < BT) {
                                    if (!EARLY) load_ring(slot, idx, bt + 1, 0);
                                    if ((FULLPF || EARLY) && R1 > 16) load_ring(slot, idx, bt + 1, 1);
                                } else {
                                    prefetch_next();
                                }
                            },
                            [&](int r, const float2* y) {
                                if constexpr (CST) {   // (D = 512: round r writes half r)
                                    float2* Fh = F + r * 2048;
#pragma unroll
                                    for (int m2 = 0; m2 < 16; ++m2) Fh[(m2 * 16 + h8) * 8 + s8] = cmw(y[m2], e);
                                    tma::fence_proxy_async_smem();
                                    if (tid == 0) {
                                        cst_box[0] = 1;
                                        cst_box[1] = r;
                                        cst_box[2] = idx * 16 + 8 * bt;
                                        cst_box[3] = 16 * r;
                                        cst_box[4] = w * (M / R1);
                                    }
                                } else {
                                    if (A.dbg & (4 | 64)) return;
#pragma unroll
                                    for (int m2 = 0; m2 < 16; ++m2) {
                                        const int m = 16 * r + h8 + R1 * m2;
                                        __stcs(dst + m * N, cmw(y[m2], e));
                                    }
                                }
                            }, A.dbg, mark, NoMid(),
                            [&] {
                                if (EARLY) {
                                    if (bt + 1 < BT) load_ring(slot, idx, bt + 1, 0);
                                    else prefetch_next0();
                                }
                            },
                            [&](int) {   // the half this round's emit writes is read by no store
                                if (CST && tid == 0) tma::bulk_wait_read0();
                            },
                            [&](int) {   // every thread's box of the previous round is written
                                if (CST && tid == 0) cst_issue();
                            });
            }
            // The ring lines this job read are dead (this job is their only reader; the
            // exchange barriers ordered every load before this point): drop them from L2 so
            // they are never written back to HBM.  Thread tid drops lines j = tid, tid + 128, ...
#pragma unroll
            for (int j = tid; j < M; j += K::NT)
                asm volatile("discard.global.L2 [%0], 128;" ::"l"(wsl + (int64_t)j * (Q * D) + idx * 16) : "memory");
            if (tid == 0) pend = doneB + slot;
        }
    }
    __syncthreads();   // the last job's stores are ordered before its completion signal
    if (tid == 0) {
        flush();
        if (CST) {
            cst_issue();
            tma::bulk_wait0();
        }
    }
}

// ------------------------------------------------------------------------------------
// fused7t: fused7 with the bulk input tiles (the Zak tile's f and the B tiles' ring lines,
// 32 KB each) brought into shared memory by the TMA engine instead of per-thread loads.
// The destination is the F buffer, which is idle exactly when those tiles are needed: an A
// job's f tile lands there and is overwritten by F after the Zak stage 1; a B job never uses
// F.  Thread 0 issues the copy of the next tile as soon as the current one's stage-1 inputs
// are consumed (the first exchange barrier) -- for the next job in the last tile, when it is
// ready -- so the tile loads need no registers and no L1 capacity, and arrive by an mbarrier
// (transaction bytes).  Everything else (G' register prefetch, exchange, ring, c stores,
// queue, counters) is fused7's.
// ------------------------------------------------------------------------------------
template <int D, int MINB, bool XDB = false, bool FULLPF = (MINB <= 3)>
__global__ void __launch_bounds__(128, MINB) fused7t_kernel(Args A, const __grid_constant__ Maps tm) {
    using K = Cfg<D>;
    constexpr int R1 = K::R1, Q = K::Q, M = D, AC = K::ACOL, BT = K::BT;
    constexpr int N = Q * D;
    constexpr uint32_t TILE_BYTES = (uint32_t)D * 8 * 8;   // 8 columns x D rows x 8 bytes
    static_assert(K::FE * 8 >= (int)TILE_BYTES, "F buffer holds one input tile");
    static_assert((K::XE * 8) % 128 == 0, "TMA destination alignment");
    extern __shared__ __align__(128) unsigned char smem_tma[];
    float2* X2 = reinterpret_cast<float2*>(smem_tma);
    float2* F = X2 + K::XE * (XDB ? 2 : 1);
    float2* twt = F + K::FE;
    __shared__ int jobsm[2];
    __shared__ int jobdec[4];
    __shared__ __align__(8) uint64_t mbar;
    const int tid = threadIdx.x;
    const int s8 = tid & 7, h8 = tid >> 3;
    for (int e = tid; e < 16 * R1; e += K::NT) {
        const int tt = e / R1, m = e % R1;
        double sn, cs;
        sincospi(-2.0 * (double)((tt * m) % D) / (double)D, &sn, &cs);
        twt[tt * K::TWS + m] = make_float2((float)cs, (float)sn);
    }
    const float2* tw = twt + h8 * K::TWS;
    auto mark = [](int) {};
    int xb = 0;   // XDB: exchange buffer of the next round
    // one tile: fused7's dft_tile, or the double-buffered one
    auto tile = [&](float2* v, int os, int oi, auto&& before, auto&& after, auto&& emit, auto&& mid) {
        if constexpr (XDB)
            dft_tile_db<D>(v, tw, X2, xb, s8, h8, os, oi, before, after, emit, A.dbg, mid);
        else
            dft_tile<D>(v, tw, X2, s8, h8, os, oi, before, after, emit, A.dbg, mark, mid);
    };
    int* queue = A.ctr;
    int* doneA = A.ctr + 1;
    int* doneB = A.ctr + 1 + A.S;
    const int64_t MQD = (int64_t)M * Q * D;
    if (tid == 0) {
        if (tma::saddr(F) & 127) __trap();   // TMA destinations are 128-byte aligned
        tma::prefetch_map(&tm.f);
        tma::prefetch_map(&tm.ws);
        tma::mbar_init(&mbar, 1);
        tma::fence_mbar_init();
    }
    uint32_t phase = 0;
    // thread 0: copy the input tile of (isA, w, idx, bt) into F (two boxes of 256 rows)
    auto issue = [&](int isA, int w, int idx, int bt) {
        tma::fence_proxy_async();
        tma::mbar_expect_tx(&mbar, TILE_BYTES);
        if (isA) {
            const int x = idx * AC, y = w * D;
            tma::load_2d(F, &tm.f, x, y, &mbar);
            if (D > 256) tma::load_2d(F + 256 * 8, &tm.f, x, y + 256, &mbar);
        } else {
            const int x = idx * 16 + 8 * bt, y = (w % A.S) * M;
            tma::load_2d(F, &tm.ws, x, y, &mbar);
            if (D > 256) tma::load_2d(F + 256 * 8, &tm.ws, x, y + 256, &mbar);
        }
    };
    // every thread: wait for the tile, then take its column s8, rows h8 + 16 k
    float2 pre[R1];
    auto take = [&]() {
        tma::mbar_wait(&mbar, phase);
        phase ^= 1;
#pragma unroll
        for (int k = 0; k < R1; ++k) pre[k] = F[(h8 + 16 * k) * 8 + s8];
    };
    auto load_g = [&](int j0, int h, int b) {
        const float4* G4 = A.Gp + ((int64_t)((j0 / AC) * 4 + h) * (R1 / 2)) * 128 + h8 * 8 + s8;
#pragma unroll
        for (int kp = 8 * b; kp < 8 * b + 8 && kp < R1 / 2; ++kp) {
            const float4 g = (A.dbg & 32) ? make_float4(1.f, 0.f, 1.f, 0.f) : ldg_na(G4 + kp * 128);
            pre[2 * kp] = make_float2(g.x, g.y);
            pre[2 * kp + 1] = make_float2(g.z, g.w);
        }
    };
    int pnext = -1;
    // thread 0 (after the tile's first exchange barrier: F is free): publish the next job and,
    // when its inputs may be read now, start their copy
    auto claim_issue = [&]() {
        int isA0, idx0, w0, ready = 0;
        if (decode(pnext, A.W, A.lag, A.nA, A.nB, &isA0, &w0, &idx0)) {
            const int gen0 = w0 / A.S, slot0 = w0 - gen0 * A.S;
            ready = isA0 || (A.dbg & 1) || ld_acquire(doneA + slot0) >= (gen0 + 1) * A.nA;
            if (ready) issue(isA0, w0, idx0, 0);
        }
        jobsm[0] = pnext;
        jobsm[1] = ready;
    };
    int* pend = nullptr;
    auto flush = [&]() {
        if (pend) {
            signal_release(pend);
            pend = nullptr;
        }
    };
    if (tid == 0) {
        jobsm[0] = atomicAdd(queue, 1);
        jobsm[1] = 0;
    }
    __syncthreads();
    for (;;) {
        const int pref = jobsm[1];
        if (tid == 0) {
            int isA0, idx0, w0;
            if (decode(jobsm[0], A.W, A.lag, A.nA, A.nB, &isA0, &w0, &idx0)) {
                jobdec[0] = isA0; jobdec[1] = w0; jobdec[2] = idx0;
            } else {
                jobdec[0] = -1;
            }
        }
        __syncthreads();
        const int isA = jobdec[0];
        if (isA < 0) break;
        const int w = jobdec[1], idx = jobdec[2];
        const int gen = w / A.S, slot = w - gen * A.S;
        float2* wsl = A.ws + (int64_t)slot * MQD;
        if (tid == 0) {
            if (!(A.dbg & 1)) {
                const int* cnt = isA ? doneB + slot : (pref ? nullptr : doneA + slot);
                const int target = isA ? gen * A.nB : (gen + 1) * A.nA;
                if (cnt && ld_acquire(cnt) < target) {
                    flush();
                    spin_until(cnt, target);
                }
            }
            if (!pref) issue(isA, w, idx, 0);   // (B: after the dependency spin)
        }
        take();
        if (isA) {
            const int j0 = idx * AC;
            tile(pre, s8, h8, [&] { if (tid == 0) flush(); },
                 [&] {
                     load_g(j0, 0, 0);
                     if (FULLPF && R1 > 16) load_g(j0, 0, 1);
                 },
                 [&](int r, const float2* y) {
#pragma unroll
                     for (int m2 = 0; m2 < 16; ++m2) F[s8 * K::FS + 16 * r + h8 + R1 * m2] = y[m2];
                 },
                 [] {});
            __syncthreads();   // F complete; X free
            const int wq = tid >> 5, ln = tid & 31;
            const int colM = wq >> 1, uM = ln >> 3, iM = (ln & 7) + 8 * (wq & 1);
#pragma unroll 1
            for (int h = 0; h < 4; ++h) {
                const int fcol = 2 * h + (s8 >> 2);
                const int jS = j0 + fcol;
                const int sig = (int)((((int64_t)jS * A.beta - ((int64_t)A.Kmod * jS) % D) % D + D) % D);
                if (h == 3 && tid == 0) pnext = atomicAdd(queue, 1);
                const float2* Fc = F + fcol * K::FS;
                const int e0 = (sig - h8) & (D - 1);
#pragma unroll
                for (int k = 0; k < 16; ++k) pre[k] = cmw(Fc[(e0 - 16 * k) & (D - 1)], pre[k]);
                if (R1 > 16) {
                    if (!FULLPF) {
                        asm volatile("" ::: "memory");
                        load_g(j0, h, 1);
                    }
#pragma unroll
                    for (int k = 16; k < R1; ++k) pre[k] = cmw(Fc[(e0 - 16 * k) & (D - 1)], pre[k]);
                }
                if (!XDB || h == 3) __syncthreads();   // previous tile's readers are done with X; (h = 3) F is dead
                if (h == 3 && tid == 0) claim_issue();
                const int jM = j0 + 2 * h + colM;
                const int kap = ((jM / A.c - uM) % Q + Q) % Q;
                float2* dst = wsl + (int64_t)jM * (Q * D) + (iM >> 2) * 16 + (iM & 3) * 4 + kap;
                tile(pre, 4 * colM + uM, iM, [] {},
                     [&] {
                         if (h < 3) {
                             load_g(j0, h + 1, 0);
                             if (FULLPF && R1 > 16) load_g(j0, h + 1, 1);
                         }
                     },
                     [&](int r, const float2* y) {
                         if (A.dbg & (4 | 128)) return;
#pragma unroll
                         for (int m2 = 0; m2 < 16; ++m2) dst[(4 * r + (R1 / 4) * m2) * 16] = y[m2];
                     },
                     [] {});
            }
            if (tid == 0) pend = doneA + slot;
        } else {
#pragma unroll 1
            for (int bt = 0; bt < BT; ++bt) {
                if (bt == BT - 1 && tid == 0) pnext = atomicAdd(queue, 1);
                const int n = idx * 16 + 8 * bt + s8;
                const float2 e = ldg_na2(A.E + n);
                float2* dst = A.out + (int64_t)w * M * N + n;
                if (bt) {
                    if (!XDB) __syncthreads();   // previous tile's readers are done with X
                    take();
                }
                tile(pre, s8, h8, [&] { if (tid == 0) flush(); }, [] {},
                     [&](int r, const float2* y) {
                         if (A.dbg & (4 | 64)) return;
#pragma unroll
                         for (int m2 = 0; m2 < 16; ++m2) {
                             const int m = 16 * r + h8 + R1 * m2;
                             __stcs(dst + m * N, cmw(y[m2], e));
                         }
                     },
                     [&] {   // F free: the next tile's copy
                         if (tid == 0) {
                             if (bt + 1 < BT) issue(0, w, idx, bt + 1);
                             else claim_issue();
                         }
                     });
            }
#pragma unroll
            for (int j = tid; j < M; j += K::NT)
                asm volatile("discard.global.L2 [%0], 128;" ::"l"(wsl + (int64_t)j * (Q * D) + idx * 16) : "memory");
            if (tid == 0) pend = doneB + slot;
        }
    }
    __syncthreads();
    if (tid == 0) flush();
}

// ------------------------------------------------------------------------------------
// plan-time table G' (fp64 arithmetic, stored once as complex64)
// ------------------------------------------------------------------------------------
struct GpArgs {
    float4* Gp;            // [M][Q][R1/2][16] float4
    const double2* G64;    // [(r*Q + u)*D + nu] = conj(Gamma_r(u; nu))/d
    int64_t L, K;          // chirp exponent K = sigma (L+1) mod 2L
    int M, D, Q, c, beta, R1;
    int layout;            // 0: fused7 stage-1 order; 1: fused7a stage-2 order [j/8][h][r][m2][col][oi][u]
    int alpha[16];         // alpha_{l,u}, l,u < Q
};

__global__ void k_gprime(GpArgs a) {
    const int64_t total = (int64_t)a.M * a.Q * a.D;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int mu = (int)(i % a.D);
        const int u = (int)((i / a.D) % a.Q);
        const int j = (int)(i / ((int64_t)a.D * a.Q));
        const int r = j % a.c, l = j / a.c;
        const int e = (l >= u) ? 0 : -1;   // floor((l - u)/q) for l, u < q
        const int gi = (int)((((int64_t)j * a.beta - mu) % a.D + a.D) % a.D);
        const double2 g = a.G64[((int64_t)r * a.Q + u) * a.D + gi];
        // C(j) = exp(i pi (K j^2 mod 2L) / L)
        const unsigned __int128 twoL = 2 * (unsigned __int128)a.L;
        const unsigned __int128 ce = ((unsigned __int128)a.K * (((unsigned __int128)j * j) % twoL)) % twoL;
        double s1, c1;
        sincospi((double)(int64_t)ce / (double)a.L, &s1, &c1);
        // W_D^{j alpha - mu e}
        const int64_t ex = (((int64_t)j * a.alpha[l * a.Q + u] - (int64_t)mu * e) % a.D + a.D) % a.D;
        double s2, c2;
        sincospi(-2.0 * (double)ex / (double)a.D, &s2, &c2);
        const double pr = c1 * c2 - s1 * s2, pi = c1 * s2 + s1 * c2;
        const double vr = g.x * pr - g.y * pi, vi = g.x * pi + g.y * pr;
        // layout [j / 8][h][kp][t][slot][2]: j = 8 jb + 2 h + col, slot = 4 col + u, mu = t + 16 k,
        // k = 2 kp + hh (the order one product tile of fused7_kernel reads it)
        const int jb = j / 8, hq = (j % 8) / 2, col = j % 2, sl = 4 * col + u;
        float2* dst;
        if (a.layout == 0) {
            const int t = mu & 15, k = mu >> 4;
            dst = reinterpret_cast<float2*>(a.Gp) +
                  (((((int64_t)jb * 4 + hq) * (a.R1 / 2) + (k >> 1)) * 16 + t) * 8 + sl) * 2 + (k & 1);
        } else {
            // mu = 16 r + oi + R1 m2 (the stage-2 output index of lane oi, round r)
            const int r = (mu % a.R1) >> 4, oi = (mu % a.R1) & 15, m2 = mu / a.R1;
            dst = reinterpret_cast<float2*>(a.Gp) +
                  ((((((int64_t)jb * 4 + hq) * (a.R1 / 16) + r) * 16 + m2) * 2 + col) * 64 + oi * 4 + u);
        }
        *dst = make_float2((float)vr, (float)vi);
    }
}

}  // namespace v7
}  // namespace nsdgt
