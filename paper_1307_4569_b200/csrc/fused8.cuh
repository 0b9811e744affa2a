// fused8.cuh -- round-2 hot-path kernel for the time-shear / separable branch with p = 1,
// q = 4, d = M in {256, 512}, complex64 (BASELINE configs 3 and 5).  DESIGN.md §4.3.
//
// Same transform as fused7 (fused7.cuh header; Alg. 1 of PAPER.md:852-873 on the
// factorisation DGT of PAPER.md:790-804):
//
//   pass A, column j:  F_j(mu) = sum_s f(j + sM) W_D^{s mu}                        (Zak DFT)
//                      x_{j,u}(mu) = F_j((sigma_j - mu) mod D) G'_{j,u}(mu),  u < q
//                      ws[j][kappa][n'] = DFT_D[x_{j,u}](n'),  kappa = (l - u) mod q
//   pass B, column n:  c[m][n] = E(n) sum_j ws[j][n mod q][n div q] W_M^{j m}
//
// What changes against fused7 is the tile: 16 slots x 16 lanes (a CTA of 256 threads, two
// per SM) instead of 8 x 16.  Sixteen slots are sixteen consecutive columns, i.e. 128 bytes of
// a row of f, of a ring line or of a row of c, so every global access of the kernel is whole
// 128-byte lines: a warp instruction of the stage-1 role (16 slots x 2 lanes t) reads two
// whole lines of f or of the ring, a warp of the B-tile stage-2 role writes two whole lines of
// c, a warp of the product stage-2 role two whole ring lines, and the window table G' is read
// in 512-byte runs.  (fused7's 8-column tiles touched 64 bytes per line, so f, ring loads and
// c stores cost two L1 wavefronts per 128 bytes.)  Further:
//  * exchange buffer rows of 20 (16 + 4) and slot stride 321 (= 1 mod 16): the stage-1 writes
//    (16 slots at one t) and all three stage-2 read roles hit 16 distinct bank pairs;
//  * F column stride D + 3 (= 3 mod 16): the Zak-tile F stores (16 columns at one index) and the
//    product-tile F gathers (4 columns x 4 u, the four u broadcast) are conflict-free;
//  * the twiddle row of a lane t is shared by its half-warp (broadcast).
// Jobs: A = 16 consecutive columns j (one Zak tile + four product tiles of 4 columns x 4 u),
// B = 16 consecutive columns n (one tile, one ring line per row j).  Queue, ring slots,
// dependency counters, deferred completion signals, L2 discards and the cross-tile register
// prefetch are fused7's (see there).
#pragma once
#include "fused7.cuh"

namespace nsdgt {
namespace v8 {

using v7::Args;
using v7::cmw;
using v7::decode;
using v7::dft16;
using v7::dftR;
using v7::ld_acquire;
using v7::ld_cg;
using v7::ldg_na;
using v7::ldg_na2;
using v7::lds128_nohoist;
using v7::spin_until;

template <int D>
struct Cfg {
    static constexpr int R1 = D / 16;            // stage-1 length (32 or 16)
    static constexpr int NR = R1 / 16;           // exchange rounds (2 or 1)
    static constexpr int Q = 4;
    static constexpr int NS = 16;                // tile slots
    static constexpr int NT = 16 * NS;           // 256 threads
    static constexpr int ACOL = 16;              // columns j per A job
    static constexpr int RS = 20;                // exchange row stride (16 t + 4), = 4 mod 16
    static constexpr int SS = 16 * RS + 1;       // exchange slot stride, = 1 mod 16
    static constexpr int XE = NS * SS;           // one exchange round, complex (41 KB)
    static constexpr int FS = D + 3;             // F column stride, = 3 mod 16
    static constexpr int FE = ACOL * FS;
    static constexpr int TWS = R1 + 2;           // twiddle row stride (even: 16-byte pairs)
    static constexpr int TW = 16 * TWS;
    static constexpr size_t SMEM = (size_t)(XE + FE + TW) * 8;
};

// Stage 1 -> exchange -> stage 2 of a 16-slot D-point DFT tile (256 threads).
//   in:  v[k] = x(t + 16 k) of slot s, lane t  (role S1: s = tid & 15, t = tid >> 4)
//   out: emit(r, y), y[m2] = X(16 r + oi + R1 m2) of slot os
// Per round: write 16 values (twiddled), barrier, read one sequence, [barrier].  before_sync
// runs after the first-round writes, after_sync after the last round's reads (v is dead).
template <int D, class Before, class After, class Emit>
__device__ __forceinline__ void dft_tile(float2* v, const float2* tw, float2* X, int s, int t, int os, int oi,
                                         Before&& before_sync, After&& after_sync, Emit&& emit, int dbg) {
    using K = Cfg<D>;
    constexpr int R1 = K::R1, NR = K::NR;
    if (!(dbg & 8)) dftR<R1>(v);
    const float4* tw4 = reinterpret_cast<const float4*>(tw);
    float2* xw = X + s * K::SS + t;                 // + RS m1'
    const float2* xr = X + os * K::SS + oi * K::RS; // + tt
#pragma unroll
    for (int r = 0; r < NR; ++r) {
#pragma unroll
        for (int m = 0; m < 16; m += 2) {
            const float4 w2 = lds128_nohoist(tw4 + ((16 * r + m) >> 1));
            const float2 a = (r || m) ? cmw(v[16 * r + m], make_float2(w2.x, w2.y)) : v[16 * r];
            const float2 b = cmw(v[16 * r + m + 1], make_float2(w2.z, w2.w));
            xw[K::RS * m] = a;
            xw[K::RS * (m + 1)] = b;
            if ((m & 7) == 6) asm volatile("" ::: "memory");
        }
        if (r == 0) before_sync();
        __syncthreads();
        float2 y[16];
#pragma unroll
        for (int tt = 0; tt < 16; ++tt) y[tt] = xr[tt];
        if (r + 1 < NR) __syncthreads();
        if (r == NR - 1) after_sync();
        if (!(dbg & 8)) dft16(y);
        emit(r, y);
    }
}

template <int D, int MINB, bool REAL = false>
__global__ void __launch_bounds__(256, MINB) fused8_kernel(Args A) {
    using K = Cfg<D>;
    constexpr int R1 = K::R1, Q = K::Q, M = D, AC = K::ACOL;
    constexpr int N = Q * D;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float2* X = reinterpret_cast<float2*>(smem_raw);
    float2* F = X + K::XE;         // F[col * FS + nu], col < 16
    float2* twt = F + K::FE;       // twt[t][m] = W_D^{t m}
    __shared__ int jobsm[2];       // next job, 1 if its first tile's inputs were prefetched
    __shared__ int jobdec[4];
    const int tid = threadIdx.x;
    // roles: S1 (every stage 1; stage 2 of Zak and B tiles): slot s16 = tid & 15, t = h16 = tid >> 4
    //        P2 (stage 2 of product tiles): u = L & 3, oi = 4 (w & 3) + ((L >> 2) & 3), col = 2 (w >> 2) + (L >> 4)
    const int s16 = tid & 15, h16 = tid >> 4;
    const int wq = tid >> 5, ln = tid & 31;
    const int uP = ln & 3, oiP = 4 * (wq & 3) + ((ln >> 2) & 3), colP = 2 * (wq >> 2) + (ln >> 4);
    for (int e = tid; e < 16 * R1; e += K::NT) {
        const int tt = e / R1, m = e % R1;
        double sn, cs;
        sincospi(-2.0 * (double)((tt * m) % D) / (double)D, &sn, &cs);
        twt[tt * K::TWS + m] = make_float2((float)cs, (float)sn);
    }
    const float2* tw = twt + h16 * K::TWS;
    int* queue = A.ctr;
    int* doneA = A.ctr + 1;
    int* doneB = A.ctr + 1 + A.S;
    const int64_t MQD = (int64_t)M * Q * D;

    float2 pre[R1];
    auto load_f = [&](int w, int j0) {   // Zak input: column j0 + s16, rows t + 16 k
        if constexpr (REAL) {
            const float* fr = reinterpret_cast<const float*>(A.f) + (int64_t)w * M * D + j0 + s16;
#pragma unroll
            for (int k = 0; k < R1; ++k) pre[k] = make_float2(__ldcs(fr + (int64_t)(h16 + 16 * k) * M), 0.f);
        } else {
            const float2* fw = A.f + (int64_t)w * M * D + j0 + s16;
#pragma unroll
            for (int k = 0; k < R1; ++k) pre[k] = ldg_na2(fw + (int64_t)(h16 + 16 * k) * M);
        }
    };
    // G' of product tile h: layout [j / 16][h][kp][t][slot] of float4 (k = 2 kp, 2 kp + 1)
    auto load_g = [&](int j0, int h) {
        const float4* G4 = A.Gp + ((int64_t)((j0 / AC) * 4 + h) * (R1 / 2)) * 256 + h16 * 16 + s16;
#pragma unroll
        for (int kp = 0; kp < R1 / 2; ++kp) {
            const float4 g = (A.dbg & 32) ? make_float4(1.f, 0.f, 1.f, 0.f) : ldg_na(G4 + kp * 256);
            pre[2 * kp] = make_float2(g.x, g.y);
            pre[2 * kp + 1] = make_float2(g.z, g.w);
        }
    };
    // B input: ring line (j, idx) of signal w, position s16, rows j = t + 16 k
    auto load_ring = [&](int w, int idx) {
        const float2* src = A.ws + (int64_t)(w % A.S) * MQD + (int64_t)h16 * (Q * D) + idx * 16 + s16;
#pragma unroll
        for (int k = 0; k < R1; ++k) pre[k] = ld_cg(src + (int64_t)(16 * k) * (Q * D));
    };
    auto load_first = [&](int isA, int w, int idx) {
        if (isA) load_f(w, idx * AC);
        else load_ring(w, idx);
    };
    int pnext = -1;
    auto claim_ready = [&]() {
        int isA0, idx0, w0, ready = 0;
        if (decode(pnext, A.W, A.lag, A.nA, A.nB, &isA0, &w0, &idx0)) {
            const int gen0 = w0 / A.S, slot0 = w0 - gen0 * A.S;
            ready = isA0 || (A.dbg & 1) || ld_acquire(doneA + slot0) >= (gen0 + 1) * A.nA;
        }
        jobsm[0] = pnext;
        jobsm[1] = ready;
    };
    auto prefetch_next = [&]() {
        int isA0, idx0, w0;
        if (jobsm[1] && decode(jobsm[0], A.W, A.lag, A.nA, A.nB, &isA0, &w0, &idx0)) load_first(isA0, w0, idx0);
    };
    int* pend = nullptr;
    auto flush = [&]() {
        if (pend) {
            v7::signal_release(pend);
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
        if (tid == 0 && !(A.dbg & 1)) {
            const int* cnt = isA ? doneB + slot : (pref ? nullptr : doneA + slot);
            const int target = isA ? gen * A.nB : (gen + 1) * A.nA;
            if (cnt && ld_acquire(cnt) < target) {
                flush();
                spin_until(cnt, target);
            }
        }
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
            if (!isA) __syncthreads();   // B inputs only after the dependency spin
            load_first(isA, w, idx);
        }
        if (isA) {
            // ---------------- pass A: columns j0 .. j0 + 15 ----------------
            const int j0 = idx * AC;
            dft_tile<D>(pre, tw, X, s16, h16, s16, h16, [&] { if (tid == 0) flush(); },
                        [&] { load_g(j0, 0); },
                        [&](int r, const float2* y) {
#pragma unroll
                            for (int m2 = 0; m2 < 16; ++m2) F[s16 * K::FS + 16 * r + h16 + R1 * m2] = y[m2];
                        }, A.dbg);
            __syncthreads();   // F complete; X free
            const int fcolS = s16 >> 2;   // S1 role in product tiles: column (within the tile), u = s16 & 3
            const int lP = j0 / A.c;      // l of every column of the job (16 | c)
            const int kap = ((lP - uP) % Q + Q) % Q;
#pragma unroll 1
            for (int h = 0; h < 4; ++h) {
                const int fcol = 4 * h + fcolS;
                const int jS = j0 + fcol;
                const int sig = (int)((((int64_t)jS * A.beta - ((int64_t)A.Kmod * jS) % D) % D + D) % D);
                if (h == 3 && tid == 0) pnext = atomicAdd(queue, 1);
                const float2* Fc = F + fcol * K::FS;
                const int e0 = (sig - h16) & (D - 1);
#pragma unroll
                for (int k = 0; k < R1; ++k) pre[k] = cmw(Fc[(e0 - 16 * k) & (D - 1)], pre[k]);
                __syncthreads();   // previous tile's readers are done with X
                const int jM = j0 + 4 * h + colP;
                float2* dst = wsl + (int64_t)jM * (Q * D) + (oiP >> 2) * 16 + (oiP & 3) * 4 + kap;
                dft_tile<D>(pre, tw, X, s16, h16, 4 * colP + uP, oiP,
                            [&] { if (h == 3 && tid == 0) claim_ready(); },
                            [&] {
                                if (h < 3) load_g(j0, h + 1);
                                else prefetch_next();
                            },
                            [&](int r, const float2* y) {
                                if (A.dbg & (4 | 128)) return;
#pragma unroll
                                for (int m2 = 0; m2 < 16; ++m2) dst[(4 * r + (R1 / 4) * m2) * 16] = y[m2];
                            }, A.dbg);
            }
            if (tid == 0) pend = doneA + slot;
        } else {
            // ---------------- pass B: columns 16 idx .. 16 idx + 15 (ring line idx) ----------------
            if (tid == 0) pnext = atomicAdd(queue, 1);
            const int n = idx * 16 + s16;
            const float2 e = ldg_na2(A.E + n);
            float2* dst = A.out + (int64_t)w * M * N + n;
            dft_tile<D>(pre, tw, X, s16, h16, s16, h16,
                        [&] {
                            if (tid == 0) {
                                flush();
                                claim_ready();
                            }
                        },
                        [&] { prefetch_next(); },
                        [&](int r, const float2* y) {
                            if (A.dbg & (4 | 64)) return;
#pragma unroll
                            for (int m2 = 0; m2 < 16; ++m2) {
                                const int m = 16 * r + h16 + R1 * m2;
                                __stcs(dst + m * N, cmw(y[m2], e));
                            }
                        }, A.dbg);
            // the ring lines of this job are dead: drop them from L2 (no write-back)
#pragma unroll
            for (int j = tid; j < M; j += K::NT)
                asm volatile("discard.global.L2 [%0], 128;" ::"l"(wsl + (int64_t)j * (Q * D) + idx * 16) : "memory");
            if (tid == 0) pend = doneB + slot;
        }
        // (the loop-top barrier frees X / F for the next job and orders this job's stores and
        // discards before its deferred completion signal)
    }
    if (tid == 0) flush();
}

// G' (fused7.cuh k_gprime, fp64) in fused8's stage-1 order: [j / 16][h][kp][t][slot16][2],
// j = 16 jb + 4 h + col, slot16 = 4 col + u, mu = t + 16 k, k = 2 kp + (k & 1)
__global__ void k_gprime8(v7::GpArgs a) {
    const int64_t total = (int64_t)a.M * a.Q * a.D;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int mu = (int)(i % a.D);
        const int u = (int)((i / a.D) % a.Q);
        const int j = (int)(i / ((int64_t)a.D * a.Q));
        const int r = j % a.c, l = j / a.c;
        const int e = (l >= u) ? 0 : -1;
        const int gi = (int)((((int64_t)j * a.beta - mu) % a.D + a.D) % a.D);
        const double2 g = a.G64[((int64_t)r * a.Q + u) * a.D + gi];
        const unsigned __int128 twoL = 2 * (unsigned __int128)a.L;
        const unsigned __int128 ce = ((unsigned __int128)a.K * (((unsigned __int128)j * j) % twoL)) % twoL;
        double s1, c1;
        sincospi((double)(int64_t)ce / (double)a.L, &s1, &c1);
        const int64_t ex = (((int64_t)j * a.alpha[l * a.Q + u] - (int64_t)mu * e) % a.D + a.D) % a.D;
        double s2, c2;
        sincospi(-2.0 * (double)ex / (double)a.D, &s2, &c2);
        const double pr = c1 * c2 - s1 * s2, pi = c1 * s2 + s1 * c2;
        const double vr = g.x * pr - g.y * pi, vi = g.x * pi + g.y * pr;
        const int jb = j / 16, hq = (j % 16) / 4, col = j % 4, sl = 4 * col + u;
        const int t = mu & 15, k = mu >> 4;
        float2* dst = reinterpret_cast<float2*>(a.Gp) +
                      (((((int64_t)jb * 4 + hq) * (a.R1 / 2) + (k >> 1)) * 16 + t) * 16 + sl) * 2 + (k & 1);
        *dst = make_float2((float)vr, (float)vi);
    }
}

}  // namespace v8
}  // namespace nsdgt
