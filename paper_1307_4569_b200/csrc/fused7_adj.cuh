// fused7_adj.cuh -- synthesis (the adjoint of fused7) for the same lattices: time shear /
// separable, p = 1, q = 4, d = M in {256, 512}, complex64 (BASELINE configs 3 and 5).
// DESIGN.md §4.5.  The plan's window is the synthesis window gamma (pass the canonical dual
// to invert); f = sum c(m,n) M_{b(m+w(n))} T_{an} gamma, the inversion formula of
// PAPER.md:171-175.
//
// fused7 computes, per signal (fused7.cuh header):
//   pass A, column j:  F_j(mu) = sum_s f(j + sM) W^{s mu};  x_{j,u}(mu) = F_j((sigma_j - mu) mod D) G'_{j,u}(mu);
//                      ws[j][n] = DFT_D[x_{j,u}](n'),  n = kappa + q n', kappa = (l - u) mod q
//   pass B, column n:  c[m][n] = E(n) sum_j ws[j][n] W^{j m}
// Its adjoint runs the passes in the opposite order, every map replaced by its adjoint and
// every inverse DFT computed as conj(DFT(conj(.))) on the same tile machinery:
//   pass B', column n: ws'[j][n] = conj(E(n) Y_n(j)),  Y_n = DFT_M[conj(c[.][n])]
//   pass A', column j: X_{j,u} = DFT_D[conj(ws'[j][kappa + q .])],
//                      Fc_j(nu) = sum_u G'_{j,u}(mu) X_{j,u}(mu) at nu = (sigma_j - mu) mod D
//                      (= conj of the adjoint's F'_j; the sum over u is a shuffle reduction:
//                      the four u of a column sit in lanes L, L^8, L^16, L^24 of one warp),
//                      f(j + sM) = conj(DFT_D[Fc_j](s)).
// The ring ws (same slots and line layout as fused7: row j holds the N columns n in natural
// order) now carries pass B' -> pass A'; each A' job is the only reader of its eight rows and
// discards them from L2 afterwards.  Jobs: B'(w) (16 columns n) are queued lag signals ahead
// of A'(w) (8 columns j); B'(w) waits until slot w mod S is free (all A'(w - S) done), A'(w)
// waits for all B'(w).  The window table is G' of fused7 stored in the stage-2 (output)
// order of a product tile (k_gprime layout 1).
#pragma once
#include "fused7.cuh"

namespace nsdgt {
namespace v7 {

__device__ __forceinline__ float2 conjf2(float2 a) { return make_float2(a.x, -a.y); }

// A (the fused7 Args): f = coefficients c [W][M][N] (input), out = signal [W][L] (output),
// Gp = G' in layout 1 (float2 view).
template <int D, int MINB>
__global__ void __launch_bounds__(128, MINB) fused7a_kernel(Args A) {
    using K = Cfg<D>;
    constexpr int R1 = K::R1, NR = K::NR, Q = K::Q, M = D, AC = K::ACOL;
    constexpr int N = Q * D;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float2* X2 = reinterpret_cast<float2*>(smem_raw);
    float2* F = X2 + K::XE;        // Fc[col * FS + nu], col < ACOL
    float2* twt = F + K::FE;
    __shared__ int jobsm;
    __shared__ int jobdec[6];   // decoded job (thread 0): ok, isB, w, idx, gen, slot
    const int tid = threadIdx.x;
    const int s8 = tid & 7, h8 = tid >> 3;                  // roles S1 / M1
    const int wq = tid >> 5, ln = tid & 31;                 // role M3 (product tiles, stage 2)
    const int colM = wq >> 1, uM = ln >> 3, iM = (ln & 7) + 8 * (wq & 1);
    for (int e = tid; e < 16 * R1; e += K::NT) {
        const int tt = e / R1, m = e % R1;
        double sn, cs;
        sincospi(-2.0 * (double)((tt * m) % D) / (double)D, &sn, &cs);
        twt[tt * K::TWS + m] = make_float2((float)cs, (float)sn);
    }
    const float2* tw = twt + h8 * K::TWS;
    auto mark = [](int) {};
    auto none = [] {};
    int* queue = A.ctr;
    int* doneB = A.ctr + 1;
    int* doneA = A.ctr + 1 + A.S;
    const int64_t MN = (int64_t)M * N;
    const int64_t L = (int64_t)M * D;
    const float2* Gq = reinterpret_cast<const float2*>(A.Gp);
    float2 pre[R1];
    int* pend = nullptr;
    for (;;) {
        // the previous job's shared-memory readers are done and its stores (and L2 discards)
        // are ordered before thread 0's completion signal
        __syncthreads();
        if (tid == 0) {
            if (pend) {
                signal_release(pend);
                pend = nullptr;
            }
            jobsm = atomicAdd(queue, 1);
            int isB0, w0, idx0;
            jobdec[0] = decode(jobsm, A.W, A.lag, A.nB, A.nA, &isB0, &w0, &idx0) ? 1 : 0;
            const int gen0 = w0 / A.S;
            jobdec[1] = isB0; jobdec[2] = w0; jobdec[3] = idx0; jobdec[4] = gen0; jobdec[5] = w0 - gen0 * A.S;
        }
        __syncthreads();
        if (!jobdec[0]) break;
        const int isB = jobdec[1], w = jobdec[2], idx = jobdec[3];
        const int gen = jobdec[4], slot = jobdec[5];
        float2* wsl = A.ws + (int64_t)slot * MN;
        // B' reads only the (read-only) coefficients; its dependency gates the ring stores, so
        // its first tile's loads are issued before the wait and overlap it
        auto load_c = [&](int bt) {
            const float2* src = A.f + (int64_t)w * MN + idx * 16 + 8 * bt + s8;
#pragma unroll
            for (int k = 0; k < R1; ++k) pre[k] = ldg_na2(src + (int64_t)(h8 + 16 * k) * N);
        };
        if (isB) load_c(0);
        if (tid == 0 && !(A.dbg & 1)) {
            // B': slot free (all A'(w - S) done); A': all B'(w) done
            if (isB) spin_until(doneA + slot, gen * A.nA);
            else spin_until(doneB + slot, (gen + 1) * A.nB);
        }
        __syncthreads();   // every thread's ring accesses follow thread 0's acquire
        if (isB) {
            // ---------------- pass B': columns n = 16 idx .. 16 idx + 15 ----------------
            // tile bt's input: column n = 16 idx + 8 bt + s8, rows m = t + 16 k (conjugated when
            // used); tile 0's was issued before the dependency wait
#pragma unroll 1
            for (int bt = 0; bt < 2; ++bt) {
                const int n = idx * 16 + 8 * bt + s8;
                const float2 e = ldg_na2(A.E + n);
#pragma unroll
                for (int k = 0; k < R1; ++k) pre[k] = conjf2(pre[k]);
                if (bt) __syncthreads();   // previous tile's readers are done with X2
                dft_tile<D>(pre, tw, X2, s8, h8, s8, h8, none,
                            [&] {
                                if (bt == 0) load_c(1);   // next tile's inputs behind this tile's stage 2
                            },
                            [&](int r, const float2* y) {
#pragma unroll
                                for (int m2 = 0; m2 < 16; ++m2) {
                                    const int j = 16 * r + h8 + R1 * m2;
                                    wsl[(int64_t)j * N + n] = conjf2(cmw(y[m2], e));
                                }
                            }, A.dbg, mark);
            }
            if (tid == 0) pend = doneB + slot;
        } else {
            // ---------------- pass A': columns j0 .. j0 + 7 ----------------
            const int j0 = idx * AC;
            const int lJ = j0 / A.c;   // l of every column of the job (c % 8 == 0)
            // product tile h's input: stage-1 slot s8 = (column j0 + 2h + (s8 >> 2), u = s8 & 3),
            // lane t = h8: ws'[j][kappa + q (t + 16 k)] (conjugated when used)
            auto load_r = [&](int h) {
                const int jS = j0 + 2 * h + (s8 >> 2);
                const int kapS = (lJ - (s8 & 3)) & (Q - 1);
                const float2* src = wsl + (int64_t)jS * N + kapS + 4 * h8;
#pragma unroll
                for (int k = 0; k < R1; ++k) pre[k] = ld_cg(src + 64 * k);
            };
#pragma unroll 1
            for (int h = 0; h < 4; ++h) {
                if (h == 0) load_r(0);
#pragma unroll
                for (int k = 0; k < R1; ++k) pre[k] = conjf2(pre[k]);
                __syncthreads();   // previous tile's readers are done with X2
                const int jM = j0 + 2 * h + colM;
                const int sig = (jM * (A.beta - A.Kmod)) & (D - 1);   // (j beta - K j) mod D, D a power of 2
                float2* Fc = F + (2 * h + colM) * K::FS;
                // G' in stage-2 order: [j0/8][h][r][m2][col][oi][u]
                const float2* g = Gq + ((((int64_t)idx * 4 + h) * NR * 16) * 2 + colM) * 64 + iM * 4 + uM;
                // the G' values of a round are loaded one exchange ahead (round 0's before the
                // first barrier, round r + 1's during round r's emit) so their latency hides
                // behind the barrier, the exchange reads and the DFT-16
                // (at 3 CTAs/SM only: the 5-CTA variant has no registers to spare, measured
                // config 3 0.39 -> 0.43 ms with it; config 5 6.25 -> 6.14 ms)
                constexpr bool GPF = MINB <= 3;
                float2 gr[16];
                auto load_g = [&](int r) {
#pragma unroll
                    for (int m2 = 0; m2 < 16; ++m2) gr[m2] = ldg_na2(g + ((int64_t)(r * 16 + m2) * 2) * 64);
                };
                dft_tile<D>(pre, tw, X2, s8, h8, 4 * colM + uM, iM,
                            [&] {
                                if (GPF) load_g(0);
                            },
                            [&] {
                                if (h < 3) load_r(h + 1);   // next tile's inputs behind this tile's stage 2
                            },
                            [&](int r, const float2* y) {
                                float2 gn[16];
                                if (!GPF) load_g(r);
#pragma unroll
                                for (int m2 = 0; m2 < 16; ++m2) gn[m2] = gr[m2];
                                if (GPF && r + 1 < NR) load_g(r + 1);
#pragma unroll
                                for (int m2 = 0; m2 < 16; ++m2) {
                                    float2 p = cmw(y[m2], gn[m2]);
                                    p.x += __shfl_xor_sync(0xffffffffu, p.x, 8);
                                    p.y += __shfl_xor_sync(0xffffffffu, p.y, 8);
                                    p.x += __shfl_xor_sync(0xffffffffu, p.x, 16);
                                    p.y += __shfl_xor_sync(0xffffffffu, p.y, 16);
                                    const int mu = 16 * r + iM + R1 * m2;
                                    if (uM == (m2 & 3)) Fc[(sig - mu) & (D - 1)] = p;
                                }
                            }, A.dbg, mark);
            }
            __syncthreads();   // Fc complete; X2 free
            // Zak' tile: slot s8 = column j0 + s8, lane t = h8: Fc(t + 16 k)
#pragma unroll
            for (int k = 0; k < R1; ++k) pre[k] = F[s8 * K::FS + h8 + 16 * k];
            float2* dst = A.out + (int64_t)w * L + j0 + s8;
            dft_tile<D>(pre, tw, X2, s8, h8, s8, h8, none, none,
                        [&](int r, const float2* y) {
#pragma unroll
                            for (int m2 = 0; m2 < 16; ++m2) {
                                const int s = 16 * r + h8 + R1 * m2;
                                __stcs(dst + (int64_t)s * M, conjf2(y[m2]));
                            }
                        }, A.dbg, mark);
            // the eight ring rows this job read are dead: drop them from L2
            constexpr int LPR = N / 16;   // 128-byte lines per row
            for (int e = tid; e < AC * LPR; e += K::NT)
                asm volatile("discard.global.L2 [%0], 128;" ::"l"(wsl + (int64_t)(j0 + e / LPR) * N + (e % LPR) * 16)
                             : "memory");
            if (tid == 0) pend = doneA + slot;
        }
    }
    __syncthreads();
    if (tid == 0 && pend) {
        signal_release(pend);
    }
}

}  // namespace v7
}  // namespace nsdgt
