// zak_rr.cuh -- register-resident all-u Zak kernel for d = 180, q = 4, p = 1 (config 4's
// inner separable DGT after the frequency shear, Alg. 1 lines 23-27 with the Zak /
// factorisation steps of Eqs. (zak)-(phi), §3.1).  Same result as zak_ct_kernel<T, 180, 4, ...>
// (gather with the chirp on load, DFT_180 over s, the q products with the window factors, one
// DFT_180 per product, scatter), but each DFT_180 is two register passes, 180 = 12 x 15:
//
//   DFT 1 (s -> nu), s = 12 a + b, nu = k1 + 15 k2:
//     Phi(k1 + 15 k2) = sum_b W12^{b k2} [ W180^{b k1} sum_a v(12 a + b) W15^{a k1} ]
//     "b-thread" (b < 12): gathers its 15 samples straight from global memory, DFT_15,
//     twiddle, one shared-memory exchange; "k1-thread" (k1 < 15): DFT_12 -> 12 values of Phi.
//   DFT 2 (nu -> tau) per u, nu = k1 + 15 k2, tau = t2 + 12 t1:
//     Y(t2 + 12 t1) = sum_k1 W15^{k1 t1} [ W180^{k1 t2} sum_k2 Yb(k1 + 15 k2) W12^{k2 t2} ]
//     the k1-thread multiplies its Phi values by the window factors and runs DFT_12 in
//     registers (its inputs are exactly the Phi it holds -- no exchange between the DFTs),
//     one exchange, the "t2-thread" runs DFT_15 and scatters to the intermediate directly.
//
// Shared memory carries 3 exchanges per u-pair instead of the Stockham engine's 2 passes per
// DFT plus the gather / product / scatter round trips (10 vs 33 transfers of a 180-vector per
// column), and 5 barriers per CTA instead of 13.  RBC consecutive residues per CTA (rr fastest
// in every thread mapping: 16 * RBC-byte runs in global memory, conflict-free exchanges).
// Included inside namespace nsdgt by dgt.cu, after ZakArgs.
#pragma once

#ifndef NSDGT_ZRR_MINB
#define NSDGT_ZRR_MINB 4
#endif
constexpr int kZrrMinB = NSDGT_ZRR_MINB;   // CTAs per SM the register budget is sized for
// dynamic shared memory of zak_rr_kernel<T, 8, *>: the twiddle table and two exchange buffers
template <typename T> constexpr int zrr_smem() { return (180 + 2 * 8 * 180) * (int)sizeof(cx<T>); }

template <typename T, int RBC, int MINB>
__global__ void __launch_bounds__(16 * RBC, MINB) zak_rr_kernel(ZakArgs A) {
    constexpr int D = 180, Q = 4, NT = 16 * RBC;
    using C = cx<T>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C* tws = (C*)smem_raw;              // W180^e, e < 180
    C* X0 = tws + D;                    // exchange buffers, RBC D each
    C* X1 = X0 + RBC * D;
    const int c = (int)A.c;
    const int nrb = c / RBC;
    const int rblk = blockIdx.x % nrb, l = blockIdx.x / nrb;
    const int64_t w = blockIdx.y;
    const int r0 = rblk * RBC;
    const int tid = threadIdx.x;
    const int rr = tid % RBC, hi = tid / RBC;   // hi: b (pass 15) or k1 (pass 12)
    static_assert((12 * RBC) % 32 == 0, "the b-threads are whole warps (named barrier 1)");
    // ---- DFT 1, pass 1 (b-threads): gather v(12 a + b), a < 15, with the chirp; DFT_15 ----
    if (hi < 12) {
        const int b = hi;
        const C* fc = (const C*)A.f + w * A.L;
        const T* fr = (const T*)A.f + w * A.L;
        const C* __restrict__ chirp = (const C*)A.chirp;
        const int x0 = r0 + rr + c * (l + Q * b);   // s = b; each a adds 12 Q c
        const int xs = 12 * Q * c;
        C v[15];
#pragma unroll
        for (int a = 0; a < 15; ++a) v[a] = A.real_in ? mk<T>(fr[x0 + a * xs], T(0)) : fc[x0 + a * xs];
        if (chirp) {
#pragma unroll
            for (int a = 0; a < 15; ++a) v[a] = cmul(v[a], __ldg(chirp + x0 + a * xs));
        }
        // the twiddle table, written by the b-threads only (named barrier 1 among them)
        for (int i = tid; i < D; i += 12 * RBC) tws[i] = ((const C*)A.tw)[i];
        dft_pq<T, 3, 5, 180>(v, 12);
        asm volatile("bar.sync 1, %0;" ::"r"(12 * RBC) : "memory");
#pragma unroll
        for (int k1 = 0; k1 < 15; ++k1) X0[(b * 15 + k1) * RBC + rr] = k1 ? cmul(v[k1], tws[b * k1]) : v[k1];
    }
    __syncthreads();
    // ---- DFT 1, pass 2 (k1-threads): DFT_12 -> Phi(k1 + 15 k2), k2 < 12, kept in registers ----
    C ph[12];
    const int k1 = hi;
    if (hi < 15) {
#pragma unroll
        for (int b = 0; b < 12; ++b) ph[b] = X0[(b * 15 + k1) * RBC + rr];
        dft_pq<T, 4, 3, 180>(ph, 15);
    }
    const C* __restrict__ G = (const C*)A.G + (int64_t)(r0 + rr) * Q * D;
    C* Cw = (C*)A.C + w * A.iM * Q * D;
    const int jbase = r0 + c * (l % Q);
    const int iM = (int)A.iM;
#pragma unroll 1
    for (int u = 0; u < Q; ++u) {
        C* Xu = (u & 1) ? X0 : X1;
        // ---- DFT 2, pass 1 (k1-threads): products with the window factors, DFT_12, twiddle ----
        if (hi < 15) {
            C y[12];
#pragma unroll
            for (int k2 = 0; k2 < 12; ++k2) y[k2] = __ldg(G + u * D + k1 + 15 * k2);
#pragma unroll
            for (int k2 = 0; k2 < 12; ++k2) y[k2] = cmul(ph[k2], y[k2]);
            dft_pq<T, 4, 3, 180>(y, 15);
#pragma unroll
            for (int t2 = 0; t2 < 12; ++t2) Xu[(k1 * 12 + t2) * RBC + rr] = t2 ? cmul(y[t2], tws[k1 * t2]) : y[t2];
        }
        __syncthreads();
        // ---- DFT 2, pass 2 (t2-threads): DFT_15 -> Y(t2 + 12 t1), scatter T_r(l, u; tau) ----
        if (hi < 12) {
            const int t2 = hi;
            C z[15];
#pragma unroll
            for (int k = 0; k < 15; ++k) z[k] = Xu[(k * 12 + t2) * RBC + rr];
            dft_pq<T, 3, 5, 180>(z, 12);
            // n = (l - u - q tau) mod N: kappa = (l - u) mod q, n' = (-tau - [l < u]) mod d
            const int kappa = (l - u + Q) % Q;
            const int off = l < u ? 1 : 0;
#pragma unroll
            for (int t1 = 0; t1 < 15; ++t1) {
                const int tau = t2 + 12 * t1;
                int np = D - tau - off;
                if (np >= D) np -= D;
                if (np < 0) np += D;
                if (A.cnj) Cw[(int64_t)(kappa + Q * np) * iM + jbase + rr] = z[t1];
                else Cw[((jbase + rr) * Q + kappa) * D + np] = z[t1];
            }
        }
    }
}

