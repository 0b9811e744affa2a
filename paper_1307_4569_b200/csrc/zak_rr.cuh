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
// Shared memory carries one exchange per DFT (5 per column: 10 transfers of a 180-vector
// against 33 for the Stockham engine's two passes per DFT plus the gather / product / scatter
// round trips) and 5 barriers per CTA instead of 13.  RBC consecutive residues per CTA (rr
// fastest in every thread mapping: 16 * RBC-byte runs in global memory, conflict-free
// exchanges).
//
// Also here: front_f4096_kernel (the frequency shear's length-L FFT for L = 180 x 4096 as
// 4096-point DFTs of the 180 residues; its adjoint with ADJ), zak_rr0_kernel (zak_rr with the
// FFT's DFT_180 over the residues in front: six DFT_180s per column, still one exchange each)
// and zak_rr0_adj_kernel (the adjoint of zak_rr0, for the synthesis).
// Included inside namespace nsdgt by dgt.cu, after ZakArgs.
#pragma once

#ifndef NSDGT_ZRR_MINB
#define NSDGT_ZRR_MINB 4
#endif
constexpr int kZrrMinB = NSDGT_ZRR_MINB;   // CTAs per SM the register budget is sized for
#ifndef NSDGT_ZRR0_MINB
#define NSDGT_ZRR0_MINB 3
#endif
constexpr int kZrr0MinB = NSDGT_ZRR0_MINB;
// dynamic shared memory of zak_rr_kernel<T, 8, *>: the twiddle table and two exchange buffers
template <typename T> constexpr int zrr_smem() { return (180 + 2 * 8 * 180) * (int)sizeof(cx<T>); }

template <typename T, int RBC, int MINB>
__global__ void __launch_bounds__(16 * RBC, MINB) zak_rr_kernel(ZakArgs A) {
    constexpr int D = 180, Q = 4;
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
    pdl_trigger();
    pdl_wait();
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


// ---------------------------------------------------------------------------------------
// Frequency-shear front end for L = 180 x 4096 (config 4) without cuFFT: the length-L FFT of
// Alg. 1 line 23 (f^ = fft(pchirp(L, s1) f)) split as l = 180 q + r, nu = x + 4096 j:
//   f^(x + 4096 j) = sum_r W_180^{r j} H(r, x),   H(r, x) = W_L^{r x} sum_q f(180 q + r) W_4096^{q x}
// front_f4096_kernel computes H (one CTA per residue r and signal: a 4096-point DFT in three
// register radix-16 passes, the W_L^{r x} twiddle, contiguous stores H[w][r][x]);
// zak_rr0_kernel runs the DFT_180 over r as one more register pass pair in front of the Zak
// kernel's two DFTs, so f^ never exists in memory.
// ---------------------------------------------------------------------------------------
struct FrontArgs {
    const void* f;      // [W][L] input (complex, or real with real_in)
    int real_in;
    const void* pre;    // [L] pchirp(L, s1) multiplier (nullable)
    void* H;            // [W][180][4096] output
    const void* tw;     // W_4096^k, k < 4096
    const void* twL;    // W_L^e, e < 180 * 256
    int64_t L;
};
constexpr int kFrontElems = 256 * 17;   // exchange buffer per residue (elements), padded for pass 3
#ifndef NSDGT_FRONT_RES
#define NSDGT_FRONT_RES 2
#endif
constexpr int kFrontRes = NSDGT_FRONT_RES;   // residues per front_f4096 CTA
#ifndef NSDGT_FRONT_MINB
#define NSDGT_FRONT_MINB (2 / NSDGT_FRONT_RES)
#endif
constexpr int kFrontMinB = NSDGT_FRONT_MINB;   // CTAs per SM the register budget is sized for
constexpr int front_smem(int esz) { return (kFrontRes * (kFrontElems + 4)) * esz; }

// v[k] *= b0 * w^k, k < 16 (w^k from three squarings and products: <= 6 roundings)
template <typename C>
__device__ __forceinline__ void twiddle16b(C* v, C b0, C w1) {
    const C w2 = cmul(w1, w1), w4 = cmul(w2, w2), w8 = cmul(w4, w4);
    C p[16];
    p[0] = b0; p[1] = cmul(b0, w1); p[2] = cmul(b0, w2); p[4] = cmul(b0, w4); p[8] = cmul(b0, w8);
    p[3] = cmul(p[1], w2); p[5] = cmul(p[1], w4); p[6] = cmul(p[2], w4); p[7] = cmul(p[3], w4);
#pragma unroll
    for (int k = 9; k < 16; ++k) p[k] = cmul(p[k - 8], w8);
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = cmul(v[k], p[k]);
}

// v[k] *= w^k, k < 16
template <typename C>
__device__ __forceinline__ void twiddle16(C* v, C w1) {
    const C w2 = cmul(w1, w1), w4 = cmul(w2, w2), w8 = cmul(w4, w4);
    C p[16];
    p[1] = w1; p[2] = w2; p[4] = w4; p[8] = w8;
    p[3] = cmul(w1, w2); p[5] = cmul(w1, w4); p[6] = cmul(w2, w4); p[7] = cmul(p[3], w4);
#pragma unroll
    for (int k = 9; k < 16; ++k) p[k] = cmul(p[k - 8], w8);
#pragma unroll
    for (int k = 1; k < 16; ++k) v[k] = cmul(v[k], p[k]);
}

// 4096-point DFT, q = q0 + 16 q1 + 256 q2 -> x = x0 + 16 x1 + 256 x2:
//   pass 1, lane (q0, q1): A = W_256^{q1 x0} sum_q2 W_16^{q2 x0} g(q)
//   pass 2, lane (q0, x0): B = W_4096^{q0 (x0 + 16 x1)} sum_q1 W_16^{q1 x1} A
//   pass 3, lane (x0, x1): X(x0 + 16 x1 + 256 x2) = sum_q0 W_16^{q0 x2} B     (lane = x mod 256)
// RES residues per CTA of 256 RES threads, lane = (t, h) with h = tid mod RES fastest: the
// RES samples f(180 q + r0 + h) of a lane pair are adjacent (RES = 2: 32-byte sectors used
// whole instead of half), each residue has its own exchange buffer (offset by 4 elements so the
// two halves of a quarter warp hit different banks).
// ADJ (synthesis, the adjoint of the front end): input h(r, x) = conj(H'(r, x)) as written by
// zak_rr0_adj_kernel, contiguous in x; the W_L^{r x} twiddle on load, the same three passes
// (now over x -> q) and f(180 q + r) = conj(X(q)) conj(pchirp(L, s1)) stored at stride 180
// (the unnormalised inverse DFT of Alg. 1 line 23's FFT, as conj(DFT(conj(.)))).
template <typename T, int MINB, int RES, bool ADJ = false>
__global__ void __launch_bounds__(256 * RES, MINB) front_f4096_kernel(FrontArgs A) {
    using C = cx<T>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int tid = threadIdx.x % (256 * RES) / RES;   // t
    const int h = threadIdx.x % RES;
    C* S = (C*)smem_raw + h * (kFrontElems + 4);
    const int r = blockIdx.x * RES + h;
    const int64_t w = blockIdx.y;
    const C* __restrict__ tw = (const C*)A.tw;
    pdl_trigger();
    pdl_wait();   // f may come from a preceding kernel; H may still be read by the previous Zak kernel
    C v[16];
    if constexpr (ADJ) {
        const C* hr = (const C*)A.f + w * A.L + (int64_t)r * 4096;
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = hr[tid + 256 * i];
        twiddle16b(v, __ldg((const C*)A.twL + r * tid), __ldg((const C*)A.twL + 256 * r));
    } else {
        const int64_t base = w * A.L + r;
        const C* __restrict__ pre = (const C*)A.pre;
#pragma unroll
        for (int q2 = 0; q2 < 16; ++q2) {
            const int l = 180 * (tid + 256 * q2);
            v[q2] = A.real_in ? mk<T>(((const T*)A.f)[base + l], T(0)) : ((const C*)A.f)[base + l];
        }
        if (pre) {
#pragma unroll
            for (int q2 = 0; q2 < 16; ++q2) v[q2] = cmul(v[q2], __ldg(pre + r + 180 * (tid + 256 * q2)));
        }
    }
    dft16<T>(v);
    {
        const int q1 = tid >> 4;
        if (q1) twiddle16(v, __ldg(tw + 16 * q1));
    }
#pragma unroll
    for (int x0 = 0; x0 < 16; ++x0) S[x0 * 256 + tid] = v[x0];
    __syncthreads();
    {
        const int q0 = tid & 15, x0 = tid >> 4;
#pragma unroll
        for (int q1 = 0; q1 < 16; ++q1) v[q1] = S[x0 * 256 + q0 + 16 * q1];
        __syncthreads();
        dft16<T>(v);
        if (q0) twiddle16b(v, __ldg(tw + q0 * x0), __ldg(tw + 16 * q0));
        // B(q0, x1, x0) at (x1 * 16 + x0) * 17 + q0
#pragma unroll
        for (int x1 = 0; x1 < 16; ++x1) S[(x1 * 16 + x0) * 17 + q0] = v[x1];
    }
    __syncthreads();
#pragma unroll
    for (int q0 = 0; q0 < 16; ++q0) v[q0] = S[tid * 17 + q0];
    dft16<T>(v);
    if constexpr (ADJ) {
        // f(180 (tid + 256 k) + r) = conj(X) conj(pre): lane pairs (h = 0, 1) write 32 bytes
        const C* __restrict__ pre = (const C*)A.pre;
        C* fo = (C*)A.H + w * A.L + r;
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            const int l = 180 * (tid + 256 * k);
            C y = mk<T>(v[k].x, -v[k].y);
            if (pre) y = cmulc(y, __ldg(pre + r + l));
            fo[l] = y;
        }
        return;
    }
    // H(r, x) = W_L^{r x} X(x), x = tid + 256 x2: W_L^{r tid} (W_L^{256 r})^{x2}
    twiddle16b(v, __ldg((const C*)A.twL + r * tid), __ldg((const C*)A.twL + 256 * r));
    C* H = (C*)A.H + w * A.L + (int64_t)r * 4096;
#pragma unroll
    for (int x2 = 0; x2 < 16; ++x2) H[tid + 256 * x2] = v[x2];
}

// zak_rr_kernel with the front end's DFT_180 over r in front (config 4 without cuFFT):
//   stage 0, r = 12 a + b -> j = p + 15 k:  f^(x + 4096 j), x = r0 + rr + c l
//     b-thread: DFT_15 over a, W180^{b p}; exchange; p-thread: DFT_12 over b; chirp on j
//   stage 1 (Zak DFT), j = p + 15 k -> nu = t + 12 e:
//     p-thread: DFT_12 over k, W180^{p t}; exchange; t-thread: DFT_15 over p -> Phi(t + 12 e)
//   stage 2 per u (factor DFT), nu = t + 12 e -> tau = p + 15 k:
//     t-thread: products, DFT_15 over e, W180^{t p}; exchange; p-thread: DFT_12 over t, scatter
// 6 barriers per CTA; Phi (15 values) stays in the t-threads' registers.
template <typename T, int RBC, int MINB>
__global__ void __launch_bounds__(16 * RBC, MINB) zak_rr0_kernel(ZakArgs A) {
    constexpr int D = 180, Q = 4;
    using C = cx<T>;
    static_assert((12 * RBC) % 32 == 0, "the 12-lane groups are whole warps (named barrier 1)");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C* tws = (C*)smem_raw;
    C* X0 = tws + D;
    C* X1 = X0 + RBC * D;
    const int c = (int)A.c;
    const int nrb = c / RBC;
    const int rblk = blockIdx.x % nrb, l = blockIdx.x / nrb;
    const int64_t w = blockIdx.y;
    const int r0 = rblk * RBC;
    const int tid = threadIdx.x;
    const int rr = tid % RBC, hi = tid / RBC;
    const int x = r0 + rr + c * l;            // column of H / f^ (x < 4096)
    pdl_trigger();
    pdl_wait();
    // ---- stage 0, pass 1 (b-threads): H(12 a + b, x), DFT_15 over a ----
    if (hi < 12) {
        const int b = hi;
        const C* Hc = (const C*)A.f + w * A.L + (int64_t)b * 4096 + x;
        C v[15];
#pragma unroll
        for (int a = 0; a < 15; ++a) v[a] = Hc[a * 12 * 4096];
        for (int i = tid; i < D; i += 12 * RBC) tws[i] = ((const C*)A.tw)[i];
        dft_pq<T, 3, 5, 180>(v, 12);
        asm volatile("bar.sync 1, %0;" ::"r"(12 * RBC) : "memory");
#pragma unroll
        for (int p = 0; p < 15; ++p) X0[(b * 15 + p) * RBC + rr] = p ? cmul(v[p], tws[b * p]) : v[p];
    }
    __syncthreads();
    // ---- stage 0, pass 2 + stage 1, pass 1 (p-threads) ----
    if (hi < 15) {
        const int p = hi;
        C e[12];
#pragma unroll
        for (int b = 0; b < 12; ++b) e[b] = X0[(b * 15 + p) * RBC + rr];
        dft_pq<T, 4, 3, 180>(e, 15);     // e[k] = f^(x + 4096 (p + 15 k))
        const C* __restrict__ chirp = (const C*)A.chirp;
        if (chirp) {
#pragma unroll
            for (int k = 0; k < 12; ++k) e[k] = cmul(e[k], __ldg(chirp + x + 4096 * (p + 15 * k)));
        }
        dft_pq<T, 4, 3, 180>(e, 15);     // over k -> t
#pragma unroll
        for (int t = 0; t < 12; ++t) X1[(p * 12 + t) * RBC + rr] = t ? cmul(e[t], tws[p * t]) : e[t];
    }
    __syncthreads();
    // ---- stage 1, pass 2 (t-threads): Phi(t + 12 e), e < 15 ----
    C ph[15];
    if (hi < 12) {
        const int t = hi;
#pragma unroll
        for (int p = 0; p < 15; ++p) ph[p] = X1[(p * 12 + t) * RBC + rr];
        dft_pq<T, 3, 5, 180>(ph, 12);
    }
    const C* __restrict__ G = (const C*)A.G + (int64_t)(r0 + rr) * Q * D;
    C* Cw = (C*)A.C + w * A.iM * Q * D;
    const int jbase = r0 + c * (l % Q);
    const int iM = (int)A.iM;
#pragma unroll 1
    for (int u = 0; u < Q; ++u) {
        C* Xu = (u & 1) ? X1 : X0;
        if (hi < 12) {
            const int t = hi;
            C y[15];
#pragma unroll
            for (int e = 0; e < 15; ++e) y[e] = __ldg(G + u * D + t + 12 * e);
#pragma unroll
            for (int e = 0; e < 15; ++e) y[e] = cmul(ph[e], y[e]);
            dft_pq<T, 3, 5, 180>(y, 12);  // over e -> p
#pragma unroll
            for (int p = 0; p < 15; ++p) Xu[(t * 15 + p) * RBC + rr] = p ? cmul(y[p], tws[t * p]) : y[p];
        }
        __syncthreads();
        if (hi < 15) {
            const int p = hi;
            C z[12];
#pragma unroll
            for (int t = 0; t < 12; ++t) z[t] = Xu[(t * 15 + p) * RBC + rr];
            dft_pq<T, 4, 3, 180>(z, 15);  // over t -> k: Y(p + 15 k)
            const int kappa = (l - u + Q) % Q;
            const int off = l < u ? 1 : 0;
#pragma unroll
            for (int k = 0; k < 12; ++k) {
                const int tau = p + 15 * k;
                int np = D - tau - off;
                if (np >= D) np -= D;
                if (np < 0) np += D;
                if (A.cnj) Cw[(int64_t)(kappa + Q * np) * iM + jbase + rr] = z[k];
                else Cw[((jbase + rr) * Q + kappa) * D + np] = z[k];
            }
        }
    }
}

// Adjoint of zak_rr0_kernel (synthesis, config 4): C' [n][j] -> h(r, x) = conj(H'(r, x)), kept
// conjugated so that every DFT is a forward one (conj(DFT^H(y)) = DFT(conj y)):
//   S2 per u, tau = p + 15 k -> nu = t + 12 e: gather conj(T'_u(tau)) through the forward
//      scatter map, p-thread DFT_12 over k, W180^{p t}, exchange, t-thread DFT_15 over p;
//      acc(nu) += y_u(nu) G_u(nu) in the t-thread's registers (= conj(Phi'(nu)))
//   S1 nu = t + 12 e -> j = p + 15 k: t-thread DFT_15 over e, W180^{t p}, exchange, p-thread
//      DFT_12 over t; times the chirp P_{-s0}(x + 4096 j)  (= conj of the adjoint's value)
//   S0 j = p + 15 k -> r = b + 12 a: p-thread DFT_12 over k, W180^{p b}, exchange, b-thread
//      DFT_15 over p; h(b + 12 a, x) stored [w][r][x] for front_f4096_kernel<..., ADJ>.
template <typename T, int RBC, int MINB>
__global__ void __launch_bounds__(16 * RBC, MINB) zak_rr0_adj_kernel(ZakArgs A, void* hout) {
    constexpr int D = 180, Q = 4;
    using C = cx<T>;
    static_assert((12 * RBC) % 32 == 0, "the 12-lane groups are whole warps");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C* tws = (C*)smem_raw;
    C* X0 = tws + D;
    C* X1 = X0 + RBC * D;
    const int c = (int)A.c;
    const int nrb = c / RBC;
    const int rblk = blockIdx.x % nrb, l = blockIdx.x / nrb;
    const int64_t w = blockIdx.y;
    const int r0 = rblk * RBC;
    const int tid = threadIdx.x;
    const int rr = tid % RBC, hi = tid / RBC;
    const int x = r0 + rr + c * l;
    pdl_trigger();
    for (int i = tid; i < D; i += 16 * RBC) tws[i] = ((const C*)A.tw)[i];
    pdl_wait();
    __syncthreads();
    const C* __restrict__ G = (const C*)A.G + (int64_t)(r0 + rr) * Q * D;
    const C* Cw = (const C*)A.C + w * A.iM * Q * D;
    const int jbase = r0 + c * (l % Q);
    const int iM = (int)A.iM;
    C acc[15];
#pragma unroll
    for (int e = 0; e < 15; ++e) acc[e] = mk<T>(T(0), T(0));
#pragma unroll 1
    for (int u = 0; u < Q; ++u) {
        C* Xu = (u & 1) ? X1 : X0;
        if (hi < 15) {
            const int p = hi;
            const int kappa = (l - u + Q) % Q;
            const int off = l < u ? 1 : 0;
            C z[12];
#pragma unroll
            for (int k = 0; k < 12; ++k) {
                const int tau = p + 15 * k;
                int np = D - tau - off;
                if (np >= D) np -= D;
                if (np < 0) np += D;
                const C v = A.cnj ? Cw[(int64_t)(kappa + Q * np) * iM + jbase + rr] : Cw[((jbase + rr) * Q + kappa) * D + np];
                z[k] = mk<T>(v.x, -v.y);
            }
            dft_pq<T, 4, 3, 180>(z, 15);   // over k -> t
#pragma unroll
            for (int t = 0; t < 12; ++t) Xu[(p * 12 + t) * RBC + rr] = t ? cmul(z[t], tws[p * t]) : z[t];
        }
        __syncthreads();
        if (hi < 12) {
            const int t = hi;
            C y[15];
#pragma unroll
            for (int p = 0; p < 15; ++p) y[p] = Xu[(p * 12 + t) * RBC + rr];
            dft_pq<T, 3, 5, 180>(y, 12);   // over p -> e: y_u(t + 12 e)
#pragma unroll
            for (int e = 0; e < 15; ++e) acc[e] = acc[e] + cmul(y[e], __ldg(G + u * D + t + 12 * e));
        }
    }
    // ---- S1: acc(t + 12 e) -> j = p + 15 k (X0 was last read in u = 2, before u = 3's barrier) ----
    if (hi < 12) {
        const int t = hi;
        dft_pq<T, 3, 5, 180>(acc, 12);     // over e -> p
#pragma unroll
        for (int p = 0; p < 15; ++p) X0[(t * 15 + p) * RBC + rr] = p ? cmul(acc[p], tws[t * p]) : acc[p];
    }
    __syncthreads();
    if (hi < 15) {
        const int p = hi;
        C e2[12];
#pragma unroll
        for (int t = 0; t < 12; ++t) e2[t] = X0[(t * 15 + p) * RBC + rr];
        dft_pq<T, 4, 3, 180>(e2, 15);      // over t -> k: j = p + 15 k
        const C* __restrict__ chirp = (const C*)A.chirp;
        if (chirp) {
#pragma unroll
            for (int k = 0; k < 12; ++k) e2[k] = cmul(e2[k], __ldg(chirp + x + 4096 * (p + 15 * k)));
        }
        // ---- S0: j = p + 15 k -> r = b + 12 a ----
        dft_pq<T, 4, 3, 180>(e2, 15);      // over k -> b
#pragma unroll
        for (int b = 0; b < 12; ++b) X1[(p * 12 + b) * RBC + rr] = b ? cmul(e2[b], tws[p * b]) : e2[b];
    }
    __syncthreads();
    if (hi < 12) {
        const int b = hi;
        C hv[15];
#pragma unroll
        for (int p = 0; p < 15; ++p) hv[p] = X1[(p * 12 + b) * RBC + rr];
        dft_pq<T, 3, 5, 180>(hv, 12);      // over p -> a: r = b + 12 a
        C* Ho = (C*)hout + w * A.L + (int64_t)b * 4096 + x;
#pragma unroll
        for (int a = 0; a < 15; ++a) Ho[a * 12 * 4096] = hv[a];
    }
}
