// tiny.cuh -- the whole shear algorithm (Alg. 1, lines 1-31) for one short signal in
// one CTA: BASELINE config 1 (L = 240) and other lattices whose tables and buffers fit shared
// memory.  The chunked path runs a pre-chirp kernel, cuFFT and two kernels per chunk, each
// starting with cold loads of its tables (about 35 us of dependent launches and DRAM round
// trips for 360 coefficients); here every table is fetched into shared memory in one round at
// the start and the steps follow in one CTA, each batched over all residues and columns:
//   0. f (real input promoted), times pchirp(L, s1) in the frequency shear (Alg. 1 line 23)
//   1. F-branch: f^ = DFT_L (Stockham engine, fft_smem.cuh)
//   2. Zak gather x = r + c ((k q + p l + s p q) mod L/c) with the chirp on load, all (l, r, k)
//   3. DFT_d over s of the q c p sequences
//   4. Y(l, r, u; nu) = sum_k Phi(l, r, k; nu) G(r, u, k; nu) for all (l, r, u)   (Eq. phi)
//   5. DFT_d over nu of the q c q products, scatter T_r(l, u; tau) to C[n][j]:
//      j = r + c ((l p) mod q), n = kappa + q n', kappa = (l - u) mod q, n' = (-tau - [l < u]) mod d
//   6. DFT over j (iM) of the iN columns
//   7. output: T-branch c[(m - rot n) mod M][n] = E(n) X(m, n); F-branch the Alg. 1 remap
//      with its phase (the same per-coefficient residues as out_kernel's fb_* helpers)
// Included inside namespace nsdgt by dgt.cu after the output kernels.
#pragma once

struct TinyArgs {
    const void* f;        // [W][L] input (complex, or real with real_in)
    int real_in;
    const void* pre;      // F-branch pchirp(L, s1) on f (nullable)
    const void* chirp;    // chirp on the Zak load (nullable): T-branch P_{s1}, F-branch P_{-s0}
    const void* G;        // window factors [c][q][p][d]
    const void* twL;      // W_L^k, k < L (F-branch)
    const void* twd;      // W_d^k
    const void* twm;      // W_iM^k
    const void* odst;           // F-branch: destination c index (uint32) of X[n iM + kc] (plan table)
    const void* oph;            // F-branch: its Alg. 1 phase
    Radices rdL, rdd, rdm;
    int L, c, d, p, q, iM, iN;
    OutArgs B;            // output constants (out, M, N, E / rot or the F-branch remap)
};

// Plan time (F-branch): the output remap of every X[n iM + kc] -- destination index and phase,
// the same residues fb_column computes per coefficient (fb_col, fb_iter, fb_dest).
template <typename T>
__global__ void k_tiny_remap(OutArgs B, unsigned int* odst, cx<T>* oph, int iM, int iN) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= iM * iN) return;
    const int kc = i % iM, n = i / iM;
    const FbCol cc = fb_col(B, (unsigned long long)n);
    const FbIter<cx<T>> it = fb_iter<cx<T>>(B, cc, kc ? (unsigned long long)B.Nr - (unsigned long long)kc : 0ull);
    size_t dst;
    cx<T> ph;
    fb_dest(B, it, &dst, &ph);
    odst[i] = (unsigned int)dst;
    oph[i] = ph;
}

// shared-memory elements of tiny_kernel (also the host's fit test)
__host__ __device__ inline int64_t tiny_elems(int64_t L, int64_t q, int64_t p, int64_t d, int64_t iM, bool freq) {
    const int64_t LQ = L * q / p;   // products / intermediate (= iM iN)
    const int64_t LX = LQ > L ? LQ : L;   // work buffers: the Zak gather (L) and the products (LQ)
    // + F-branch: W_L, the output phases (LQ) and destinations (LQ x 4 bytes, counted as LQ / 2
    //   16-byte or LQ / 2 8-byte elements rounded up)
    return 2 * L + 2 * LX + L /* G */ + L /* chirp */ + (freq ? L + LQ + (LQ + 1) / 2 : 0) + d + iM;
}

#ifdef NSDGT_TINY_TRACE
// experiment builds only (tools): %globaltimer at the phase boundaries of block 0
__device__ unsigned long long g_tiny_trace[16];
#define TINY_MARK(k)                                                                            \
    do {                                                                                        \
        if (blockIdx.x == 0 && threadIdx.x == 0) {                                              \
            unsigned long long t_;                                                              \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                              \
            g_tiny_trace[k] = t_;                                                               \
        }                                                                                       \
    } while (0)
#else
#define TINY_MARK(k) do { } while (0)
#endif

// One Stockham pass of compile-time radix R on nseq sequences of compile-time length N (the
// one-CTA path's compile-time variant): R = 15 runs as 3 x 5 in registers (inner twiddles
// W_15 = W_180^12 from the constant table), other radices as register butterflies.
template <typename T, int N, int R, int NS>
__device__ __forceinline__ void tstage(const cx<T>* __restrict__ in, cx<T>* __restrict__ out, int nseq,
                                       const cx<T>* __restrict__ tw) {
    using C = cx<T>;
    constexpr int nb = N / R, tstep = N / (NS * R);
    for (int t = threadIdx.x; t < nb * nseq; t += blockDim.x) {
        const int seq = t / nb, j = t - seq * nb;
        const int k = j % NS;
        const C* src = in + seq * N;
        C* dst = out + seq * N;
        C v[R];
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = src[j + r * nb];
        if constexpr (NS > 1) {
            const C w1 = tw[k * tstep];
            C wr = w1;
            v[1] = cmul(v[1], w1);
#pragma unroll
            for (int r = 2; r < R; ++r) {
                wr = cmul(wr, w1);
                v[r] = cmul(v[r], wr);
            }
        }
        if constexpr (R == 15) dft_pq<T, 3, 5, 180>(v, 12);
        else dft_fixed<T, R>(v);
        const int base = (j / NS) * NS * R + k;
#pragma unroll
        for (int r = 0; r < R; ++r) dst[base + r * NS] = v[r];
    }
}

// SL > 0: a compile-time lattice shape (L, c, d, p, q) = (SL, SC, SD, SP, SQ) -- config 1's
// (240, 5, 8, 2, 3): every index divides by constants and the DFTs run as compile-time passes
// (DFT_240 = 16 x 15, DFT_8, DFT_15 = 3 x 5 in one pass) instead of the runtime-radix engine.
template <typename T, int SL = 0, int SC = 0, int SD = 0, int SP = 0, int SQ = 0>
__global__ void __launch_bounds__(256) tiny_kernel(const __grid_constant__ TinyArgs A) {
    using C = cx<T>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr bool CT = SL > 0;
    const int L = CT ? SL : A.L, c = CT ? SC : A.c, d = CT ? SD : A.d, p = CT ? SP : A.p, q = CT ? SQ : A.q;
    const int iM = CT ? SC * SQ : A.iM, iN = CT ? SQ * SD : A.iN;
    const bool freq = A.B.branch == DGT_BRANCH_FREQ;
    const int LQ = L / p * q;
    const int LX = LQ > L ? LQ : L;
    C* sF = (C*)smem_raw;        // L
    C* sF2 = sF + L;             // L
    C* sX = sF2 + L;             // max(L, LQ)
    C* sY = sX + LX;             // max(L, LQ)
    C* sG = sY + LX;             // L
    C* sCh = sG + L;             // L
    C* sTwL = sCh + L;           // L (F-branch)
    C* sPh = sTwL + (freq ? L : 0);            // LQ (F-branch)
    unsigned int* sDst = (unsigned int*)(sPh + (freq ? LQ : 0));   // LQ (F-branch)
    C* sTwd = (C*)((char*)sPh + (freq ? (int64_t)LQ * sizeof(C) + (LQ + 1) / 2 * sizeof(C) : 0));
    C* sTwm = sTwd + d;
    const int tid = threadIdx.x, nt = blockDim.x;
    const int64_t w = blockIdx.x;
    TINY_MARK(0);
    pdl_trigger();
    // the output-stage tables go to L2 now (read once at the end)
    if (tid == 0) {
        const char* e = freq ? (const char*)A.B.ptab : (const char*)A.B.E;
        if (!e) e = (const char*)A.G;   // (no output table: a harmless re-fetch)
        const int64_t eb = freq ? 2 * A.B.N * (int64_t)sizeof(C) : A.B.N * (int64_t)sizeof(C);
        for (int64_t o = 0; o < eb; o += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(e + o));
        if (!freq)
            for (int64_t o = 0; o < A.B.N * 4; o += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"((const char*)A.B.rot + o));
    }
    // ---- 0. one round of loads: f (x pre), G, chirp, twiddles ----
    {
        const C* __restrict__ pre = (const C*)A.pre;
        const C* __restrict__ chirp = (const C*)A.chirp;
        // the plan's tables first (never written by a kernel of the stream), then -- once the
        // predecessor grid is complete (PDL) -- the input, which a preceding kernel may produce
        for (int i = tid; i < L; i += nt) {
            sG[i] = __ldg((const C*)A.G + i);
            sCh[i] = chirp ? __ldg(chirp + i) : mk<T>(T(1), T(0));
            if (freq) sTwL[i] = __ldg((const C*)A.twL + i);
        }
        for (int i = tid; i < d; i += nt) sTwd[i] = __ldg((const C*)A.twd + i);
        for (int i = tid; i < iM; i += nt) sTwm[i] = __ldg((const C*)A.twm + i);
        if (freq && A.odst) {
            for (int i = tid; i < LQ; i += nt) {
                sPh[i] = __ldg((const C*)A.oph + i);
                sDst[i] = __ldg((const unsigned int*)A.odst + i);
            }
        }
        pdl_wait();
        for (int i = tid; i < L; i += nt) {
            C v = A.real_in ? mk<T>(((const T*)A.f)[w * L + i], T(0)) : ((const C*)A.f)[w * L + i];
            if (pre) v = cmul(v, __ldg(pre + i));
            sF[i] = v;
        }
    }
    __syncthreads();
    TINY_MARK(1);
    // ---- 1. F-branch: f^ = DFT_L(f) ----
    const C* fh = sF;
    if constexpr (CT) {
        static_assert(SL == 240 && SD == 8 && SC * SQ == 15, "compile-time shape: config 1 only");
        if (freq) {
            tstage<T, 240, 16, 1>(sF, sF2, 1, sTwL);
            __syncthreads();
            tstage<T, 240, 15, 16>(sF2, sF, 1, sTwL);
            __syncthreads();
        }
    } else if (freq) {
        fh = fft_smem<T>(sF, sF2, A.rdL, 1, L, sTwL);
    }
    TINY_MARK(2);
    // ---- 2. Zak gather of all (l, r, k, s): sX[((l c + r) p + k) d + s] ----
    {
        const int Lc = L / c;
        for (int i = tid; i < L; i += nt) {
            const int s = i % d, t = i / d;          // t = (l c + r) p + k
            const int k = t % p, lr = t / p;
            const int r = lr % c, l = lr / c;
            const int z = (k * q + p * l + s * p * q) % Lc;
            const int x = r + c * z;
            sX[i] = cmul(fh[x], sCh[x]);
        }
    }
    __syncthreads();
    TINY_MARK(3);
    // ---- 3. DFT_d over s ----
    C* phi;
    if constexpr (CT) {
        tstage<T, 8, 8, 1>(sX, sY, q * c * p, sTwd);
        __syncthreads();
        phi = sY;
    } else {
        phi = fft_smem<T>(sX, sY, A.rdd, q * c * p, d, sTwd);
    }
    TINY_MARK(4);
    C* Yb = phi == sX ? sY : sX;
    // ---- 4. products Y(l, r, u; nu) at Yb[((l c + r) q + u) d + nu] ----
    for (int i = tid; i < LQ; i += nt) {
        const int nu = i % d, t = i / d;              // t = (l c + r) q + u
        const int u = t % q, lr = t / q;
        const int r = lr % c;
        const C* ph = phi + lr * p * d + nu;
        const C* gk = sG + (r * q + u) * p * d + nu;
        C acc = cmul(ph[0], gk[0]);
        for (int k = 1; k < p; ++k) acc = acc + cmul(ph[k * d], gk[k * d]);
        Yb[i] = acc;
    }
    __syncthreads();
    TINY_MARK(5);
    // ---- 5. DFT_d over nu; scatter to C[n][j] ----
    C* Yd;   // phi is dead: its buffer is the scratch
    if constexpr (CT) {
        tstage<T, 8, 8, 1>(Yb, phi, q * c * q, sTwd);
        __syncthreads();
        Yd = phi;
    } else {
        Yd = fft_smem<T>(Yb, phi, A.rdd, q * c * q, d, sTwd);
    }
    TINY_MARK(6);
    C* Cn = Yd == sX ? sY : sX;
    for (int i = tid; i < LQ; i += nt) {
        const int np = i % d, t = i / d;              // destination n', source row t = (l c + r) q + u
        const int u = t % q, lr = t / q;
        const int r = lr % c, l = lr / c;
        const int kappa = ((l - u) % q + q) % q;
        const int off = l < u ? 1 : 0;
        int tau = d - np - off;
        if (tau >= d) tau -= d;
        if (tau < 0) tau += d;
        const int j = r + c * ((l * p) % q);
        Cn[(kappa + q * np) * iM + j] = Yd[t * d + tau];
    }
    __syncthreads();
    TINY_MARK(7);
    // ---- 6. DFT over j of the iN columns ----
    C* X;
    if constexpr (CT) {
        tstage<T, 15, 15, 1>(Cn, Yd, iN, sTwm);
        __syncthreads();
        X = Yd;
    } else {
        X = fft_smem<T>(Cn, Yd, A.rdm, iN, iM, sTwm);
    }
    TINY_MARK(8);
    // ---- 7. output ----
    C* out = (C*)A.B.out + w * A.B.M * A.B.N;
    if (!freq) {
        const C* __restrict__ E = (const C*)A.B.E;
        const int Mi = (int)A.B.M, Ni = (int)A.B.N;
        for (int i = tid; i < Mi * Ni; i += nt) {
            const int n = i % Ni, mo = i / Ni;
            int m = mo + __ldg(A.B.rot + n);
            if (m >= Mi) m -= Mi;
            out[i] = cmul(__ldg(E + n), X[n * iM + m]);
        }
    } else if (A.odst) {
        for (int i = tid; i < LQ; i += nt) out[sDst[i]] = cmul(sPh[i], X[i]);
    } else {
        const unsigned long long Nr = (unsigned long long)A.B.Nr;
        for (int i = tid; i < LQ; i += nt) {
            const int kc = i % iM, n = i / iM;
            const FbCol cc = fb_col(A.B, (unsigned long long)n);
            const FbIter<C> it = fb_iter<C>(A.B, cc, kc ? Nr - (unsigned long long)kc : 0ull);
            fb_put(A.B, out, it, X[i]);
        }
    }
    __syncthreads();
    TINY_MARK(9);
}

// Synthesis on the one-CTA path (dgt_execute_inverse of short signals): the adjoint of
// tiny_kernel, step by step in reverse, every value kept conjugated so that each DFT is a
// forward one (conj(DFT^H(y)) = DFT(conj y)); the conjugations fold into the first loads and
// the last stores.  Steps (z = conj of the adjoint's value):
//   7'. z(n, kc) = ph conj(c[dst]) (F-branch remap table) / E(n) conj(c[(m - rot n) mod M][n])
//   6'. DFT over kc of each column n                       -> z = conj C'(n, j)
//   5'. gather through the forward scatter map into rows (l, r, u), DFT_d over tau
//   4'. acc(l, r, k; nu) = sum_u z(l, r, u; nu) G(r, u, k; nu)
//   3'. DFT_d over nu                                       -> z = conj v'(l, r, k; s)
//   2'. scatter through the Zak map with the chirp: z(x) = chirp(x) z(l, r, k; s)
//   1'. F-branch: DFT_L, f = conj(pre z); T-branch: f = conj(z)
template <typename T, int SL = 0, int SC = 0, int SD = 0, int SP = 0, int SQ = 0>
__global__ void __launch_bounds__(256) tiny_adj_kernel(const __grid_constant__ TinyArgs A, const void* cin, void* fout) {
    using C = cx<T>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr bool CT = SL > 0;
    const int L = CT ? SL : A.L, c = CT ? SC : A.c, d = CT ? SD : A.d, p = CT ? SP : A.p, q = CT ? SQ : A.q;
    const int iM = CT ? SC * SQ : A.iM, iN = CT ? SQ * SD : A.iN;
    const bool freq = A.B.branch == DGT_BRANCH_FREQ;
    const int LQ = L / p * q;
    const int LX = LQ > L ? LQ : L;
    C* sF = (C*)smem_raw;        // L
    C* sF2 = sF + L;             // L
    C* sX = sF2 + L;             // max(L, LQ)
    C* sY = sX + LX;             // max(L, LQ)
    C* sG = sY + LX;             // L
    C* sCh = sG + L;             // L
    C* sTwL = sCh + L;           // L (F-branch)
    C* sPh = sTwL + (freq ? L : 0);
    unsigned int* sDst = (unsigned int*)(sPh + (freq ? LQ : 0));
    C* sTwd = (C*)((char*)sPh + (freq ? (int64_t)LQ * sizeof(C) + (LQ + 1) / 2 * sizeof(C) : 0));
    C* sTwm = sTwd + d;
    const int tid = threadIdx.x, nt = blockDim.x;
    const int64_t w = blockIdx.x;
    pdl_trigger();
    {
        const C* __restrict__ chirp = (const C*)A.chirp;
        for (int i = tid; i < L; i += nt) {
            sG[i] = __ldg((const C*)A.G + i);
            sCh[i] = chirp ? __ldg(chirp + i) : mk<T>(T(1), T(0));
            if (freq) sTwL[i] = __ldg((const C*)A.twL + i);
        }
        for (int i = tid; i < d; i += nt) sTwd[i] = __ldg((const C*)A.twd + i);
        for (int i = tid; i < iM; i += nt) sTwm[i] = __ldg((const C*)A.twm + i);
        if (freq && A.odst) {
            for (int i = tid; i < LQ; i += nt) {
                sPh[i] = __ldg((const C*)A.oph + i);
                sDst[i] = __ldg((const unsigned int*)A.odst + i);
            }
        }
    }
    __syncthreads();
    pdl_wait();
    // ---- 7'. z(n, kc) into sX[n iM + kc] ----
    const C* cw = (const C*)cin + w * A.B.M * A.B.N;
    if (!freq) {
        const C* __restrict__ E = (const C*)A.B.E;
        const int Mi = (int)A.B.M, Ni = (int)A.B.N;
        for (int i = tid; i < Mi * Ni; i += nt) {
            const int n = i % Ni, mo = i / Ni;
            int m = mo + __ldg(A.B.rot + n);
            if (m >= Mi) m -= Mi;
            const C v = cw[i];
            sX[n * iM + m] = cmul(__ldg(E + n), mk<T>(v.x, -v.y));
        }
    } else {
        for (int i = tid; i < LQ; i += nt) {
            const C v = cw[sDst[i]];
            sX[i] = cmul(sPh[i], mk<T>(v.x, -v.y));
        }
    }
    __syncthreads();
    // ---- 6'. DFT over kc of the iN columns ----
    C* Z;
    if constexpr (CT) {
        tstage<T, 15, 15, 1>(sX, sY, iN, sTwm);
        __syncthreads();
        Z = sY;
    } else {
        Z = fft_smem<T>(sX, sY, A.rdm, iN, iM, sTwm);
    }
    C* R = Z == sX ? sY : sX;
    // ---- 5'. gather rows (l, r, u) through the forward scatter map, DFT_d over tau ----
    for (int i = tid; i < LQ; i += nt) {
        const int np = i % d, t = i / d;          // row t = (l c + r) q + u, source n' of tau
        const int u = t % q, lr = t / q;
        const int r = lr % c, l = lr / c;
        const int kappa = ((l - u) % q + q) % q;
        const int off = l < u ? 1 : 0;
        int tau = d - np - off;
        if (tau >= d) tau -= d;
        if (tau < 0) tau += d;
        const int j = r + c * ((l * p) % q);
        R[t * d + tau] = Z[(kappa + q * np) * iM + j];
    }
    __syncthreads();
    C* Yd;
    if constexpr (CT) {
        tstage<T, 8, 8, 1>(R, Z, q * c * q, sTwd);
        __syncthreads();
        Yd = Z;
    } else {
        Yd = fft_smem<T>(R, Z, A.rdd, q * c * q, d, sTwd);
    }
    C* Acc = Yd == sX ? sY : sX;
    // ---- 4'. acc(l, r, k; nu) = sum_u z(l, r, u; nu) G(r, u, k; nu) ----
    for (int i = tid; i < L; i += nt) {
        const int nu = i % d, t = i / d;          // t = (l c + r) p + k
        const int k = t % p, lr = t / p;
        const int r = lr % c;
        C acc = mk<T>(T(0), T(0));
        for (int u = 0; u < q; ++u)
            acc = acc + cmul(Yd[(lr * q + u) * d + nu], sG[((r * q + u) * p + k) * d + nu]);
        Acc[i] = acc;
    }
    __syncthreads();
    // ---- 3'. DFT_d over nu ----
    C* V;
    if constexpr (CT) {
        tstage<T, 8, 8, 1>(Acc, Yd, q * c * p, sTwd);
        __syncthreads();
        V = Yd;
    } else {
        V = fft_smem<T>(Acc, Yd, A.rdd, q * c * p, d, sTwd);
    }
    // ---- 2'. scatter through the Zak map with the chirp ----
    {
        const int Lc = L / c;
        for (int i = tid; i < L; i += nt) {
            const int s = i % d, t = i / d;
            const int k = t % p, lr = t / p;
            const int r = lr % c, l = lr / c;
            const int x = r + c * ((k * q + p * l + s * p * q) % Lc);
            sF[x] = cmul(sCh[x], V[i]);
        }
    }
    __syncthreads();
    // ---- 1'. F-branch DFT_L; f = conj(pre z) / conj(z) ----
    const C* fz = sF;
    if (freq) {
        if constexpr (CT) {
            tstage<T, 240, 16, 1>(sF, sF2, 1, sTwL);
            __syncthreads();
            tstage<T, 240, 15, 16>(sF2, sF, 1, sTwL);
            __syncthreads();
        } else {
            fz = fft_smem<T>(sF, sF2, A.rdL, 1, L, sTwL);
        }
    }
    const C* __restrict__ pre = (const C*)A.pre;
    C* fo = (C*)fout + w * L;
    for (int i = tid; i < L; i += nt) {
        C v = fz[i];
        if (pre) v = cmul(__ldg(pre + i), v);
        fo[i] = mk<T>(v.x, -v.y);
    }
}
