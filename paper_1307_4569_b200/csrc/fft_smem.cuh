// fft_smem.cuh -- batched forward DFTs of runtime length on shared memory.
//
// All DFTs of the method are FORWARD, X(k) = sum_j x(j) exp(-2 pi i jk/n): the Zak
// DFT over s, the "inverse factorisation" DFT over nu (with exp(-2 pi i nu tau/d),
// DESIGN.md §4.2) and the output FFT over j.  This header is the
// generic engine: Stockham autosort passes (no bit reversal), one radix-R butterfly
// per thread per pass, ping-pong between two shared buffers, twiddles from a table
// tw[k] = exp(-2 pi i k / n) built in fp64 at plan time.  Radices 2,3,4,5,8,16 are
// register butterflies; any other prime factor uses a direct O(R^2) butterfly.
#pragma once
#include "cplx.cuh"

namespace nsdgt {

constexpr int kMaxStages = 24;

struct Radices {
    int n;
    int nst;
    int r[kMaxStages];
};

template <typename T> struct Consts;
template <> struct Consts<float> {
    static constexpr float r2 = 0.70710678118654752440f;
    static constexpr float s3 = 0.86602540378443864676f;
    static constexpr float c51 = 0.30901699437494742410f, c52 = -0.80901699437494742410f;
    static constexpr float s51 = 0.95105651629515357212f, s52 = 0.58778525229247312917f;
    static constexpr float c16 = 0.92387953251128675613f, s16 = 0.38268343236508977173f;
};
template <> struct Consts<double> {
    static constexpr double r2 = 0.70710678118654752440;
    static constexpr double s3 = 0.86602540378443864676;
    static constexpr double c51 = 0.30901699437494742410, c52 = -0.80901699437494742410;
    static constexpr double s51 = 0.95105651629515357212, s52 = 0.58778525229247312917;
    static constexpr double c16 = 0.92387953251128675613, s16 = 0.38268343236508977173;
};

template <typename T> __device__ __forceinline__ void dft2(cx<T>* v) {
    cx<T> a = v[0], b = v[1];
    v[0] = a + b; v[1] = a - b;
}

template <typename T> __device__ __forceinline__ void dft4(cx<T>& v0, cx<T>& v1, cx<T>& v2, cx<T>& v3) {
    cx<T> t0 = v0 + v2, t1 = v0 - v2, t2 = v1 + v3, t3 = mul_mi(v1 - v3);
    v0 = t0 + t2; v2 = t0 - t2; v1 = t1 + t3; v3 = t1 - t3;
}

template <typename T> __device__ __forceinline__ void dft3(cx<T>* v) {
    const T s = Consts<T>::s3;
    cx<T> t1 = v[1] + v[2];
    cx<T> t2 = v[0] - scale(t1, T(0.5));
    cx<T> t3 = scale(mul_mi(v[1] - v[2]), s);
    v[0] = v[0] + t1;
    v[1] = t2 + t3;
    v[2] = t2 - t3;
}

template <typename T> __device__ __forceinline__ void dft5(cx<T>* v) {
    const T c1 = Consts<T>::c51, c2 = Consts<T>::c52, s1 = Consts<T>::s51, s2 = Consts<T>::s52;
    cx<T> a1 = v[1] + v[4], a2 = v[2] + v[3], b1 = v[1] - v[4], b2 = v[2] - v[3];
    cx<T> y0 = v[0] + a1 + a2;
    cx<T> t1 = v[0] + scale(a1, c1) + scale(a2, c2);
    cx<T> t2 = v[0] + scale(a1, c2) + scale(a2, c1);
    cx<T> u1 = scale(b1, s1) + scale(b2, s2);
    cx<T> u2 = scale(b1, s2) - scale(b2, s1);
    v[0] = y0;
    v[1] = t1 + mul_mi(u1);
    v[4] = t1 - mul_mi(u1);
    v[2] = t2 + mul_mi(u2);
    v[3] = t2 - mul_mi(u2);
}

// multiply by W8^1 = (1 - i)/sqrt2, W8^3 = (-1 - i)/sqrt2
template <typename T> __device__ __forceinline__ cx<T> w8_1(cx<T> a) {
    const T r = Consts<T>::r2;
    return mk<T>((a.x + a.y) * r, (a.y - a.x) * r);
}
template <typename T> __device__ __forceinline__ cx<T> w8_3(cx<T> a) {
    const T r = Consts<T>::r2;
    return mk<T>((a.y - a.x) * r, -(a.x + a.y) * r);
}

template <typename T> __device__ __forceinline__ void dft8(cx<T>* v) {
    cx<T> e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6];
    cx<T> o0 = v[1], o1 = v[3], o2 = v[5], o3 = v[7];
    dft4<T>(e0, e1, e2, e3);
    dft4<T>(o0, o1, o2, o3);
    o1 = w8_1<T>(o1);
    o2 = mul_mi(o2);
    o3 = w8_3<T>(o3);
    v[0] = e0 + o0; v[4] = e0 - o0;
    v[1] = e1 + o1; v[5] = e1 - o1;
    v[2] = e2 + o2; v[6] = e2 - o2;
    v[3] = e3 + o3; v[7] = e3 - o3;
}

template <typename T> __device__ __forceinline__ void dft16(cx<T>* v) {
    const T c = Consts<T>::c16, s = Consts<T>::s16;
    // columns j1: DFT4 over j2 of v[j1 + 4 j2]
#pragma unroll
    for (int j1 = 0; j1 < 4; ++j1) dft4<T>(v[j1], v[j1 + 4], v[j1 + 8], v[j1 + 12]);
    // twiddle X[j1][k1] (stored at v[j1 + 4 k1]) *= W16^{j1 k1}
    v[5] = cmul(v[5], mk<T>(c, -s));    // j1=1,k1=1: W16^1
    v[9] = w8_1<T>(v[9]);               // j1=1,k1=2: W16^2
    v[13] = cmul(v[13], mk<T>(s, -c));  // j1=1,k1=3: W16^3
    v[6] = w8_1<T>(v[6]);               // j1=2,k1=1: W16^2
    v[10] = mul_mi(v[10]);              // j1=2,k1=2: W16^4
    v[14] = w8_3<T>(v[14]);             // j1=2,k1=3: W16^6
    v[7] = cmul(v[7], mk<T>(s, -c));    // j1=3,k1=1: W16^3
    v[11] = w8_3<T>(v[11]);             // j1=3,k1=2: W16^6
    v[15] = cmul(v[15], mk<T>(-c, s));  // j1=3,k1=3: W16^9 = -W16^1
    // rows k1: DFT4 over j1 of v[j1 + 4 k1] -> y[k1 + 4 k2]
    cx<T> y[16];
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) {
        cx<T> a0 = v[4 * k1], a1 = v[4 * k1 + 1], a2 = v[4 * k1 + 2], a3 = v[4 * k1 + 3];
        dft4<T>(a0, a1, a2, a3);
        y[k1] = a0; y[k1 + 4] = a1; y[k1 + 8] = a2; y[k1 + 12] = a3;
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = y[i];
}

template <typename T, int R> __device__ __forceinline__ void dft_fixed(cx<T>* v) {
    if constexpr (R == 2) dft2<T>(v);
    else if constexpr (R == 3) dft3<T>(v);
    else if constexpr (R == 4) dft4<T>(v[0], v[1], v[2], v[3]);
    else if constexpr (R == 5) dft5<T>(v);
    else if constexpr (R == 8) dft8<T>(v);
    else if constexpr (R == 16) dft16<T>(v);
}

// One Stockham pass of fixed radix R on `nseq` sequences (stride `ld`) of length n.
template <typename T, int R>
__device__ __forceinline__ void stage_fixed(const cx<T>* __restrict__ in, cx<T>* __restrict__ out, int n,
                                            int Ns, int nseq, int ld, const cx<T>* __restrict__ tw) {
    const int nb = n / R;
    const int total = nb * nseq;
    const int tstep = n / (Ns * R);
    for (int t = threadIdx.x; t < total; t += blockDim.x) {
        const int seq = t / nb;
        const int j = t - seq * nb;
        const cx<T>* src = in + seq * ld;
        cx<T>* dst = out + seq * ld;
        const int k = j % Ns;
        cx<T> v[R];
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = src[j + r * nb];
        if (Ns > 1) {
            const int step = k * tstep;
#pragma unroll
            for (int r = 1; r < R; ++r) v[r] = cmul(v[r], tw[r * step]);
        }
        dft_fixed<T, R>(v);
        const int base = (j / Ns) * Ns * R + k;
#pragma unroll
        for (int r = 0; r < R; ++r) dst[base + r * Ns] = v[r];
    }
}

// Generic radix (any R): direct O(R^2) butterfly using the length-n twiddle table.
template <typename T>
__device__ void stage_generic(const cx<T>* __restrict__ in, cx<T>* __restrict__ out, int n, int R, int Ns,
                              int nseq, int ld, const cx<T>* __restrict__ tw) {
    const int nb = n / R;
    const int total = nb * nseq;
    const int tstep = n / (Ns * R);
    for (int t = threadIdx.x; t < total; t += blockDim.x) {
        const int seq = t / nb;
        const int j = t - seq * nb;
        const cx<T>* src = in + seq * ld;
        cx<T>* dst = out + seq * ld;
        const int k = j % Ns;
        const int step = k * tstep;
        const int base = (j / Ns) * Ns * R + k;
        for (int ro = 0; ro < R; ++ro) {
            cx<T> acc = mk<T>(T(0), T(0));
            for (int i = 0; i < R; ++i) {
                cx<T> x = src[j + i * nb];
                if (Ns > 1 && i) x = cmul(x, tw[i * step]);
                const int e = (i * ro) % R;
                acc = acc + (e ? cmul(x, tw[e * nb]) : x);
            }
            dst[base + ro * Ns] = acc;
        }
    }
}

// Forward DFT of nseq sequences (stride ld) held in `a`; `b` is scratch of the same
// size.  Returns the buffer holding the result.  All threads of the block must call.
template <typename T>
__device__ cx<T>* fft_smem(cx<T>* a, cx<T>* b, const Radices& rd, int nseq, int ld, const cx<T>* __restrict__ tw) {
    const int n = rd.n;
    int Ns = 1;
    for (int st = 0; st < rd.nst; ++st) {
        const int R = rd.r[st];
        switch (R) {
            case 2: stage_fixed<T, 2>(a, b, n, Ns, nseq, ld, tw); break;
            case 3: stage_fixed<T, 3>(a, b, n, Ns, nseq, ld, tw); break;
            case 4: stage_fixed<T, 4>(a, b, n, Ns, nseq, ld, tw); break;
            case 5: stage_fixed<T, 5>(a, b, n, Ns, nseq, ld, tw); break;
            case 8: stage_fixed<T, 8>(a, b, n, Ns, nseq, ld, tw); break;
            case 16: stage_fixed<T, 16>(a, b, n, Ns, nseq, ld, tw); break;
            default: stage_generic<T>(a, b, n, R, Ns, nseq, ld, tw); break;
        }
        __syncthreads();
        cx<T>* t = a; a = b; b = t;
        Ns *= R;
    }
    return a;
}

// ---- compile-time variants (lengths the planner meets on hot lattices, e.g. d = 180 of
// config 4): every index divides by a constant, composite radices run as register DFTs ----

// W_180^e, e < 180, in constant memory (fft_ct's inner twiddles have warp-uniform indices:
// constant-cache broadcasts instead of L1 data-pipe loads; filled by set_ct_twiddles)
__constant__ double2 c_tw180d[180];
__constant__ float2 c_tw180f[180];
__constant__ double2 c_tw720d[720];
__constant__ float2 c_tw720f[720];
template <typename T, int N> __device__ __forceinline__ cx<T> ctw(int e) {
    static_assert(N == 180 || N == 720, "constant twiddle tables exist for N = 180, 720");
    if constexpr (N == 180) {
        if constexpr (sizeof(cx<T>) == 16) return c_tw180d[e];
        else return c_tw180f[e];
    } else {
        if constexpr (sizeof(cx<T>) == 16) return c_tw720d[e];
        else return c_tw720f[e];
    }
}

// Length-(P Q) DFT in registers, natural order in and out (Cooley-Tukey, n = Q n1 + n2,
// k = k1 + P k2); W_{PQ}^e = W_N^{e tws} from the constant table (N = 180).
template <typename T, int P, int Q, int N>
__device__ __forceinline__ void dft_pq(cx<T>* v, int tws) {
    cx<T> a[P * Q];
#pragma unroll
    for (int n2 = 0; n2 < Q; ++n2) {
        cx<T> t[P];
#pragma unroll
        for (int n1 = 0; n1 < P; ++n1) t[n1] = v[Q * n1 + n2];
        dft_fixed<T, P>(t);
#pragma unroll
        for (int k1 = 0; k1 < P; ++k1) a[n2 * P + k1] = (n2 && k1) ? cmul(t[k1], ctw<T, N>(n2 * k1 * tws)) : t[k1];
    }
#pragma unroll
    for (int k1 = 0; k1 < P; ++k1) {
        cx<T> t[Q];
#pragma unroll
        for (int n2 = 0; n2 < Q; ++n2) t[n2] = a[n2 * P + k1];
        dft_fixed<T, Q>(t);
#pragma unroll
        for (int k2 = 0; k2 < Q; ++k2) v[k1 + P * k2] = t[k2];
    }
}

// One Stockham pass, radix R = P Q (Q = 1: a fixed radix), NS = product of earlier radices.
template <typename T, int N, int P, int Q, int NS>
__device__ __forceinline__ void stage_ct(const cx<T>* __restrict__ in, cx<T>* __restrict__ out, int nseq,
                                         const cx<T>* __restrict__ tw) {
    constexpr int R = P * Q, nb = N / R, tstep = N / (NS * R);
    for (int t = threadIdx.x; t < nb * nseq; t += blockDim.x) {
        const int seq = t / nb, j = t - seq * nb;
        const int k = j % NS;
        const cx<T>* src = in + seq * N;
        cx<T>* dst = out + seq * N;
        cx<T> v[R];
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = src[j + r * nb];
        if (NS > 1) {
            // W^{r k tstep} = (W^{k tstep})^r: one table load per butterfly (the lane-varying
            // index would cost a scattered load per element), powers by multiplication
            const cx<T> w1 = tw[k * tstep];
            cx<T> wr = w1;
            v[1] = cmul(v[1], w1);
#pragma unroll
            for (int r = 2; r < R; ++r) {
                wr = cmul(wr, w1);
                v[r] = cmul(v[r], wr);
            }
        }
        if constexpr (Q > 1) dft_pq<T, P, Q, N>(v, N / R);
        else dft_fixed<T, P>(v);
        const int base = (j / NS) * NS * R + k;
#pragma unroll
        for (int r = 0; r < R; ++r) dst[base + r * NS] = v[r];
    }
}

// DFT of nseq sequences of compile-time length N (stride N); returns the result buffer (a or
// b -- callers use the returned pointer).  The first pass has an odd radix, so its write stride
// is odd and the 16-byte stores of a quarter warp hit distinct banks.
//   N = 180 (config 4): radix 15 (3 x 5), then 12 (4 x 3)          -> result in a
//   N = 720 (config 2): radix 9 (3 x 3), then 16, then 5            -> result in b
//   N = 200 (config 2's output DFT): radix 5, then 8, then 5         -> result in b
template <typename T, int N>
__device__ cx<T>* fft_ct(cx<T>* a, cx<T>* b, int nseq, const cx<T>* __restrict__ tw) {
    static_assert(N == 180 || N == 720 || N == 200, "fft_ct: add a radix plan for this length");
    if constexpr (N == 200) {
        stage_ct<T, 200, 5, 1, 1>(a, b, nseq, tw);
        __syncthreads();
        stage_ct<T, 200, 8, 1, 5>(b, a, nseq, tw);
        __syncthreads();
        stage_ct<T, 200, 5, 1, 40>(a, b, nseq, tw);
        __syncthreads();
        return b;
    }
    else if constexpr (N == 180) {
        stage_ct<T, 180, 3, 5, 1>(a, b, nseq, tw);
        __syncthreads();
        stage_ct<T, 180, 4, 3, 15>(b, a, nseq, tw);
        __syncthreads();
        return a;
    } else {
        stage_ct<T, 720, 3, 3, 1>(a, b, nseq, tw);
        __syncthreads();
        stage_ct<T, 720, 16, 1, 9>(b, a, nseq, tw);
        __syncthreads();
        stage_ct<T, 720, 5, 1, 144>(a, b, nseq, tw);
        __syncthreads();
        return b;
    }
}

// Host: split n into radices (16, 8, 4, 2 for powers of two; then 5, 3; then primes).
inline Radices make_radices(int n) {
    Radices rd{};
    rd.n = n;
    int m = n, k = 0;
    int p2 = 0;
    while (m % 2 == 0) { m /= 2; ++p2; }
    while (p2 >= 4) { rd.r[k++] = 16; p2 -= 4; }
    if (p2 == 3) rd.r[k++] = 8;
    else if (p2 == 2) rd.r[k++] = 4;
    else if (p2 == 1) rd.r[k++] = 2;
    while (m % 5 == 0) { rd.r[k++] = 5; m /= 5; }
    while (m % 3 == 0) { rd.r[k++] = 3; m /= 3; }
    for (int p = 7; m > 1; p += 2) {
        while (m % p == 0) { rd.r[k++] = p; m /= p; }
        if ((long long)p * p > m && m > 1) { rd.r[k++] = m; m = 1; }
    }
    rd.nst = k;
    return rd;
}

}  // namespace nsdgt
