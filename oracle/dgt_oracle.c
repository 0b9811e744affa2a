/*
 * oracle/dgt_oracle.c -- CPU oracle for the DGT on a nonseparable lattice.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / "--impl reference" legs may load this library.  It shares no code,
 * header, table or constant generator with the CUDA path (paper_1307_4569_b200/),
 * and the product path never calls it.
 *
 * What it computes: the plain definition, Eq. (DGT) of the paper
 * (Sec. 2.1), with the operator conventions of PAPER.md:151-158
 * (indices cyclic mod L), under DESIGN.md readings Z1 (0-based g(l - a n): the
 * printed "+1" is a 1-based artifact) and Z2 (m counted from the lowest
 * non-negative frequency b*(m + w(n))):
 *
 *   c_w(m,n) = sum_{l=0}^{L-1} f_w(l) conj(g((l - a n) mod L)) exp(-2 pi i l (m + w(n)) / M),
 *   w(n) = (n lambda1 mod lambda2) / lambda2,     m in [0,M), n in [0,N=L/a).
 *
 * Two evaluations of the SAME finite sum (no FFT, no Zak transform, no chirps):
 *   O1 literal  : the sum exactly as written.  The phase l(m+w(n))/M is reduced
 *                 exactly in integers: k = ((m lambda2 + n lambda1 mod lambda2) l)
 *                 mod (lambda2 M), looked up in omega[k] = exp(-2 pi i k/(lambda2 M))
 *                 built in long double.
 *   O2 regrouped: the same sum reassociated by splitting l = j + t M (j<M, t<b):
 *                 h(j) = sum_t f(j+tM) conj(g(j+tM-an)) exp(-2 pi i (w' t mod lambda2)/lambda2),
 *                 c(m,n) = sum_j h(j) omega[((m lambda2 + w') j) mod (lambda2 M)],
 *                 w' = n lambda1 mod lambda2.  Cost N(L + M^2) instead of MNL.
 * Both accumulate each block of 64 products in double and the blocks in long
 * double, so the result is deterministic (OpenMP only over (w,n) columns).
 *
 * Layouts: complex numbers are interleaved (re, im) doubles.
 *   f : W x L (signal-major)        g : L
 *   cols : list of ncols column indices n (NULL => all N columns, ncols ignored)
 *   c : W x M x ncols  (n-list fastest), i.e. c[(w*M + m)*ncols + i] = c_w(m, cols[i])
 * Returns 0 on success, 2 on invalid arguments (a, M must divide L, lambda2 >= 1,
 * 0 <= lambda1 < lambda2, lambda2 | L/M and lambda2 | L/a -- Prop. minsig,
 * PAPER.md:580-615).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef long double ld;
static const ld ORACLE_PI = 3.141592653589793238462643383279502884L;

static int check_args(int64_t L, int64_t a, int64_t M, int64_t l1, int64_t l2, int64_t W) {
    if (L <= 0 || a <= 0 || M <= 0 || W < 0) return 2;
    if (L % a || L % M) return 2;
    if (l2 < 1 || l1 < 0 || l1 >= l2) return 2;
    if ((L / M) % l2 || (L / a) % l2) return 2;
    return 0;
}

/* omega[k] = exp(-2 pi i k / K), K = lambda2 * M, in long double, stored as double. */
static double* make_omega(int64_t K) {
    double* om = (double*)malloc(sizeof(double) * 2 * (size_t)K);
    for (int64_t k = 0; k < K; ++k) {
        ld th = -2.0L * ORACLE_PI * (ld)k / (ld)K;
        om[2 * k] = (double)cosl(th);
        om[2 * k + 1] = (double)sinl(th);
    }
    return om;
}

static void set_threads(int nthreads) {
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
}

int oracle_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* O1: literal direct sum of Eq. (DGT). */
int oracle_dgt_literal(const double* f, const double* g, int64_t L, int64_t a, int64_t M,
                       int64_t l1, int64_t l2, int64_t W, const int64_t* cols, int64_t ncols,
                       double* c, int nthreads) {
    int rc = check_args(L, a, M, l1, l2, W);
    if (rc) return rc;
    const int64_t N = L / a;
    if (!cols) ncols = N;
    const int64_t K = l2 * M;
    double* om = make_omega(K);
    set_threads(nthreads);
    const int64_t total = W * ncols;
#pragma omp parallel
    {
        double* h = (double*)malloc(sizeof(double) * 2 * (size_t)L);
#pragma omp for schedule(dynamic, 1)
        for (int64_t job = 0; job < total; ++job) {
            const int64_t w = job / ncols, i = job % ncols;
            const int64_t n = cols ? cols[i] : i;
            const double* fw = f + 2 * w * L;
            /* h(l) = f(l) * conj(g((l - a n) mod L)) */
            for (int64_t l = 0; l < L; ++l) {
                int64_t gi = ((l - a * n) % L + L) % L;
                double fr = fw[2 * l], fi = fw[2 * l + 1];
                double gr = g[2 * gi], gim = -g[2 * gi + 1];
                h[2 * l] = fr * gr - fi * gim;
                h[2 * l + 1] = fr * gim + fi * gr;
            }
            const int64_t wp = (n * l1) % l2;
            for (int64_t m = 0; m < M; ++m) {
                const int64_t step = m * l2 + wp; /* (m + w(n)) * lambda2 */
                ld sr = 0.0L, si = 0.0L;
                double br = 0.0, bi = 0.0;
                int64_t k = 0; /* (step * l) mod K, advanced exactly */
                for (int64_t l = 0; l < L; ++l) {
                    double orr = om[2 * k], oi = om[2 * k + 1];
                    br += h[2 * l] * orr - h[2 * l + 1] * oi;
                    bi += h[2 * l] * oi + h[2 * l + 1] * orr;
                    if ((l & 63) == 63) { sr += br; si += bi; br = bi = 0.0; }
                    k += step;
                    if (k >= K) k %= K;
                }
                sr += br; si += bi;
                double* out = c + 2 * ((w * M + m) * ncols + i);
                out[0] = (double)sr;
                out[1] = (double)si;
            }
        }
        free(h);
    }
    free(om);
    return 0;
}

/* O2: the same sum regrouped over l = j + t M. */
int oracle_dgt_regrouped(const double* f, const double* g, int64_t L, int64_t a, int64_t M,
                         int64_t l1, int64_t l2, int64_t W, const int64_t* cols, int64_t ncols,
                         double* c, int nthreads) {
    int rc = check_args(L, a, M, l1, l2, W);
    if (rc) return rc;
    const int64_t N = L / a, b = L / M;
    if (!cols) ncols = N;
    const int64_t K = l2 * M;
    double* om = make_omega(K);
    /* zeta[k] = exp(-2 pi i k / lambda2) */
    double* zeta = (double*)malloc(sizeof(double) * 2 * (size_t)l2);
    for (int64_t k = 0; k < l2; ++k) {
        ld th = -2.0L * ORACLE_PI * (ld)k / (ld)l2;
        zeta[2 * k] = (double)cosl(th);
        zeta[2 * k + 1] = (double)sinl(th);
    }
    set_threads(nthreads);
    const int64_t total = W * ncols;
#pragma omp parallel
    {
        double* h = (double*)malloc(sizeof(double) * 2 * (size_t)M);
#pragma omp for schedule(dynamic, 1)
        for (int64_t job = 0; job < total; ++job) {
            const int64_t w = job / ncols, i = job % ncols;
            const int64_t n = cols ? cols[i] : i;
            const double* fw = f + 2 * w * L;
            const int64_t wp = (n * l1) % l2;
            for (int64_t j = 0; j < M; ++j) {
                ld sr = 0.0L, si = 0.0L;
                double br = 0.0, bi = 0.0;
                for (int64_t t = 0; t < b; ++t) {
                    const int64_t l = j + t * M;
                    const int64_t gi = ((l - a * n) % L + L) % L;
                    double fr = fw[2 * l], fi = fw[2 * l + 1];
                    double gr = g[2 * gi], gim = -g[2 * gi + 1];
                    double pr = fr * gr - fi * gim, pi = fr * gim + fi * gr;
                    const int64_t zk = (wp * t) % l2;
                    double zr = zeta[2 * zk], zi = zeta[2 * zk + 1];
                    br += pr * zr - pi * zi;
                    bi += pr * zi + pi * zr;
                    if ((t & 63) == 63) { sr += br; si += bi; br = bi = 0.0; }
                }
                sr += br; si += bi;
                h[2 * j] = (double)sr;
                h[2 * j + 1] = (double)si;
            }
            for (int64_t m = 0; m < M; ++m) {
                const int64_t step = m * l2 + wp;
                ld sr = 0.0L, si = 0.0L;
                double br = 0.0, bi = 0.0;
                int64_t k = 0;
                for (int64_t j = 0; j < M; ++j) {
                    double orr = om[2 * k], oi = om[2 * k + 1];
                    br += h[2 * j] * orr - h[2 * j + 1] * oi;
                    bi += h[2 * j] * oi + h[2 * j + 1] * orr;
                    if ((j & 63) == 63) { sr += br; si += bi; br = bi = 0.0; }
                    k += step;
                    if (k >= K) k %= K;
                }
                sr += br; si += bi;
                double* out = c + 2 * ((w * M + m) * ncols + i);
                out[0] = (double)sr;
                out[1] = (double)si;
            }
        }
        free(h);
    }
    free(zeta);
    free(om);
    return 0;
}

/*
 * Synthesis (the inverse DGT with a dual window): the inversion formula
 * f = sum c(m,n) S^{-1} pi(x,omega) g of PAPER.md:171-175 (Sec. 2.1) with the canonical
 * dual gamma = S^{-1} g, indexed as Eq. (DGT) indexes the coefficients:
 *
 *   f_w(l) = sum_{n<N} sum_{m<M} c_w(m,n) gamma((l - a n) mod L) exp(+2 pi i l (m + w(n)) / M).
 *
 * This is the adjoint of Eq. (DGT) with window gamma.  gamma is an input (any window; pass
 * the canonical dual to invert).  Layout: c is W x M x N (n fastest), f is W x L, all
 * interleaved complex doubles.  Phases reduced exactly as in O1 (conjugated omega).
 *   S1 literal  : the double sum as written, per l.
 *   S2 regrouped: l = j + t M:  H_n(j) = sum_m c(m,n) exp(2 pi i j (m + w(n)) / M),
 *                 f(j + t M) = sum_n gamma(j + t M - a n) exp(2 pi i t w'(n) / lambda2) H_n(j),
 *                 w' = n lambda1 mod lambda2  (exp(2 pi i t M (m + w)/M) = exp(2 pi i t w)).
 * OpenMP over (w, l) (S1) or (w, j) (S2); every output is written by one thread.
 */
int oracle_idgt_literal(const double* c, const double* g, int64_t L, int64_t a, int64_t M,
                        int64_t l1, int64_t l2, int64_t W, double* f, int nthreads) {
    int rc = check_args(L, a, M, l1, l2, W);
    if (rc) return rc;
    const int64_t N = L / a;
    const int64_t K = l2 * M;
    double* om = make_omega(K);
    set_threads(nthreads);
    const int64_t total = W * L;
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t job = 0; job < total; ++job) {
        const int64_t w = job / L, l = job % L;
        const double* cw = c + 2 * w * M * N;
        ld sr = 0.0L, si = 0.0L;
        for (int64_t n = 0; n < N; ++n) {
            const int64_t gi = ((l - a * n) % L + L) % L;
            const double gr = g[2 * gi], gim = g[2 * gi + 1];
            const int64_t wp = (n * l1) % l2;
            double br = 0.0, bi = 0.0;
            for (int64_t m = 0; m < M; ++m) {
                /* exp(+2 pi i l (m lambda2 + w') / (lambda2 M)) = conj(omega[k]) */
                const int64_t k = ((l % K) * ((m * l2 + wp) % K)) % K;
                const double er = om[2 * k], ei = -om[2 * k + 1];
                const double cr = cw[2 * (m * N + n)], ci = cw[2 * (m * N + n) + 1];
                /* c * gamma * e */
                const double pr = cr * gr - ci * gim, pi = cr * gim + ci * gr;
                br += pr * er - pi * ei;
                bi += pr * ei + pi * er;
            }
            sr += br;
            si += bi;
        }
        f[2 * (w * L + l)] = (double)sr;
        f[2 * (w * L + l) + 1] = (double)si;
    }
    free(om);
    return 0;
}

int oracle_idgt_regrouped(const double* c, const double* g, int64_t L, int64_t a, int64_t M,
                          int64_t l1, int64_t l2, int64_t W, double* f, int nthreads) {
    int rc = check_args(L, a, M, l1, l2, W);
    if (rc) return rc;
    const int64_t N = L / a, b = L / M;
    const int64_t K = l2 * M;
    double* om = make_omega(K);
    double* zeta = (double*)malloc(sizeof(double) * 2 * (size_t)l2); /* exp(+2 pi i k / lambda2) */
    for (int64_t k = 0; k < l2; ++k) {
        ld th = 2.0L * ORACLE_PI * (ld)k / (ld)l2;
        zeta[2 * k] = (double)cosl(th);
        zeta[2 * k + 1] = (double)sinl(th);
    }
    set_threads(nthreads);
    const int64_t total = W * M;
#pragma omp parallel
    {
        double* H = (double*)malloc(sizeof(double) * 2 * (size_t)N);
#pragma omp for schedule(dynamic, 1)
        for (int64_t job = 0; job < total; ++job) {
            const int64_t w = job / M, j = job % M;
            const double* cw = c + 2 * w * M * N;
            for (int64_t n = 0; n < N; ++n) {
                const int64_t wp = (n * l1) % l2;
                ld sr = 0.0L, si = 0.0L;
                double br = 0.0, bi = 0.0;
                for (int64_t m = 0; m < M; ++m) {
                    const int64_t k = (j * ((m * l2 + wp) % K)) % K;
                    const double er = om[2 * k], ei = -om[2 * k + 1];
                    const double cr = cw[2 * (m * N + n)], ci = cw[2 * (m * N + n) + 1];
                    br += cr * er - ci * ei;
                    bi += cr * ei + ci * er;
                    if ((m & 63) == 63) { sr += br; si += bi; br = bi = 0.0; }
                }
                sr += br; si += bi;
                H[2 * n] = (double)sr;
                H[2 * n + 1] = (double)si;
            }
            for (int64_t t = 0; t < b; ++t) {
                const int64_t l = j + t * M;
                ld sr = 0.0L, si = 0.0L;
                double br = 0.0, bi = 0.0;
                for (int64_t n = 0; n < N; ++n) {
                    const int64_t gi = ((l - a * n) % L + L) % L;
                    const double gr = g[2 * gi], gim = g[2 * gi + 1];
                    const int64_t zk = (((n * l1) % l2) * t) % l2;
                    const double zr = zeta[2 * zk], zi = zeta[2 * zk + 1];
                    /* gamma * zeta * H(n) */
                    const double qr = gr * zr - gim * zi, qi = gr * zi + gim * zr;
                    br += qr * H[2 * n] - qi * H[2 * n + 1];
                    bi += qr * H[2 * n + 1] + qi * H[2 * n];
                    if ((n & 63) == 63) { sr += br; si += bi; br = bi = 0.0; }
                }
                sr += br; si += bi;
                f[2 * (w * L + l)] = (double)sr;
                f[2 * (w * L + l) + 1] = (double)si;
            }
        }
        free(H);
    }
    free(zeta);
    free(om);
    return 0;
}
