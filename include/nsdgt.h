/*
 * nsdgt.h -- C ABI of the B200-native forward DGT on a nonseparable lattice.
 *
 * Operation (the whole library computes exactly this):
 *   Eq. (DGT), PAPER.md:238-242 (Sec. 2.1), under DESIGN.md readings Z1/Z2:
 *     c_w(m,n) = sum_{l=0}^{L-1} f_w(l) conj(g((l - a n) mod L)) exp(-2 pi i l (m + w(n)) / M),
 *     w(n) = (n lambda1 mod lambda2) / lambda2,  m in [0,M), n in [0,N), N = L/a, b = L/M.
 *   Computed by the shear algorithm, Algorithm 1 of PAPER.md:852-900 (Sec. 4.1),
 *   with the frequency-domain trick of PAPER.md:902-919 and a Zak/factorization
 *   separable DGT (Eq. rect-flops) on hand-written sm_100a kernels;
 *   cuFFT is used only for the length-L FFTs of the frequency-shear branch, except where
 *   L = 180 x 4096 = d x (c q) (BASELINE config 4), whose length-L FFT and its adjoint run
 *   in the library's own kernels, and on the one-CTA path for short signals (DGT_ECUFFT
 *   cannot occur there).
 *
 * Conventions for every entry point:
 *   - Return value: a dgt_status (0 = DGT_OK).  A failed dgt_plan never returns a plan.
 *   - Complex arrays are interleaved (re, im) of the plan's precision: float for
 *     DGT_C64, double for DGT_C128.  Real arrays (DGT_REAL_INPUT) are float/double.
 *   - "device pointer" = CUDA global memory of the current device (e.g. a torch
 *     tensor's data_ptr()); "host pointer" = CPU memory (pinned memory makes the
 *     host entry points asynchronous-capable, pageable memory still works).
 *   - cuda_stream is a cudaStream_t passed as void* (NULL = legacy default stream).
 *   - No call takes ownership of caller memory.  The plan owns every table,
 *     cuFFT plan and workspace it allocates, and frees them in dgt_destroy.
 *   - Thread safety: distinct plans are independent.  One plan must not be
 *     executed concurrently from two streams (its workspace is shared).
 *   - Output is bitwise deterministic for a given (plan, f): no atomics, fixed
 *     reduction order.
 *   - Stream order: kernels may be launched with programmatic dependent launch; each waits
 *     for the preceding work on the stream before reading the caller's input or writing
 *     anything, so inputs produced by earlier kernels on the same stream are safe.
 */
#ifndef NSDGT_H
#define NSDGT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum dgt_status {
    DGT_OK = 0,
    DGT_EINVAL = 2,          /* null pointer, L/a/M <= 0, a or M not dividing L, lambda2 < 1,
                                lambda1 not in [0, lambda2), gcd(lambda1,lambda2) != 1 (unless
                                lambda = 0/1), W < 0, bad dtype/flags, f and c alias, or an
                                explicit shear that violates Eq. (modcond) */
    DGT_ENUMERIC = 3,        /* dgt_window_dual only: the window does not generate a frame on the
                                lattice (a factor of the frame operator is singular) */
    DGT_EILLEGAL_LENGTH = 4, /* L is not a multiple of L_min = lambda2*lcm(a,M) (Prop. minsig,
                                PAPER.md:580-615); dgt_last_lmin() reports L_min */
    DGT_ECUDA = 5,           /* a CUDA runtime call failed (dgt_last_error() has the text) */
    DGT_ECUFFT = 6,          /* a cuFFT call failed */
    DGT_ENOMEM = 7,          /* device or pinned-host allocation failed */
    DGT_EUNSUPPORTED = 8     /* lattice is valid but an inner transform length exceeds what the
                                kernels stage on chip (see DESIGN.md §5 limits) */
} dgt_status;

typedef enum dgt_dtype { DGT_C64 = 1, DGT_C128 = 2 } dgt_dtype;

typedef enum dgt_flags {
    DGT_REAL_INPUT = 1,      /* f is real (float/double); promoted to complex on load          */
    DGT_G_ON_HOST = 2,       /* g is a host pointer (else a device pointer)                      */
    DGT_SHEAR_PAPER = 4,     /* choose s1 by the proof's Eq. (s1choice) and
                                the least s0 solving Eq. (modcond), instead of the cost policy   */
    DGT_FORCE_GENERIC = 8    /* use the runtime-radix chunk kernels even where a specialised,
                                fused or one-CTA kernel exists (kernel_path 0)                   */
} dgt_flags;

typedef enum dgt_branch {
    DGT_BRANCH_SEPARABLE = 0, /* s = 0: plain separable DGT                                      */
    DGT_BRANCH_TIME = 1,      /* s0 = 0: Alg. 1 lines 7-15 (time shear only)                      */
    DGT_BRANCH_FREQ = 2       /* s0 != 0: Alg. 1 lines 16-31 (frequency shear, Fourier domain)    */
} dgt_branch;

/* Everything the planner decides (host-side integer arithmetic only). */
typedef struct dgt_lattice_info {
    int64_t L, a, M, lambda1, lambda2;   /* inputs                                                  */
    int64_t b, N, s, L_min;              /* b = L/M, N = L/a, s = b*lambda1/lambda2  */
    int64_t branch;                      /* dgt_branch                                              */
    int64_t s0, s1, b_r, a_r, M_r, N_r;  /* shear (Thm. shearform) and Alg. 1 line 17 quantities    */
    int64_t ia, iM, iN, ib;              /* inner separable lattice: time step, channels, N', b'    */
    int64_t c, d, p, q;                  /* Eqs. (cd),(pq) of the inner lattice   */
    int64_t C1, C2, C3, C4, C5, C6;      /* Alg. 1 constants (T: C1 only), reduced mod 2N / L        */
    int64_t chirp_sigma;                 /* sigma of the chirp applied on kernel-A load             */
    int64_t pre_sigma;                   /* sigma of the pre-FFT chirp (F-branch, 0 = none)         */
    int64_t chunk;                       /* signals per on-chip/L2 chunk (dgt_plan only)            */
    int64_t workspace_bytes;             /* device workspace owned by the plan (dgt_plan only)      */
    int64_t kernel_path;                 /* 0 chunk kernels, 2 fused persistent kernel, 4 the
                                            frequency-shear front path (L = 180 x 4096), 8 the
                                            one-CTA path for short signals (dgt_plan)          */
} dgt_lattice_info;

typedef struct dgt_plan_s* dgt_plan_t;

/* Host-only planner: feasibility, shear choice and integer constants for (L,a,M,lambda).
 * No GPU is touched.  flags: DGT_SHEAR_PAPER selects the proof's s1.  If force_shear
 * is nonzero, (s0, s1) are taken as given and validated against Eq. (modcond).
 * Errors: DGT_EINVAL, DGT_EILLEGAL_LENGTH. */
int dgt_lattice_plan(int64_t L, int64_t a, int64_t M, int64_t lambda1, int64_t lambda2,
                     int flags, int force_shear, int64_t s0, int64_t s1, dgt_lattice_info* out);

/* Create a plan on the current CUDA device.
 *   g         : window, L complex values of the plan precision (host if DGT_G_ON_HOST, else
 *               device).  Read during the call only; the caller may free it afterwards.
 *   dtype     : DGT_C64 or DGT_C128 (working and output precision).
 *   flags     : dgt_flags.
 *   max_chunk : signals per L2-resident chunk (0 = automatic from the L2 size).
 *   force_shear, s0, s1 : as in dgt_lattice_plan.
 * Precomputes (on cuda_stream, synchronised before return): chirps, the Alg. 1 window
 * transform and its Zak factorisation, phase tables.
 * Errors: DGT_EINVAL, DGT_EILLEGAL_LENGTH, DGT_EUNSUPPORTED, DGT_ECUDA, DGT_ECUFFT, DGT_ENOMEM. */
int dgt_plan(dgt_plan_t* out, int64_t L, int64_t a, int64_t M, int64_t lambda1, int64_t lambda2,
             const void* g, int dtype, int flags, int64_t max_chunk, int force_shear, int64_t s0,
             int64_t s1, void* cuda_stream);

/* Shear-OLA plan: the DGT on the lattice (a, M,
 * lambda) of length-L signals with an FIR window g of Lg taps, computed block-wise: blocks of
 * Lb samples (a multiple of L_min dividing L) are zero-extended to Lx >= Lb + Lg + 2a (a
 * multiple of L_min with a 7-smooth quotient) and transformed by the shear algorithm
 * with the window zero-extended to Lx; the block coefficients are overlap-added.  The result is
 * exactly Eq. (DGT) with the full-length window that equals g on its support and 0 elsewhere.
 * Lb = 0 picks the smallest admissible Lb >= max(16 Lg, 2^18) (throughput); a short Lb bounds
 * the processing delay of block-wise / streaming use.
 * g: Lg complex of dtype in FIR order -- entries [0, ceil(Lg/2)) are times 0, 1, ..., the rest
 * times -floor(Lg/2), ..., -1 (host memory with DGT_G_ON_HOST, else device).  The returned plan
 * runs dgt_execute / dgt_execute_host / dgt_plan_query / dgt_destroy; dgt_execute_inverse and
 * dgt_window_dual return DGT_EUNSUPPORTED for it.  When Lx would not be shorter than L the
 * function returns an ordinary full-length plan of the zero-extended window.
 * Errors: as dgt_plan, DGT_EINVAL for Lg outside [1, L] or an Lb that is not a multiple of
 * L_min dividing L. */
int dgt_plan_fir(dgt_plan_t* out, int64_t L, int64_t a, int64_t M, int64_t lambda1, int64_t lambda2,
                 const void* g, int64_t Lg, int64_t Lb, int dtype, int flags, void* cuda_stream);

/* Multiwindow plan (the comparison algorithm of, Sec. 3.1):
 * the same transform Eq. (DGT) on the lattice (a, M, lambda1/lambda2), computed through the
 * co-set decomposition of Prop. mwindec -- lambda2 separable DGTs on the lattice (lambda2 a, b)
 * with the windows g_m = M_{m s mod b} T_{m a} g, m < lambda2, joined by the phases of
 * Eq. (mw_phases): c(k, n) = exp(-2 pi i nt (lambda2 a) (m s mod b) / L) d_m(k, nt) for
 * n = nt lambda2 + m (reading Z12: m = n mod lambda2).  Its cost grows linearly with lambda2,
 * the shear algorithm's does not (Fig. 2).  The windows g_m are made on the
 * host in fp64 (exact integer phase indices), rounded once to dtype; each inner transform runs
 * the plan path of dgt_plan for its separable lattice.  Arguments as dgt_plan (flags:
 * DGT_REAL_INPUT, DGT_G_ON_HOST, DGT_FORCE_GENERIC).  The returned plan runs dgt_execute /
 * dgt_execute_host / dgt_plan_query (kernel_path = 32 + the inner plans' path) / dgt_destroy;
 * dgt_execute_inverse and dgt_window_dual return DGT_EUNSUPPORTED.
 * Errors: as dgt_plan. */
int dgt_plan_multiwindow(dgt_plan_t* out, int64_t L, int64_t a, int64_t M, int64_t lambda1, int64_t lambda2,
                         const void* g, int dtype, int flags, void* cuda_stream);

/* c = DGT(f) for W signals.  f: device, W x L (complex, or real with DGT_REAL_INPUT),
 * signal-major.  c: device, W x M x N complex, n fastest (c[(w*M + m)*N + n]).  Fully
 * overwritten.  Asynchronous and stream-ordered on cuda_stream; allocates nothing.
 * W = 0 is a no-op.  Errors: DGT_EINVAL (null/aliasing), DGT_ECUDA, DGT_ECUFFT. */
int dgt_execute(dgt_plan_t plan, const void* f, void* c, int64_t W, void* cuda_stream);

/* Synthesis (inverse DGT) with the plan's window as the synthesis window gamma
 * (the inversion formula of PAPER.md:171-175, Sec. 2.1):
 *   f_w(l) = sum_{n<N} sum_{m<M} c_w(m,n) gamma((l - a n) mod L) exp(+2 pi i l (m + w(n)) / M),
 * i.e. the adjoint of dgt_execute.  A plan built with the canonical dual window S^{-1} g
 * inverts the DGT of a plan built with g.  c: device, W x M x N complex (n fastest), read
 * only.  f: device, W x L complex of the plan's dtype (always complex, also for
 * DGT_REAL_INPUT plans), fully overwritten.  Asynchronous and stream-ordered; allocates nothing
 * (the synthesis workspace is made by dgt_plan).  Runs the fused adjoint kernel on the fused
 * lattices and the generic (adjoint) kernels elsewhere.  W = 0 is a no-op.
 * Errors: DGT_EINVAL (null/aliasing, W < 0), DGT_ECUDA, DGT_ECUFFT, DGT_ENOMEM. */
int dgt_execute_inverse(dgt_plan_t plan, const void* c, void* f, int64_t W, void* cuda_stream);

/* Canonical dual (kind 0, S^{-1} g) or canonical tight (kind 1, S^{-1/2} g) window of the plan's
 * window on the plan's lattice: Alg. 2 of PAPER.md:951-994 -- the plan's shear
 * (chirp, and for the frequency shear the length-L FFT), the separable dual/tight window by the
 * factorisation of the frame operator (per (r, nu) the p x p matrix
 * H = Gamma Gamma^H, dual factor H^{-1} Gamma / M', tight factor H^{-1/2} Gamma / sqrt(M')),
 * then the shear undone.  fp64 throughout, rounded once to the plan's dtype.
 * out: L complex of the plan's dtype, host memory when flags has DGT_G_ON_HOST, else device.
 * Synchronous on cuda_stream; allocates and frees its fp64 workspace.  S is the frame operator
 * of Eq. (frameop); a plan built with the dual window inverts the DGT
 * through dgt_execute_inverse.
 * Errors: DGT_EINVAL, DGT_EUNSUPPORTED (p > 8 or q > 64; tight with p > 2), DGT_ENUMERIC,
 * DGT_ECUDA, DGT_ECUFFT, DGT_ENOMEM. */
int dgt_window_dual(dgt_plan_t plan, int kind, void* out, int flags, void* cuda_stream);

/* End-to-end variant with HOST buffers: copies f (host, W x L) to the device, runs the
 * transform and copies c (host, W x M x N) back, chunk by chunk with the copies overlapped
 * on two extra streams.  Returns after c is complete on the host (synchronous), also on an
 * error once a copy was enqueued (the caller may reuse its buffers on return).  The staging
 * buffers (two slots of ~64 MB of output) and copy streams are made by the plan constructors;
 * this call allocates nothing.  Errors: as dgt_execute. */
int dgt_execute_host(dgt_plan_t plan, const void* f_host, void* c_host, int64_t W, void* cuda_stream);

/* Release everything the plan owns.  The caller must have synchronised its streams. */
int dgt_destroy(dgt_plan_t plan);

/* Copy the plan's planner record (with chunk, workspace and kernel path filled in). */
int dgt_plan_query(dgt_plan_t plan, dgt_lattice_info* info);

/* Number of this library's own kernel launches (and memsets) one dgt_execute of W signals
 * issues; the frequency-shear path's cuFFT calls are library launches and not counted.
 * Used by bench.py for its gpu_launches claim. */
int64_t dgt_launches_per_execute(dgt_plan_t plan, int64_t W);

/* Per-kernel profiling (used by bench.py for its roofline line).  After dgt_profile_begin,
 * every dgt_execute on this plan records a CUDA event pair around each kernel launch on
 * the launch stream; dgt_profile_end synchronises those events, fills up to max_stats
 * records (one per kernel kind, *n_stats of them) and stops recording.  bytes/flops are
 * ALGORITHMIC: the share of "f, window factors and c moved once" and of the
 * Table-1 flop model that each kernel kind is responsible for. */
typedef struct dgt_kernel_stat {
    char name[32];
    int64_t launches;
    double ms;      /* summed CUDA-event duration of all launches of this kind */
    double bytes;   /* summed algorithmic bytes */
    double flops;   /* summed model flops */
} dgt_kernel_stat;
int dgt_profile_begin(dgt_plan_t plan);
int dgt_profile_end(dgt_plan_t plan, dgt_kernel_stat* stats, int max_stats, int* n_stats);

/* Static text for a status code; dgt_last_error() gives the last failure's detail
 * (thread-local); dgt_last_lmin() the L_min of the last DGT_EILLEGAL_LENGTH. */
const char* dgt_strerror(int status);
const char* dgt_last_error(void);
int64_t dgt_last_lmin(void);

/* Library version string. */
const char* dgt_version(void);

#ifdef __cplusplus
}
#endif
#endif /* NSDGT_H */
