/*
 * adaptsolve.h -- C ABI of libadaptsolve.so, a B200-native (sm_100a)
 * implementation of the adaptive solver for A X = B of
 *   C. Sanderson, R. Curtin, "An Adaptive Solver for Systems of Linear
 *   Equations", arXiv 2007.11208 (cited as P:<line> of PAPER.md).
 *
 * The operation (Eq. 1/2 with m = n): given a square n x n matrix A
 * and n x nrhs right-hand sides B, find X with A X = B.  The solver detects,
 * in this order, a banded structure, a lower or upper
 * triangular structure, or a likely symmetric positive definite
 * matrix (Fig. 4), and uses banded LU, triangular
 * substitution (Eq. 3), Cholesky (on failure the general
 * solver) or LU with partial pivoting.  Each path estimates the
 * 1-norm reciprocal condition number; if a factorization fails or
 * rcond < 0.5 eps an SVD-based minimum-norm solution is computed
 * instead, unless disabled.
 *
 * Conventions (all entry points):
 *  - Storage: column-major, element (i,j) at base[i + j*ld], zero-based
 *    (P:120-126).
 *  - Residency: A, B, X are DEVICE pointers (cudaMalloc / torch CUDA tensors)
 *    unless the entry point says otherwise.  Host out-pointers (info_flags,
 *    rcond, report) may be NULL.
 *  - Ownership: A and B are read-only and owned by the caller.  X is owned by
 *    the caller and must hold ldb*nrhs elements; X == B (exact alias, in-place
 *    solve) is allowed, any other overlap is undefined.  Factors live in a
 *    library-owned workspace cached per (device, stream, dtype, n, nrhs, lda,
 *    ldb, options, 16-byte alignment of A: aligned matrices with 16-byte
 *    aligned columns take the TMA detection pass, n >= 1024) and released by
 *    as_release_all().  Calls on different
 *    streams therefore never share a workspace; calls on one stream are
 *    ordered by the stream.
 *  - Streams: all device work is enqueued on `stream`; the call synchronizes
 *    that stream exactly once (to read the device-resident report), and not at
 *    all for as_solve_async().
 *  - Errors: 0 = X valid; -i = the i-th argument is illegal (LAPACK
 *    convention, nothing enqueued); positive AS_ERR_* codes below; CUDA errors
 *    are returned as AS_ERR_CUDA_BASE + cudaError_t.
 */
#ifndef ADAPTSOLVE_H
#define ADAPTSOLVE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum { AS_F64 = 0, AS_F32 = 1 } as_dtype;

/* ---- info_flags bits ---------------------------------------------------- */
/* bits 0-3: literal detection verdicts; each is the exact
 * predicate of the paper, evaluated on the whole matrix (bit-exact vs the
 * oracle).  After an early exit (all four false) they are all 0. */
#define AS_FLAG_BANDED        0x1u   /* band capacity <= 25% of n^2 (Z2/Z3) */
#define AS_FLAG_LOWER         0x2u   /* all elements above the diagonal are 0 */
#define AS_FLAG_UPPER         0x4u   /* all elements below the diagonal are 0 */
#define AS_FLAG_SPD_CANDIDATE 0x8u   /* Fig. 4 likely_sympd returned true */
/* bits 4-7: method that produced X (AS_METHOD_*) */
#define AS_FLAG_METHOD_SHIFT  4
#define AS_FLAG_METHOD_MASK   0xF0u
#define AS_FLAG_CHOL_FAILED   (1u << 8)   /* POTRF failed -> general LU */
#define AS_FLAG_SINGULAR      (1u << 9)   /* primary factor had an exact zero pivot */
#define AS_FLAG_RCOND_LOW     (1u << 10)  /* the gate fired: singular or !(rcond >= thr) */
#define AS_FLAG_FALLBACK      (1u << 11)  /* X is the SVD minimum-norm solution */
#define AS_FLAG_POORLY_COND   (1u << 12)  /* gate fired with AS_OPT_NO_FALLBACK: X is the primary solution */
#define AS_FLAG_NONFINITE     (1u << 13)  /* a NaN/Inf was seen: in A or B under AS_OPT_CHECK_FINITE (the call
                                             returns AS_ERR_NONFINITE before any factorization), or in the
                                             fallback's singular values (non-finite input reached the SVD, whose
                                             minimum-norm solution is then undefined: AS_ERR_NONFINITE).
                                             (robustness to floating-point limits), Z28/Z29 */
#define AS_FLAG_SVD_NOCONV    (1u << 14)  /* Jacobi hit max_sweeps */
#define AS_FLAG_RANK_DEF      (1u << 15)  /* fallback effective rank < n */
#define AS_FLAG_SYMMETRIC     (1u << 16)  /* A is exactly symmetric (evaluated only with AS_OPT_SYM_INDEF, n <= 128) */

/* ---- methods ------------------------------------------------------------- */
#define AS_METHOD_NONE      0
#define AS_METHOD_BAND      1   /* GBTRF/GBCON/GBTRS */
#define AS_METHOD_TRI_LOWER 2   /* TRCON/TRTRS, forward substitution (Eq. 3) */
#define AS_METHOD_TRI_UPPER 3   /* TRCON/TRTRS, back-substitution */
#define AS_METHOD_CHOL      4   /* POTRF/POCON/POTRS */
#define AS_METHOD_LU        5   /* GETRF/GECON/GETRS */
#define AS_METHOD_SVD       6   /* QR + one-sided Jacobi min-norm */
#define AS_METHOD_LDLT      7   /* symmetric indefinite L D L^T, Bunch-Kaufman (xSYTRF/xSYCON/xSYTRS; the paper's
                                   future work P:741-743; AS_OPT_SYM_INDEF, n <= 128) */

/* ---- options ------------------------------------------------------------- */
#define AS_OPT_NO_FALLBACK  0x1u   /* disable the SVD fallback */
#define AS_OPT_FORCE_METHOD 0x2u   /* use opt.force_method (1..5) instead of the detected one */
#define AS_OPT_CHECK_FINITE 0x4u   /* reject NaN/Inf in A or B (AS_ERR_NONFINITE, flag AS_FLAG_NONFINITE, X untouched):
                                      the detection pass then reads every element of A (no early exit) and B is
                                      scanned once; off by default (the paper is silent on non-finite input, Z28) */
#define AS_OPT_FULLSCAN     0x8u   /* detection never exits early; kl/ku always exact */
#define AS_OPT_SYM_INDEF    0x20u  /* the symmetric-indefinite specialisation (Z30): for
                                      n <= 128 an exactly symmetric matrix that is not likely-sympd (or whose
                                      Cholesky fails) is solved by Bunch-Kaufman L D L^T on the one-block
                                      solver; larger systems ignore the option */
#define AS_OPT_SKIP_DETECT  0x10u  /* with AS_OPT_FORCE_METHOD (LU, CHOL, TRI_*): no structure detection at all --
                                      the "standard solver" of the paper's comparison; report bits
                                      0..3 are 0.  Illegal (-9) without FORCE_METHOD or with AS_METHOD_BAND,
                                      which needs the detected kl/ku. */

/* ---- return codes ------------------------------------------------------- */
#define AS_OK                        0
#define AS_ERR_SINGULAR_NO_FALLBACK  1   /* exact zero pivot and NO_FALLBACK: X unspecified */
#define AS_ERR_SVD_NOT_CONVERGED     2   /* fallback Jacobi hit max_sweeps (X is its last iterate) */
#define AS_ERR_NONFINITE             3   /* NaN/Inf input (AS_OPT_CHECK_FINITE) or non-finite singular values in the
                                            fallback: X unspecified, flags carry AS_FLAG_NONFINITE */
#define AS_ERR_NOT_IMPLEMENTED       4
#define AS_ERR_NO_DEVICE             5
#define AS_ERR_CUDA_BASE             1000

typedef struct {
    uint32_t flags;            /* AS_OPT_* */
    int32_t force_method;      /* AS_METHOD_BAND..AS_METHOD_LU when AS_OPT_FORCE_METHOD */
    double rcond_threshold;    /* < 0: 0.5 eps of the dtype */
    double lsq_cutoff;         /* < 0: n*eps (Z14): keep sigma_k > cut * sigma_max */
    int32_t max_sweeps;        /* <= 0: 30 */
    int32_t reserved;
} as_options;

typedef struct {
    uint32_t flags;            /* AS_FLAG_* as above */
    int32_t method;            /* method that produced X (AS_METHOD_*) */
    int32_t primary_method;    /* structured / LU path that ran (before any fallback) */
    int32_t sweeps;            /* Jacobi sweeps executed by the fallback (0 otherwise) */
    int64_t kl, ku;            /* band extent; -1 unless banded (exact always with FULLSCAN) */
    double rcond;              /* primary path's estimate (0 if singular); never the SVD's (Z25) */
    double anorm;              /* 1-norm of A used by the estimate */
    int64_t rank;              /* fallback effective rank, -1 if the fallback did not run */
    int64_t info;              /* 1 + first zero-pivot column of the primary factor, else 0 */
    int64_t chol_fail_col;     /* 0-based column where POTRF failed (valid with CHOL_FAILED) */
} as_report;

typedef struct {
    uint32_t flags;            /* AS_FLAG_BANDED | LOWER | UPPER | SPD_CANDIDATE */
    int32_t method;            /* first-match dispatch */
    int64_t kl, ku;            /* exact if banded or FULLSCAN, else -1 */
    double max_diag;           /* Fig. 4 max_diag (largest positive diagonal entry) */
    int32_t nonfinite_seen;    /* 1 if A holds a NaN/Inf (only evaluated with AS_OPT_CHECK_FINITE, else 0) */
    int32_t reserved;
} as_structure;

/*
 * as_solve: the north-star entry point.  Solves A X = B adaptively.
 *   dt        AS_F64 (double) or AS_F32 (float); all buffers of that type.
 *   A         device, n x n, column-major, lda >= max(1,n); read-only.
 *   B         device, n x nrhs, ldb >= max(1,n); read-only (unless X == B).
 *   X         device, n x nrhs with leading dimension ldb (no separate ldx).
 *   info_flags host, may be NULL: AS_FLAG_* of the report.
 *   rcond     host, may be NULL: report.rcond.
 *   stream    cudaStream_t (0 = legacy default stream).
 * Returns AS_OK / AS_ERR_* / -i.  n == 0 or nrhs == 0: returns 0 at once with
 * flags 0 and rcond 1.
 */
int as_solve(as_dtype dt, const void* A, int64_t lda, int64_t n, const void* B, int64_t ldb, int64_t nrhs,
             void* X, uint32_t* info_flags, double* rcond, void* stream);
int as_solve_f64(const double* A, int64_t lda, int64_t n, const double* B, int64_t ldb, int64_t nrhs,
                 double* X, uint32_t* info_flags, double* rcond, void* stream);
int as_solve_f32(const float* A, int64_t lda, int64_t n, const float* B, int64_t ldb, int64_t nrhs,
                 float* X, uint32_t* info_flags, double* rcond, void* stream);

/* as_solve_ex: as_solve with options (opt may be NULL = defaults) and the
 * full report (rep, host, may be NULL).  sigma_out: optional DEVICE buffer of
 * n elements (dtype) receiving the fallback's singular values, descending
 * (untouched if the fallback does not run). */
int as_solve_ex(as_dtype dt, const void* A, int64_t lda, int64_t n, const void* B, int64_t ldb, int64_t nrhs,
                void* X, const as_options* opt, as_report* rep, void* sigma_out, void* stream);

/* as_solve_async: enqueue the whole adaptive solve (one CUDA-graph launch,
 * dispatch on device-resident flags) and return without synchronizing.  The
 * report is written to `rep_dev` (a DEVICE as_report*, may be NULL) when the
 * stream reaches it.  Used by the benchmark's device-timed loop. */
int as_solve_async(as_dtype dt, const void* A, int64_t lda, int64_t n, const void* B, int64_t ldb, int64_t nrhs,
                   void* X, const as_options* opt, as_report* rep_dev, void* sigma_out, void* stream);

/* as_solve_batched: `batch` independent systems A_b X_b = B_b of one shape (
 * the paper's workload is "1000 unique random systems" per size), each solved by the
 * full adaptive flowchart (detection, dispatch, factor, rcond gate, SVD fallback) with its own
 * verdict.  n <= 128 and nrhs <= 16: ONE thread block per system, matrix in shared memory, one
 * launch for the whole batch (detection reads every element, so kl/ku are always exact); larger
 * shapes: one single-system graph launch per system (then ldx must equal ldb).
 *   A, B, X   DEVICE, column-major; system b at A + b*strideA (leading dimension lda), B + b*strideB
 *             (ldb), X + b*strideX (ldx); strides in elements, strideA >= lda*n etc.  A, B read-only;
 *             X == B (same strides) allowed.
 *   opt       host, may be NULL (AS_OPT_SKIP_DETECT is illegal here).
 *   rep       DEVICE array of `batch` reports, may be NULL; ret: DEVICE int32[batch] per-system
 *             return codes (AS_OK / AS_ERR_*), may be NULL; sigma_out: DEVICE batch*n fallback
 *             singular values (system b at b*n, descending), may be NULL.
 * No host synchronization: everything is enqueued on `stream`.  Returns 0, -i (illegal i-th
 * argument, nothing enqueued) or AS_ERR_CUDA_BASE + e. */
int as_solve_batched(as_dtype dt, int64_t n, int64_t nrhs, int64_t batch, const void* A, int64_t lda, int64_t strideA,
                     const void* B, int64_t ldb, int64_t strideB, void* X, int64_t ldx, int64_t strideX,
                     const as_options* opt, as_report* rep, int32_t* ret, void* sigma_out, void* stream);

/* as_solve_host: same contract with HOST buffers A, B, X (pageable or
 * pinned); copies H2D, solves, copies X D2H on `stream`.  The end-to-end entry
 * point timed by bench.py's "e2e" leg. */
int as_solve_host(as_dtype dt, const void* A, int64_t lda, int64_t n, const void* B, int64_t ldb, int64_t nrhs,
                  void* X, const as_options* opt, as_report* rep, void* stream);

/* as_detect: structure detection only (P:164-175, P:328-343, P:382-384,
 * Fig. 4).  detect_flags: AS_OPT_FULLSCAN and/or AS_OPT_CHECK_FINITE (which
 * implies a full scan and fills out->nonfinite_seen), or 0.  out: host. */
int as_detect(as_dtype dt, const void* A, int64_t lda, int64_t n, uint32_t detect_flags, as_structure* out,
              void* stream);

/* ---- test-only / diagnostic exports: only in libadaptsolve_debug.so, the same
 * sources built with -DAS_DEBUG (SURVEY 8(b) "Test-only exports").  Never used by
 * the solve, the benchmark or smoke(). */
#ifdef AS_DEBUG
/* as_debug_factor: test-only (T3 reconstruction tests; never used by the
 * solve or the bench).  Runs the primary factorization `method` alone, with
 * the launchers the solve uses (AS_METHOD_LU: xGETRF, P:505-515;
 * AS_METHOD_CHOL: xPOTRF), on device A (read-only, ld lda) and
 * copies the factors into caller DEVICE buffers: W (n*n, ld n; LU: L\U with
 * unit-diagonal L, every interchange applied to every column; CHOL: L in the
 * lower triangle, the strict upper triangle unspecified) and, for LU, ipiv
 * (int64, n, 0-based: row j was interchanged with row ipiv[j], in order
 * j = 0..n-1).  kl/ku are unused.  Enqueued on `stream`, which it
 * synchronises once.  Returns 0, info > 0 (LU: 1 + first exact zero pivot;
 * CHOL: 1 + first column with a non-positive or NaN pivot), or a negative
 * error: -1 dt, -3 A, -4 lda, -5 n <= 0, -8 W, -9 ipiv (not device pointers),
 * -AS_ERR_NOT_IMPLEMENTED for AS_METHOD_BAND (the band factors are checked
 * through the solve parity tests). */
int64_t as_debug_factor(as_dtype dt, int32_t method, const void* A, int64_t lda, int64_t n, int64_t kl, int64_t ku,
                        void* W, int64_t* ipiv, void* stream);

/* Diagnostics: %globaltimer stamps (ns) recorded by the last call's kernels
 * at phase boundaries (out: 16 values; 0 = not recorded). */
int as_debug_timestamps(unsigned long long* out16);

/* Diagnostics (only with the environment variable AS_LU_TRACE set when the library loads):
 * per 128-column LU block k, slots 4k+0 trailing GEMM (main stream), 4k+1 panel 1, 4k+2 panel 2,
 * 4k+3 look-ahead GEMM; tmin = first CTA start, tmax = last CTA end (%globaltimer ns) of the last
 * factorization.  Host arrays of `cap` entries.  Returns the number of slots written, or -1 when
 * tracing is off. */
/* Diagnostics (not part of the solve path): average device time in microseconds of one panel
 * factorization of the column block k0 .. k0+nbp of the n x n column-major matrix W (device,
 * leading dimension ldw), restored from the device copy Wsrc before each of `iters` launches (the
 * first launch is not averaged when iters > 1).  kind 0: LU register/cluster panel,
 * 1: LU cooperative panel, 2: Cholesky cluster panel, 3: Cholesky POTF2 + L21.
 * dbg: ablation bits of the LU register panel (1 skip interchanges on other columns, 2 skip the
 * deferred update, 8 skip the column loop) -- timing studies only, results are then wrong;
 * kind 3: 2 = POTF2 only (no L21), 4 = restore only the panel columns (L2 stays warm).
 * Returns < 0 on an illegal argument or a CUDA error (-error code). */
double as_debug_panel_time(int dtype, int kind, void* W, int64_t ldw, int64_t n, int64_t k0, int nbp, const void* Wsrc,
                           int iters, int dbg);
int as_debug_lu_trace(unsigned long long* tmin, unsigned long long* tmax, int cap);

#endif /* AS_DEBUG */

/* Benchmark instrumentation.  When enabled, plans built afterwards record
 * CUDA events (graph event-record nodes) around the top-level stages of the
 * solve; as_last_stage_ms() returns the device-timed durations (ms) of the
 * last synchronous call on this thread: [0] detection (diag + tile-pair
 * pass + dispatch), [1] the method body (factor + rcond estimate),
 * [2] gate + post (primary solve or SVD fallback), [3] whole graph.
 * Returns 0, or -1 if the last plan was not instrumented. */
void as_set_instrumentation(int enable);
int as_last_stage_ms(double* out4);

/* Execution mode of plans built afterwards: 0 (default) = one CUDA graph with
 * device-side conditional nodes, one host sync per call; 1 = eager profiling
 * mode: the same kernels launched directly, branch decisions read back by the
 * host (several syncs; for kernel-by-kernel ncu launch lists only). */
void as_set_exec_mode(int eager);

/* Roofline denominator probe (benchmark only, not part of a solve): fp64
 * tensor-core (DMMA) throughput in TFLOP/s of a register-resident MMA loop. */
double as_measure_fp64_peak(int iters, void* stream);
/* Benchmark only: TFLOP/s of the library's C -= A op(B) kernel (dtype AS_F64 / AS_F32)
 * on internal zero-filled buffers, M x N x K, op(B) = B^T if trans_b. */
double as_bench_gemm(int dtype, int64_t M, int64_t N, int64_t K, int trans_b, int iters);

/* Workspace bytes (device) a plan for this shape and these AS_OPT_* option
 * flags allocates (FORCE_METHOD reserves room for a forced band factor of
 * any width).  Returns -1 on an illegal argument (dt, n < 0, nrhs < 0). */
int64_t as_workspace_bytes(as_dtype dt, int64_t n, int64_t nrhs, uint32_t opts);
/* Number of kernel launches the last as_solve* on this thread enqueued
 * (graph kernel nodes executed are not observable; this counts the nodes of
 * the graph branches the device took, as recorded by the finalize kernel). */
int64_t as_last_kernel_nodes(void);
/* Free all cached plans/workspaces (all devices). */
void as_release_all(void);
const char* as_strerror(int code);
int as_version(void);

#ifdef __cplusplus
}
#endif
#endif /* ADAPTSOLVE_H */
