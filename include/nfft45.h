/*
 * nfft45.h — C ABI of the B200-native type-1/2/4/5 NFFT (arXiv 1604.06236).
 *
 * The reference (`nufft1d` 0.1.0, pure Python/numpy) has no FFI layer; its
 * boundary is the Python API.  Each entry point below replaces one reference
 * function (cited as pkg/src/nufft1d/<file>:<line>) and is bound through
 * ctypes by `paper_1604_06236_b200/_lib.py`, which keeps the reference's
 * Python names, defaults and exceptions.
 *
 * Conventions
 *  - complex128 arrays are interleaved (re, im) doubles (`double2`), passed
 *    as `double*`; every vector is 1-D contiguous; batched arrays are
 *    [batch][len] row-major (one contiguous signal per row).
 *  - "dev" pointers are CUDA device pointers on the handle's device; "host"
 *    pointers are ordinary host memory.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  Calls are
 *    stream-ordered and asynchronous unless noted "synchronizes".
 *  - Node-indexed vectors are in the caller's node order (grid.py:38-41).
 *  - Every call returns an nfft45_status; on failure the thread-local
 *    message from nfft45_last_error() says why.
 *  - Handles are immutable after creation and may be shared by threads;
 *    concurrent calls on one handle are safe (per-call scratch is
 *    stream-ordered), and every kernel is deterministic (no floating-point
 *    atomics), so results are bitwise reproducible.
 */
#ifndef NFFT45_H
#define NFFT45_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes; the Python shim maps them onto errors.py:4-45. */
typedef enum {
  NFFT45_OK = 0,
  NFFT45_ERR_OUT_OF_RANGE = 1,          /* OutOfRangeError          errors.py:8   */
  NFFT45_ERR_DUPLICATE_NODE = 2,        /* DuplicateNodeError       errors.py:12  */
  NFFT45_ERR_NON_POSITIVE_DAMPING = 3,  /* NonPositiveDampingError  errors.py:16  */
  NFFT45_ERR_LENGTH_MISMATCH = 4,       /* LengthMismatchError      errors.py:20  */
  NFFT45_ERR_SIZE_MISMATCH = 5,         /* SizeMismatchError        errors.py:24  */
  NFFT45_ERR_KERNEL_OVERFLOW = 6,       /* KernelOverflowError      errors.py:28  */
  NFFT45_ERR_SINGULAR_DERIVATIVE = 7,   /* SingularDerivativeError  errors.py:32  */
  NFFT45_ERR_NON_CONVERGENCE = 8,       /* NonConvergenceError      errors.py:40  */
  NFFT45_ERR_INVALID_ARGUMENT = 9,      /* ValueError (grid.py:143-150)           */
  NFFT45_ERR_CUDA = 10,                 /* CUDA runtime failure                   */
  NFFT45_ERR_NO_DEVICE = 11,            /* no usable sm_100 device                */
  NFFT45_ERR_SINGULAR_MATRIX = 12       /* SingularMatrixError      errors.py     */
} nfft45_status;

typedef struct nfft45_grid nfft45_grid;  /* device-resident node set */
typedef struct nfft45_plan nfft45_plan;  /* device-resident inverse plan */

/* ----------------------------------------------------------------- misc */

/* Thread-local description of the last failure on this thread. */
const char* nfft45_last_error(void);
/* ABI version (major*100 + minor). */
int nfft45_version(void);
/* Number of launches of this library's kernels so far in this process
 * (all threads); used by bench.py to report `gpu_launches`. */
int64_t nfft45_launch_count(void);

/* Per-launch device timing (for bench.py's roofline): while enabled, every
 * kernel launch of this library is bracketed by CUDA events recorded on the
 * launching stream.  nfft45_profile_read synchronizes on them, writes lines
 * "<kernel> <launches> <total_ms>\n" into buf (NUL-terminated, at most cap
 * bytes), clears the record and returns the full text length. */
int nfft45_profile_enable(int on);
int nfft45_profile_read(char* buf, int64_t cap);

/* --------------------------------------------------------------- grids */

/* validate_grid(instants, min_gap) — grid.py:64-96.  Host-side range /
 * finiteness / circular-gap check; writes the stable ascending sort order
 * into order_host[Q].  Errors: OUT_OF_RANGE, DUPLICATE_NODE. */
int nfft45_validate_grid(const double* t_host, int64_t Q, double min_gap,
                         int64_t* order_host);

/* Upload a validated node set (NonuniformGrid, grid.py:35-61) to `device`:
 * sorted instants, the permutation, and the compensated instant sum used by
 * lagrange.py:92.  Synchronizes (host copies). */
int nfft45_grid_create(const double* t_host, const int64_t* order_host, int64_t Q,
                       int device, nfft45_grid** out);
void nfft45_grid_destroy(nfft45_grid* g);
int64_t nfft45_grid_size(const nfft45_grid* g);

/* ------------------------------------------------------ forward NFFTs */

/* nfft_type1(grid, amplitudes, R, kernel) — forward.py:26-64.
 * out[b][p] = sum_q a[b][q] e^{-2 pi i p t_q}, p < R; Gaussian gridding at
 * oversampling 2 with half-width m (gridding.py:75-98).
 * a_dev: [batch][Q]; out_dev: [batch][R]. */
int nfft45_type1(const nfft45_grid* g, const double* a_dev, int64_t batch, int64_t R,
                 int m, double* out_dev, void* stream);

/* nfft_type2(coefficients, grid, kernel) — forward.py:67-102.
 * out[b][q] = sum_p S[b][p] e^{+2 pi i p t_q}; S_dev: [batch][P]; out_dev:
 * [batch][Q]. */
int nfft45_type2(const nfft45_grid* g, const double* S_dev, int64_t batch, int64_t P,
                 int m, double* out_dev, void* stream);

/* nonuniform_conv(grid, amplitudes, lam_coefficients, P, kernel) —
 * forward.py:133-162.  lam_dev: complex [R], R a multiple of P (else
 * SIZE_MISMATCH); a_dev: [batch][Q]; out_dev: [batch][P]. */
int nfft45_nonuniform_conv(const nfft45_grid* g, const double* a_dev, int64_t batch,
                           const double* lam_dev, int64_t R, int64_t P, int m,
                           double* out_dev, void* stream);

/* nfft_type1_direct / nfft_type2_direct — forward.py:105-130.  Exact O(RQ)
 * sums with exactly reduced phases (oracle-quality; for tests/residuals). */
int nfft45_type1_direct(const nfft45_grid* g, const double* a_dev, int64_t batch,
                        int64_t R, double* out_dev, void* stream);
int nfft45_type2_direct(const nfft45_grid* g, const double* S_dev, int64_t batch,
                        int64_t P, double* out_dev, void* stream);

/* Unnormalised DFTs along the last axis (np.fft.fft / forward.py:21-23):
 * sign = -1: X_k = sum_j x_j e^{-2 pi i jk/N};  sign = +1: e^{+...}, no 1/N.
 * in_dev / out_dev: [batch][N]; in-place allowed. */
int nfft45_dft(const double* in_dev, double* out_dev, int64_t batch, int64_t N, int sign,
               void* stream);

/* ------------------------------------------------------- CG baseline */

/* cg_solve(grid, rhs, which, tol, max_iter, spread_width) — baselines.py:108-181.
 * CGNR, unpreconditioned: each iteration applies the system matrix and its
 * Hermitian transpose (one type-1 and one type-2 NFFT of width m).  kind 4:
 * A = type1 (amplitudes -> spectrum), kind 5: A = type2 (coefficients ->
 * samples).  rhs_dev, x_dev: [batch][P] device (P = grid size); every row runs
 * its own recurrence.  Host outputs per row: iterations, converged (0/1),
 * relres = ||r|| / ||b||, stalled (|A p| = 0 stop; may be NULL).  tol <= 0 or
 * an unknown kind: INVALID_ARGUMENT. */
int nfft45_cg_solve(const nfft45_grid* g, int kind, const double* rhs_dev, int64_t batch, double tol,
                    int64_t max_iter, int m, double* x_dev, int64_t* iterations, int* converged,
                    double* relres, int* stalled, void* stream);

/* ge_solve(DenseSystem) — baselines.py:64-105.  Dense right-looking
 * Gaussian elimination with partial pivoting on the device, in the
 * reference's operation order.  A_dev: complex [n][n] row-major and b_dev:
 * complex [n], both device and OVERWRITTEN (U and the eliminated rhs);
 * x_dev: complex [n].  A pivot magnitude below pivot_floor (1e-300) at
 * elimination step k < n-1, or on the last diagonal entry (k = n-1), returns
 * SINGULAR_MATRIX; *bad_step (host) is that k, or n on success, and
 * *bad_pivot its magnitude. */
int nfft45_ge_solve(double* A_dev, double* b_dev, int64_t n, double* x_dev, double pivot_floor,
                    int64_t* bad_step, double* bad_pivot, void* stream);

/* ------------------------------------------------- Lagrange quantities */

/* compute_v_samples(grid, params) — lagrange.py:57-75. v_dev: complex [P]. */
int nfft45_v_samples(const nfft45_grid* g, double damping_a, int eta, int m,
                     double* v_dev, void* stream);

/* Extension (fractional oversampling, BASELINE config 5's eta = 1.5): the
 * same with R = number of log-series terms given directly (the reference
 * requires R = eta P with integer eta, grid.py:143-144, forward.py:149-154;
 * here any R >= 2, the fold onto P summing a partial last slice). */
int nfft45_v_samples_terms(const nfft45_grid* g, double damping_a, int64_t R, int m,
                           double* v_dev, void* stream);

/* kernel_samples_from_v(v, grid) — lagrange.py:78-97.  ks = exp(i pi P +
 * 2 pi i sum t + v).  Synchronizes to apply the KERNEL_OVERFLOW guard. */
int nfft45_kernel_samples(const nfft45_grid* g, const double* v_dev, double* ks_dev,
                          void* stream);

/* kernel_coefficients(kernel_samples, params) — lagrange.py:100-134 (Eq. 43).
 * ks_dev, L_dev: complex [P].  (The AmplificationWarning is raised by the
 * shim from the scalars a, P.) */
int nfft45_kernel_coefficients(const double* ks_dev, int64_t P, double damping_a,
                               double* L_dev, void* stream);

/* The differentiated coefficient vector of lagrange.py:150-152:
 * dcoef_k = (k+1) L_{k+1} for k < P-1, dcoef_{P-1} = P (L_P = 1). */
int nfft45_derivative_coefficients(const double* L_dev, int64_t P, double* dcoef_dev, void* stream);

/* min_q |x_q| over a complex device vector (the guard of lagrange.py:158);
 * synchronizes and writes the result to *out_host. */
int nfft45_min_abs(const double* x_dev, int64_t n, double* out_host, void* stream);

/* derivative_samples(coefficients, grid, kernel) — lagrange.py:137-164.
 * Synchronizes to apply the SINGULAR_DERIVATIVE guard (min |L'| >= 1e-300). */
int nfft45_derivative_samples(const nfft45_grid* g, const double* L_dev, int m,
                              double* dL_dev, void* stream);

/* ------------------------------------------------------------- plans */

/* build_plan(grid, params) — inverse.py:58-98 (+ build_kernel_data,
 * lagrange.py:167-181).  The plan keeps a reference to `g` (which must
 * outlive it).  Synchronizes; errors KERNEL_OVERFLOW, SINGULAR_DERIVATIVE,
 * NON_POSITIVE_DAMPING. */
int nfft45_plan_create(const nfft45_grid* g, double damping_a, int eta, int m,
                       void* stream, nfft45_plan** out);
/* Extension: build_plan with R = round(eta P) log-series terms for a
 * fractional oversampling factor eta (see nfft45_v_samples_terms). */
int nfft45_plan_create_terms(const nfft45_grid* g, double damping_a, int64_t R, int m,
                             void* stream, nfft45_plan** out);
void nfft45_plan_destroy(nfft45_plan* p);

/* Plan tables (InversePlan fields, inverse.py:44-55; KernelData,
 * lagrange.py:36-39), copied to a device buffer of P complex values. */
typedef enum {
  NFFT45_TABLE_V = 0,            /* kernel_data.v_samples           */
  NFFT45_TABLE_KS = 1,           /* kernel_data.kernel_samples      */
  NFFT45_TABLE_L = 2,            /* kernel_data.coefficients        */
  NFFT45_TABLE_DL = 3,           /* kernel_data.derivative_samples  */
  NFFT45_TABLE_NODE_WEIGHTS = 4, /* node_weights (caller order)     */
  NFFT45_TABLE_DECAY = 5,        /* h1_coefficients (real, im = 0)  */
  NFFT45_TABLE_COEF_SCALE = 6    /* coef_scale (real, im = 0)       */
} nfft45_table;
int nfft45_plan_table(const nfft45_plan* p, int which, double* dst_dev, void* stream);

/* type5(plan, samples) — inverse.py:101-120 (Fig. 2).  s_dev, S_dev:
 * [batch][P]. */
int nfft45_type5(const nfft45_plan* p, const double* s_dev, int64_t batch, double* S_dev,
                 void* stream);

/* type4(plan, spectrum) — inverse.py:123-143 (Fig. 3).  A_dev, a_dev:
 * [batch][P]. */
int nfft45_type4(const nfft45_plan* p, const double* A_dev, int64_t batch, double* a_dev,
                 void* stream);

/* refine_type5 / refine_type4 (plan, data, passes) — inverse.py:146-202
 * (Section V).  passes = 0 is bitwise the plain solve.  For passes >= 2 the
 * call synchronizes once at the end and returns NON_CONVERGENCE if, for any
 * signal of the batch, a residual norm grew between passes (inverse.py:155).
 * In-place calls (S_dev overlapping s_dev) are allowed: the refinement re-reads
 * its operand after writing x, so an overlapping operand is first copied to
 * stream-ordered scratch (cost: one D2D copy; the CUDA-graph cache is skipped). */
int nfft45_refine_type5(const nfft45_plan* p, const double* s_dev, int64_t batch,
                        int passes, double* S_dev, void* stream);
int nfft45_refine_type4(const nfft45_plan* p, const double* A_dev, int64_t batch,
                        int passes, double* a_dev, void* stream);

/* type5 / type4 / refine_type5 / refine_type4 on HOST-resident operands —
 * the reference's own calling convention (numpy arrays in host memory,
 * inverse.py:101-202).  kind = 5 or 4; passes = -1 for the plain solve, else
 * the refine passes.  in_host, out_host: [batch][P] complex128 (pinned memory
 * for asynchronous copies; pageable memory works but copies synchronously).
 * The batch is streamed through the device in chunks of `chunk` signals on a
 * per-(device, stream) pipeline of H2D / solve / D2H streams that persists
 * across calls, so copies in both directions overlap the solves and the next
 * call's uploads.  `stream` waits for the results; blocking != 0 also waits
 * on the host.  With blocking == 0 the result is valid once `stream` (or the
 * device) is synchronized; an output fed back as a later call's input is
 * ordered after its download. */
int nfft45_solve_host(const nfft45_plan* p, int kind, int passes, const double* in_host,
                      int64_t batch, double* out_host, int64_t chunk, int blocking,
                      void* stream);

/* nfft45_solve_host with flags.  Pageable operands (ordinary numpy / malloc
 * memory, detected with cudaPointerGetAttributes) are staged through pinned
 * library buffers by a pool of host copy threads, overlapped with the device
 * work of the neighbouring chunks; such calls always block.
 *   NFFT45_HOST_CHECK_FINITE: scan every staged input chunk on the device and
 *     return NFFT45_ERR_INVALID_ARGUMENT ("operand contains NaN or Inf
 *     entries") if any entry is not finite (grid.py:30-31 as_complex_vector);
 *     the output is then unspecified.  Pageable path only.
 *   NFFT45_HOST_NO_STAGING: copy pageable operands directly (A/B runs). */
#define NFFT45_HOST_CHECK_FINITE 1
#define NFFT45_HOST_NO_STAGING 2
int nfft45_solve_host_ex(const nfft45_plan* p, int kind, int passes, const double* in_host,
                         int64_t batch, double* out_host, int64_t chunk, int blocking, int flags,
                         void* stream);

#ifdef __cplusplus
}
#endif

#endif /* NFFT45_H */
