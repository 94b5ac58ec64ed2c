/*
 * nsreflector.h — C ABI of the B200-native (sm_100a) Newton–Schulz prescribed-index
 * reflector library, libnsreflector.so.
 *
 * WHAT IT COMPUTES (arxiv/paper_2605_24840; P:n = /root/reference/PAPER.md line n):
 *   For a dense symmetric H (d x d), a shift s in the target spectral gap
 *   (lambda_k, lambda_{k+1}) and a scale alpha >= ||H - sI||_2, the prescribed-index
 *   reflector  R_k = I - 2 P_k = sgn(H - sI)   (prop:exact; eq:Pk P:143-145)
 *   by the scaled Newton–Schulz iteration (eq:NS), written in the
 *   BASELINE north_star's divide convention:
 *       X_0 = (H - s I) / alpha,     X_{j+1} = 1.5 X_j - 0.5 X_j (X_j^2).
 *   Loop convention (reading C2): at step j the library forms
 *   Y_j = X_j^2, r_j = ||Y_j - I||_F; it stops with CONVERGED when rho_j < tol
 *   (rho = r_j, or r_j/sqrt(d) in NS_TOL_PER_SQRT_D mode; strict '<', C3/C4), or with
 *   MAX_STEPS when j == max_steps; otherwise it applies the update.  The returned
 *   R = X_steps, residual = r_steps, trace = tr R, index_cert = round((d - tr R)/2)
 *   (half away from zero, C7).  tol = 0 gives fixed-step mode (C5).
 *
 * MEMORY, LAYOUT, OWNERSHIP
 *   - Matrices are FP64, row-major with leading dimension ld >= d (elements).  H is
 *     symmetric; ONLY ITS UPPER TRIANGLE (i <= j) IS READ.  R is written in full and
 *     is bitwise symmetric.  R must not alias H.
 *   - Device pointers: caller-owned CUDA device memory (e.g. torch tensors).  The
 *     workspace is caller-owned device memory of at least ns_workspace_bytes(...)
 *     bytes, 256-byte aligned; the library never allocates device memory on the
 *     hot path.  Work is enqueued on the caller's stream; the call returns after
 *     the result record is on the host (one stream synchronisation at the end, plus
 *     bounded look-ahead waits on tiny status records while iterating).
 *   - `out` / `outs` are HOST memory owned by the caller.
 *
 * ERRORS
 *   Argument violations are detected on the host before any launch and return
 *   NS_ERR_INVALID_ARG (message via ns_last_error()).  CUDA failures return
 *   NS_ERR_CUDA.  Numerical outcomes are FLAGS in ns_result_t, never errors
 *   ("rejection is a value"):  NS_F_CONVERGED, NS_F_MAX_STEPS,
 *   NS_F_INDEX_MISMATCH (cert != k; R is still sgn(H - sI) for the index the shift
 *   selects), NS_F_SCALING_SUSPECT (residual rose: alpha < ||H - sI||_2, cor:NS
 *   P:404-419), NS_F_NONFINITE (NaN/Inf residual; iteration stops at once),
 *   NS_F_SHIFT_ON_SPECTRUM (|(d - tr R)/2 - cert| > 0.25).
 *
 * THREADING: reentrant; at most one call in flight per (stream, workspace).
 */
#ifndef NSREFLECTOR_H
#define NSREFLECTOR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  NS_PREC_FP64 = 0,          /* FP64 DMMA contraction (accuracy path) */
  NS_PREC_MIXED_BF16X3 = 1,  /* tcgen05 BF16x3 steps -> switch -> re-anchor -> FP64 steps (C16) */
  NS_PREC_MIXED_TF32X3 = 2,  /* as MIXED_BF16X3 with TF32 hi/lo splits (tcgen05 kind::tf32; more margin, half rate) */
  NS_PREC_FP64_OZAKI = 3     /* FP64-accurate products emulated on tcgen05 INT8 (Ozaki split, 7 balanced
                                base-256 digits, 28 digit pairs -- 34 when the tolerance is below 1e-13 d
                                in absolute terms, which lowers the residual floor from ~1.5e-15 d to
                                ~4e-17 d); single or batched, d <= 65536 (K segments of 16384
                                keep the INT32 group sums exact) */
} ns_precision_t;

typedef enum {
  NS_TOL_ABS = 0,            /* stop when ||X^2 - I||_F < tol */
  NS_TOL_PER_SQRT_D = 1      /* stop when ||X^2 - I||_F / sqrt(d) < tol */
} ns_tolmode_t;

typedef enum {
  NS_OK = 0,
  NS_ERR_INVALID_ARG = 1,
  NS_ERR_CUDA = 2,
  NS_ERR_NCCL = 3,
  NS_ERR_WORKSPACE = 4,
  NS_ERR_UNSUPPORTED = 5
} ns_status_t;

enum {
  NS_F_CONVERGED = 1,
  NS_F_MAX_STEPS = 2,
  NS_F_INDEX_MISMATCH = 4,
  NS_F_SCALING_SUSPECT = 8,
  NS_F_NONFINITE = 16,
  NS_F_SHIFT_ON_SPECTRUM = 32
};

/* Result record (host).  steps = NS updates applied to the returned R (C2);
 * residual = ||R^2 - I||_F of the returned R (the check that stopped the loop);
 * trace = tr R; index_cert = round((d - trace)/2); flags = NS_F_* bits. */
typedef struct {
  int32_t steps;
  int32_t flags;
  double residual;
  double trace;
  int64_t index_cert;
  int32_t kernel_launches;   /* device kernels this call launched (incl. early-exit look-ahead steps) */
  int32_t switch_step;       /* mixed path: j at which the low-precision phase ended (-1 = none) */
  double pre_polish_residual;/* mixed path: low-precision ||X_switch^2 - I||_F (0 if no switch) */
  double alpha;              /* the scale used (the caller's, or the device Gershgorin bound for alpha = 0) */
} ns_result_t;

/*
 * Tuning / diagnostic options (ns_reflector_ex).  ns_options_default() fills the
 * library defaults, which ns_reflector uses.
 *   switch_tol     mixed path: the BF16x3 phase ends at the first j with
 *                  ||X_j^2 - I||_F / sqrt(d) < switch_tol (default 1e-3, readings C16/C16b:
 *                  10x above the ~1e-4 noise floor of the split-precision residual).  Quadratic
 *                  convergence can still jump from above switch_tol to below that floor in one step;
 *                  when the residual at the switch reads below 5e-4 (run-to-tolerance mode) the step
 *                  that produced X_switch is taken again in FP64-class arithmetic from X_{j-1}
 *                  before the re-anchor, so the FP64 phase tracks the oracle's residuals to a few
 *                  percent and takes its step count.
 *   cg_iters       mixed path: maximum conjugate-gradient iterations of the re-anchor solve
 *                  |A|E + E|A| = sym(X~ [A, X~]); the solve stops earlier once its residual
 *                  has dropped by 1e-6 (default cap 512; 0 = polish without re-anchor).
 *   stop_at_switch mixed path: return the pre-polish iterate X_switch as R (no re-anchor,
 *                  no FP64 steps); flags then carry neither CONVERGED nor MAX_STEPS.
 *   lookahead      steps enqueued before the host reads the stop flag (0 = default: 2 for large
 *                  problems, 8 for small or batched ones); clamped to 15 (the status ring has 16
 *                  slots).  Honoured by the FP64, Ozaki and mixed single-problem paths.
 *   polish         mixed path: arithmetic of the re-anchor's two dense products and of the
 *                  polishing steps: 0 = both FP64 DMMA, 1 = both FP64 emulated on the INT8 tensor
 *                  cores (the Ozaki products of NS_PREC_FP64_OZAKI), 2 (default) = the
 *                  re-anchor products emulated on INT8, the polishing steps FP64 DMMA.
 *   filter_a/b     the step X_{j+1} = a X_j + b X_j^3 (generic odd sign-preserving
 *                  filters; with tol = 0 and max_steps = m it is the fixed-depth filter phi_m).
 *   filter_c[3]    coefficients of X^5, X^7, X^9: with any of them nonzero the step is the general odd
 *                  polynomial X_{j+1} = a X + b X^3 + c0 X^5 + c1 X^7 + c2 X^9 (eq:signpreserving P:278-289;
 *                  "low-degree odd polynomial filters" P:513-518), evaluated as X P(X^2) with Horner's
 *                  rule in Y = X^2: deg + 1 symmetric products per step (deg = highest nonzero power of Y).
 *                  FP64 and NS_PREC_FP64_OZAKI, single problem; the workspace must hold
 *                  ns_workspace_bytes_ex(d, prec, opts) bytes (one more d_pad^2 matrix).
 */
typedef struct {
  double switch_tol;
  int32_t cg_iters;
  int32_t stop_at_switch;
  int32_t lookahead;
  int32_t polish;
  int32_t reserved[2];
  double filter_a;   /* odd cubic filter step X <- filter_a X + filter_b X^3 (eq:signpreserving P:278-289); */
  double filter_b;   /* Newton–Schulz = (1.5, -0.5) (default).  FP64 paths only; mixed requires the default. */
  double filter_c[3];/* X^5, X^7, X^9 coefficients (default 0: the cubic step) */
} ns_options_t;

void ns_options_default(ns_options_t* opts);
/* Workspace for ns_reflector_ex with these options (>= ns_workspace_bytes; general filters need one more matrix). */
size_t ns_workspace_bytes_ex(int64_t d, ns_precision_t prec, const ns_options_t* opts);

/* Bytes of device workspace ns_reflector needs for dimension d (batch = 1). */
size_t ns_workspace_bytes(int64_t d, ns_precision_t prec);

/* Bytes of device workspace ns_reflector_batched needs for `batch` matrices of dimension d. */
size_t ns_workspace_bytes_batched(int64_t d, int64_t batch, ns_precision_t prec);

/*
 * ns_reflector — one reflector, run to tolerance (north_star call).
 *   H      device, d x d, row-major, leading dim ldh >= d; upper triangle read.
 *   s      shift (finite).      alpha   scale (finite, > 0); X_0 = (H - sI)/alpha.  alpha = 0:
 *          the library computes alpha = ||H - sI||_inf (>= ||H - sI||_2, the Gershgorin surrogate of
 *          the default realization) on the device first (one pass over H's upper triangle
 *          and an 8-byte readback; NS_ERR_INVALID_ARG if H - sI has a non-finite entry); out->alpha
 *          reports the scale used.
 *   k      target index, 0 <= k <= d (the paper's domain is 1..d-1); used
 *          only for NS_F_INDEX_MISMATCH.
 *   max_steps >= 0; tol >= 0 (0 = fixed max_steps updates); tm tolerance mode.
 *   prec   NS_PREC_FP64, or NS_PREC_MIXED_BF16X3: BF16x3 tcgen05 steps until the switch
 *          threshold, one FP64 re-anchor solve, FP64 steps to tol (single problem only;
 *          NS_PREC_MIXED_TF32X3 the same with TF32 splits; NS_PREC_FP64_OZAKI: FP64 products emulated
 *          on the INT8 tensor cores, d <= 65536).
 *   R      device, d x d, leading dim ldr >= d; written in full, bitwise symmetric.
 *   ws     device workspace, ws_bytes >= ns_workspace_bytes(d, prec).
 *   stream cudaStream_t (as void*); NULL = legacy default stream.
 *   out    host result record.
 */
ns_status_t ns_reflector(const double* H, int64_t d, int64_t ldh, double s, double alpha, int32_t k,
                         int32_t max_steps, double tol, ns_tolmode_t tm, ns_precision_t prec,
                         double* R, int64_t ldr, void* ws, size_t ws_bytes, void* stream,
                         ns_result_t* out);

/* ns_reflector with explicit options (NULL = defaults). */
ns_status_t ns_reflector_ex(const double* H, int64_t d, int64_t ldh, double s, double alpha, int32_t k,
                            int32_t max_steps, double tol, ns_tolmode_t tm, ns_precision_t prec,
                            double* R, int64_t ldr, void* ws, size_t ws_bytes, void* stream,
                            const ns_options_t* opts, ns_result_t* out);

/*
 * ns_reflector_host — same computation with HOST H and R (end-to-end entry point):
 * copies H (host, ldh) to the device workspace, runs ns_reflector, copies R back to
 * host memory (ldr).  Pinned host buffers give full PCIe bandwidth; pageable works.
 * FP64 path with pinned R, even d and even ldr: the device may write R during the call
 * (the iterate its stop rule predicts final is streamed to R behind the confirming
 * square product; if the prediction fails R is simply overwritten by the returned
 * iterate) -- R must not be read or reused by the caller before the call returns.
 * Set NS_SPEC_COPY=0 to disable.  The workspace must hold ns_workspace_bytes_host(d, prec) bytes.
 */
size_t ns_workspace_bytes_host(int64_t d, ns_precision_t prec);
ns_status_t ns_reflector_host(const double* H_host, int64_t d, int64_t ldh, double s, double alpha,
                              int32_t k, int32_t max_steps, double tol, ns_tolmode_t tm,
                              ns_precision_t prec, double* R_host, int64_t ldr, void* ws,
                              size_t ws_bytes, void* stream, ns_result_t* out);

/*
 * ns_reflector_batched — `batch` independent problems (configs[1]: many small H, one
 * shift each; pass the same H several times via the stride to sweep shifts).
 *   H      device, H + b*stride_h is problem b's d x d matrix (row-major, ld = d).
 *   s, alpha, k   HOST arrays [batch] (ns_reflector_batched_dev: DEVICE arrays, read back and
 *          validated on the host before any launch).  alpha[b] = 0: device Gershgorin bound.
 *   R      device, R + b*stride_r receives problem b's reflector (ld = d).
 *   outs   HOST array [batch] of result records.
 *   Each problem stops independently (its own steps/flags); problems that stopped
 *   cost no further contraction work.
 */
ns_status_t ns_reflector_batched(const double* H, int64_t d, int64_t batch, int64_t stride_h,
                                 const double* s, const double* alpha, const int32_t* k,
                                 int32_t max_steps, double tol, ns_tolmode_t tm, ns_precision_t prec,
                                 double* R, int64_t stride_r, void* ws, size_t ws_bytes, void* stream,
                                 ns_result_t* outs);
ns_status_t ns_reflector_batched_dev(const double* H, int64_t d, int64_t batch, int64_t stride_h,
                                     const double* s_dev, const double* alpha_dev, const int32_t* k_dev,
                                     int32_t max_steps, double tol, ns_tolmode_t tm, ns_precision_t prec,
                                     double* R, int64_t stride_r, void* ws, size_t ws_bytes, void* stream,
                                     ns_result_t* outs);

/*
 * ---------------- inertia probes and shift bisection (alg:ssr steps 3-4) ----------------
 * ns_inertia: count = #{i : lambda_i(H) < s} from the trace certificate of a Newton–Schulz run on
 *   X_0 = (H - sI)/alpha with alpha = ||H - sI||_inf (device): the run stops once ||X^2 - I||_F <
 *   1/(2 sqrt d), where (d - tr X)/2 is provably within 1/4 of the count (lem:NSsign sign preservation;
 *   sum(1 - |x_i|) <= sqrt(d) ||X^2 - I||_F), so round((d - tr X)/2) is exact.  resolved = 0 when that
 *   residual was not reached in max_steps (s on, or within ~1e-17 relative of, an eigenvalue).  prec:
 *   NS_PREC_FP64 or NS_PREC_FP64_OZAKI.  Workspace: ns_workspace_bytes_inertia(d, prec).  out: the
 *   probe's NS result (steps, residual, alpha used).
 * ns_shift_bisect: brackets lambda_k and lambda_{k+1} by inertia probes (bisecting the wider bracket)
 *   until the midpoint of the endpoint estimates is admissible by prop:reuse_refresh (half the
 *   estimated gap exceeds the estimate error eps) and eps <= rel_eps x estimated gap; 1 <= k <= d-1.
 *   Initial bracket [lo, hi] (must satisfy count(lo) <= k-1 and count(hi) >= k+1; lo >= hi: the device
 *   computes [-||H||_inf, ||H||_inf]).  out->ok = 0 if max_probes ran out (e.g. a closed gap).  The
 *   probe sequence is deterministic (oracle/setup.py shift_bisect is the reference algorithm).
 */
typedef struct {
  double s;                      /* certified midpoint shift (lam_k_hat + lam_k1_hat)/2 */
  double lam_k_lo, lam_k_hi;     /* lambda_k in [lam_k_lo, lam_k_hi] */
  double lam_k1_lo, lam_k1_hi;   /* lambda_{k+1} in [lam_k1_lo, lam_k1_hi] */
  double eps;                    /* max bracket half-width: |lam_hat - lam| <= eps for both endpoints */
  double alpha;                  /* ||H - sI||_inf at the returned s (0 unless ok) */
  int32_t probes;                /* inertia probes run (including nudged retries) */
  int32_t unresolved;            /* probes that had to be nudged off an eigenvalue */
  int32_t ok;                    /* 1: midpoint certified admissible with eps <= rel_eps * gap estimate */
  int32_t pad;
} ns_bisect_t;
size_t ns_workspace_bytes_inertia(int64_t d, ns_precision_t prec);
ns_status_t ns_inertia(const double* H, int64_t d, int64_t ldh, double s, ns_precision_t prec, int32_t max_steps,
                       void* ws, size_t ws_bytes, void* stream, int64_t* count, int32_t* resolved, ns_result_t* out);
ns_status_t ns_shift_bisect(const double* H, int64_t d, int64_t ldh, int32_t k, double lo, double hi, double rel_eps,
                            int32_t max_probes, ns_precision_t prec, void* ws, size_t ws_bytes, void* stream,
                            ns_bisect_t* out);

/*
 * ---------------- shift / scale setup (the step before the path) ----------------
 * ns_scale_bound: alpha_out = ||H - sI||_inf = max_i (|H_ii - s| + sum_{j!=i} |H_ij|), the
 *   Gershgorin / infinity-norm surrogate for ||H - sI||_2 (alg:ssr step 5 P:676-678; default
 *   realization P:710-712; scaling discussion P:720-736).  Always >= ||H - sI||_2, so
 *   (H - sI)/alpha_out has its spectrum in [-1, 1] (lem:NSsign).  Device H (upper triangle read),
 *   device workspace >= ns_workspace_bytes_setup(d) bytes; alpha_out is host memory.  Also bounds the
 *   endpoint drift of prop:reuse_refresh: |lambda_i(H') - lambda_i(H)| <= ||H' - H||_inf (Weyl).
 *   A NaN/Inf entry of H - sI propagates into alpha_out (never dropped by the max) and the call
 *   returns NS_ERR_INVALID_ARG after writing it.
 * ns_shift_certificate (host only): prop:reuse_refresh.  Given endpoint estimates
 *   lam_k_hat, lam_k1_hat with error <= eps, a shift s and a next-step drift bound delta:
 *     margin_hat  = min(s - lam_k_hat, lam_k1_hat - s)
 *     admissible  = margin_hat > eps           (true margin >= margin_lb = margin_hat - eps)
 *     reuse_ok    = delta < margin_hat - eps   (true margin at the next iterate >= reuse_margin_lb)
 *     midpoint    = (lam_k_hat + lam_k1_hat)/2, midpoint_ok = (lam_k1_hat - lam_k_hat)/2 > eps
 */
size_t ns_workspace_bytes_setup(int64_t d);
ns_status_t ns_scale_bound(const double* H, int64_t d, int64_t ldh, double s, void* ws, size_t ws_bytes,
                           void* stream, double* alpha_out);
typedef struct {
  double margin_hat;
  double margin_lb;
  double reuse_margin_lb;
  double midpoint;
  int32_t admissible;
  int32_t reuse_ok;
  int32_t midpoint_ok;
  int32_t pad;
} ns_shift_cert_t;
ns_status_t ns_shift_certificate(double lam_k_hat, double lam_k1_hat, double eps, double s, double delta,
                                 ns_shift_cert_t* out);

/*
 * ---------------- Algorithm 1 outer loop (the step after the path) ----------------
 * ns_alg1_rotated_quartic: nruns independent runs of alg:ssr on the dense rotated
 * quartic of §5.3:
 *   E(x) = 1/4 sum y_i^4 + 1/2 sum c_i y_i^2, y = Q^T x, c_i = -1 (i <= k_r), +1 otherwise,
 * from start x0[r] with target index k[r]: exact endpoints, midpoint shift, alpha = ||H - sI||_2,
 * R~ = m Newton–Schulz steps (m = 0: exact reflector), x <- x - eta R~ g, until ||g|| <= grad_tol or
 * max_iters.  One CTA per run, everything in shared memory (d <= 64).
 *   Q      device d x d row-major orthogonal matrix (shared by all runs)
 *   k      HOST int32[nruns], 1 <= k < d
 *   x0     device nruns x d starts;  x_out device nruns x d final states
 *   out    HOST ns_alg1_result_t[nruns]: iterations, final ||g||, Morse index of H(x_final),
 *          success = (||g|| <= grad_tol && Morse index == k), stop reason, midpoint refreshes, last shift
 *   ws     device workspace >= ns_workspace_bytes_alg1(nruns) bytes
 * ns_alg1_rotated_quartic_ex: the same with a shift policy (alg:ssr step 4; DESIGN reading N2b)
 * and the admissibility stop (step 8; prop:reuse_refresh P:604).  pol == NULL is the midpoint
 * policy with eps = 0.  Per iteration, after the ||g|| / budget test:
 *   NS_SHIFT_MIDPOINT  s = (lk + lk1)/2
 *   NS_SHIFT_DAMPED    s = min(max(damp s_prev + (1 - damp) mid, lk + clip gap), lk1 - clip gap)   (n >= 1)
 *   NS_SHIFT_REUSE     s = s_prev if min(s_prev - lk, lk1 - s_prev) > reuse_margin, else mid      (n >= 1)
 *   stop (NS_ALG1_STOP_INADMISSIBLE, no update) unless min(s - lk, lk1 - s) > eps.
 * Errors: NS_ERR_INVALID_ARG for damp outside [0, 1), clip outside (0, 1/2], a negative or non-finite
 * reuse_margin / eps, an unknown policy, and the checks of the plain entry.
 */
enum { NS_SHIFT_MIDPOINT = 0, NS_SHIFT_DAMPED = 1, NS_SHIFT_REUSE = 2 };
enum { NS_ALG1_STOP_GRAD = 0, NS_ALG1_STOP_BUDGET = 1, NS_ALG1_STOP_INADMISSIBLE = 2 };
typedef struct {
  int32_t policy;        /* NS_SHIFT_* */
  int32_t pad;
  double damp;           /* damped: weight beta of the previous shift, [0, 1) */
  double clip;           /* damped: kappa, clip into [lk + kappa gap, lk1 - kappa gap], (0, 1/2] */
  double reuse_margin;   /* reuse/refresh: threshold tau on the previous shift's margin, >= 0 */
  double eps;            /* admissibility: endpoint error bound, >= 0 */
} ns_alg1_policy_t;
typedef struct {
  int32_t iters;
  int32_t morse_index;
  int32_t success;
  int32_t stop_reason;   /* NS_ALG1_STOP_* */
  double grad_norm;
  int32_t refreshes;     /* iterations whose shift was the fresh midpoint */
  int32_t pad;
  double s_last;         /* last shift used in an update (NaN if none) */
} ns_alg1_result_t;
size_t ns_workspace_bytes_alg1(int32_t nruns);
ns_status_t ns_alg1_rotated_quartic(const double* Q, int64_t d, int32_t nruns, const int32_t* k, const double* x0,
                                    int32_t m, double eta, int32_t max_iters, double grad_tol, double* x_out,
                                    void* ws, size_t ws_bytes, void* stream, ns_alg1_result_t* out);
ns_status_t ns_alg1_rotated_quartic_ex(const double* Q, int64_t d, int32_t nruns, const int32_t* k,
                                       const double* x0, int32_t m, double eta, int32_t max_iters, double grad_tol,
                                       const ns_alg1_policy_t* pol, double* x_out, void* ws, size_t ws_bytes,
                                       void* stream, ns_alg1_result_t* out);

/*
 * ---------------- multi-GPU (one process per GPU, NCCL over NVLink/NVSwitch) ----------------
 * configs[4] (d = 49152) and configs[3] strong scaling on P GPUs (the paper motivates
 * accelerator execution of the dense sign iteration).  Every rank keeps the full FP64
 * iterate (X_j, X_{j+1} and Y = X_j^2, 3 x 8 d_pad^2 bytes: the symmetric work split below needs any
 * rank to read any row panel) and computes only its share of the upper 128x128 tiles of each symmetric
 * product: tile t of the library's upper-tile order belongs to rank t % P (balanced to one tile).
 * Exchange (default): every rank's workspace is mapped into every process (CUDA IPC; the mapping check
 * is collective on every call), and the product kernels' epilogues store each finished tile (upper
 * half only; the receivers mirror it locally after the barrier -- NS_SHARD_MIRROR=sender stores the
 * mirror remotely too) and its residual / trace partial straight into all ranks' buffers over NVLink,
 * so the transfer overlaps the contraction tile by tile; one one-double all-reduce per product is the
 * barrier.  Every rank sums the same partials in the same fixed order: identical stop decisions.
 * Fallback (a rank cannot map, e.g. VMM memory, or NS_SHARD_P2P=0): chunked NCCL all-gathers of the
 * tiles overlapped with the contraction, per-rank residual sums gathered and summed in rank order.
 *
 * ns_comm_get_unique_id  rank 0 creates the 128-byte NCCL id (ship it to the other ranks, e.g.
 *                        with torch.distributed.broadcast).
 * ns_comm_init           every rank, with its CUDA device current; collective (blocks until all
 *                        ranks joined).  nranks >= 1 (1 = single-GPU communicator).
 * ns_comm_init_host      a communicator WITHOUT NCCL: the library's collectives (IPC record exchange,
 *                        barriers, the fallback's all-gathers) call `allgather(send, recv, bytes, user)`,
 *                        which must all-gather `bytes` host bytes from every rank into recv (nranks *
 *                        bytes, rank order) and return 0 (e.g. torch.distributed over gloo).  The device
 *                        path (IPC mappings, peer-store epilogues) is unchanged; each barrier becomes a
 *                        stream synchronisation plus the callback, so no kernel ever waits on another
 *                        rank's kernel.  Used by the tests to run several ranks as processes sharing
 *                        one GPU, which NCCL does not allow.
 * ns_shard_plan          host-only: the (I, J) tile pairs rank `rank` computes for dimension d
 *                        (tiles_ij[2*i], tiles_ij[2*i+1]); returns the count via n_out; writes at
 *                        most `cap` pairs.  Lets callers/tests check balance and coverage.
 * ns_shard_rows          host-only: the block-row panel [row0, row1) rank `rank` owns in the rows entry
 *                        (d / nranks rows each; NS_ERR_INVALID_ARG unless nranks divides d).
 * ns_reflector_sharded   same arguments and result as ns_reflector (FP64 only); H (full, upper
 *                        triangle read) and R (full) are device buffers on every rank; all ranks
 *                        must call it with identical scalars.  The workspace must hold
 *                        ns_workspace_bytes_sharded(d, nranks) bytes.
 * ns_reflector_sharded_rows  SURVEY §8(b)'s sharded entry: rank r passes only its block-row panel of H,
 *                        H_rows = rows [row0, row1) of H (ns_shard_rows; (d/P) x d, leading dimension
 *                        ldh >= d, device memory; in each row i only the elements j >= i are read) and
 *                        receives only the same rows of R in R_rows ((d/P) x d, ldr >= d, every element
 *                        written).  X_0 is assembled on every rank from all ranks' panels (peer stores,
 *                        or an all-gather of the panels on the fallback path).  prec must be NS_PREC_FP64
 *                        (else NS_ERR_UNSUPPORTED); d must be divisible by nranks (else
 *                        NS_ERR_INVALID_ARG); all ranks call it with identical scalars; the result
 *                        (steps, flags, residual, trace, certificate) is identical on every rank.
 *                        Workspace: ns_workspace_bytes_sharded(d, nranks).
 */
typedef int (*ns_host_allgather_fn)(const void* send, void* recv, size_t bytes, void* user);
typedef struct ns_comm ns_comm_t;
ns_status_t ns_comm_get_unique_id(uint8_t id[128]);
ns_status_t ns_comm_init(int rank, int nranks, const uint8_t id[128], ns_comm_t** comm);
ns_status_t ns_comm_init_host(int rank, int nranks, ns_host_allgather_fn allgather, void* user, ns_comm_t** comm);
ns_status_t ns_comm_destroy(ns_comm_t* comm);
ns_status_t ns_shard_rows(int64_t d, int nranks, int rank, int64_t* row0, int64_t* row1);
ns_status_t ns_shard_plan(int64_t d, int nranks, int rank, int32_t* tiles_ij, int32_t cap, int32_t* n_out);

/*
 * ns_symm_product_shard — the sharded path's peer-memory exchange primitive at kernel level (tests):
 * rank `rank` of `nranks` computes its share of the upper 128x128 tiles of C = A B (mode 0) or of
 * C = 1.5 A - 0.5 A B (mode 1) and its epilogue stores every tile and its mirror into ALL n_dst
 * destination matrices C_list[0..n_dst-1] (device pointers, d x d, ld = d; in ns_reflector_sharded
 * these are the ranks' buffers mapped through CUDA IPC over NVLink).  Calling it for every rank of a
 * plan fills every destination with the full, bitwise-symmetric product.  d must be a multiple of 128;
 * A, B symmetric, ld = d.  C_list is a HOST array.  Workspace: ns_workspace_bytes(d, NS_PREC_FP64).
 */
ns_status_t ns_symm_product_shard(const double* A, const double* B, double* const* C_list, int32_t n_dst, int64_t d,
                                  int32_t mode, int32_t rank, int32_t nranks, void* ws, size_t ws_bytes,
                                  void* stream);
/* Exchange chunking of the sharded path: each rank's tile list is cut into n_chunks chunks of
 * chunk_slots slots (padded to the largest rank); chunk c of rank q carries the rank's local tiles
 * c*chunk_slots .. c*chunk_slots + chunk_slots - 1, i.e. global upper tiles (c*chunk_slots + s)*P + q. */
ns_status_t ns_shard_chunks(int64_t d, int nranks, int32_t* n_chunks, int32_t* chunk_slots);
/*
 * ns_reflector_sharded_emulated — the sharded algorithm with `nranks` ranks emulated on ONE GPU
 * (tests; multi-GPU behaviour without multiple GPUs): nranks workspace replicas, each rank's product
 * kernels launched in turn with the multi-GPU path's peer-store epilogue (destinations: every
 * replica), each replica deciding on its own data.  No kernel waits on another.  Returns
 * NS_ERR_CUDA ("emulated ranks diverged") if the replicas' final states differ in any bit.  Same
 * arguments and result as ns_reflector (FP64); device H and R; workspace >=
 * ns_workspace_bytes_sharded_emulated(d, nranks).  flags: bit 0 = block-row input (replica r forms
 * X_0 from rows [r d/P, (r+1) d/P) of H with the rows entry's peer-store init and writes the same
 * rows of R), bit 1 = sender-mirror epilogue (default 0: receivers mirror).
 */
size_t ns_workspace_bytes_sharded_emulated(int64_t d, int nranks);
ns_status_t ns_reflector_sharded_emulated(int32_t nranks, const double* H, int64_t d, int64_t ldh, double s,
                                          double alpha, int32_t k, int32_t max_steps, double tol, ns_tolmode_t tm,
                                          double* R, int64_t ldr, void* ws, size_t ws_bytes, void* stream,
                                          int32_t flags, ns_result_t* out);
size_t ns_workspace_bytes_sharded(int64_t d, int nranks);
ns_status_t ns_reflector_sharded(ns_comm_t* comm, const double* H, int64_t d, int64_t ldh, double s, double alpha,
                                 int32_t k, int32_t max_steps, double tol, ns_tolmode_t tm, double* R, int64_t ldr,
                                 void* ws, size_t ws_bytes, void* stream, ns_result_t* out);
ns_status_t ns_reflector_sharded_rows(ns_comm_t* comm, const double* H_rows, int64_t d, int64_t ldh, double s,
                                      double alpha, int32_t k, int32_t max_steps, double tol, ns_tolmode_t tm,
                                      ns_precision_t prec, double* R_rows, int64_t ldr, void* ws, size_t ws_bytes,
                                      void* stream, ns_result_t* out);

/*
 * ns_symm_product — kernel-level entry used by tests (the contraction core alone).
 * A and B are symmetric (only their upper triangles are read); A, B, C device, d x d,
 * leading dim ld (same for all).
 * mode 0: C = A B for commuting A, B (C symmetric): upper-triangle tiles only, mirrored,
 *         C bitwise symmetric.
 * mode 1: C = 1.5 A - 0.5 (A B) (the NS update epilogue), same tiling.
 * mode 2: C = A B, every tile (no symmetry assumed for the result).
 * prec NS_PREC_FP64: FP64 DMMA kernel; NS_PREC_MIXED_BF16X3: tcgen05 BF16x3 kernel (FP32
 * accumulation; A and B are split into BF16 hi/lo planes first).
 * The workspace must hold ns_workspace_bytes(d, prec) bytes.
 */
ns_status_t ns_symm_product(const double* A, const double* B, double* C, int64_t d, int64_t ld,
                            int32_t mode, ns_precision_t prec, void* ws, size_t ws_bytes, void* stream);

/*
 * Optional per-thread kernel timing (used by bench.py for the roofline): when enabled,
 * every contraction launch is bracketed by CUDA events on the caller's stream and,
 * at the end of each call, the durations of the launches that did work are added to
 * the thread's accumulators.  Events cost ~microseconds; off by default.
 */
typedef struct {
  int64_t n_square;     /* Y_j = X_j^2 launches that did work (steps + 1 per reflector) */
  int64_t n_update;     /* X_{j+1} = 1.5 X_j - 0.5 X_j Y_j launches that did work */
  double ms_square;     /* summed device time of those launches */
  double ms_update;
  int64_t n_calls;
  /* split-precision (BF16x3) and Ozaki (INT8 digit-pair) product launches of the mixed and Ozaki paths,
   * with the arithmetic they EXECUTE (for a roofline in their own precision): launches that exited at
   * once (queued past a stop, or a converged CG) are excluded (device time < 1/4 of the longest launch
   * of the same shape in the call). */
  int64_t n_lowp;       /* BF16x3 product launches that did work */
  double ms_lowp;       /* their summed device time */
  double lowp_flops;    /* executed BF16 flops: 3 GEMMs x 2 x 128 x 128 x d_pad per 128x128 output tile computed */
  int64_t n_oz;         /* Ozaki INT8 product launches that did work (K segments count separately) */
  double ms_oz;
  double oz_ops;        /* executed INT8 ops: digit pairs (28 or 34) x 2 x 128 x 128 x K per 128x128 output tile */
} ns_profile_t;
void ns_profile_enable(int on);
void ns_profile_reset(void);
void ns_profile_get(ns_profile_t* out);

/* Library identification: build string with the compile target (e.g. "sm_100a"). */
const char* ns_build_info(void);

/*
 * Diagnostics (tools/mx_timeline.py): when `device_buffer` is non-NULL, the 2-SM split-precision
 * kernel launched by ns_symm_product (prec NS_PREC_MIXED_*) writes 12 uint64 per CTA into it
 * (%globaltimer at start, when the accumulators are in registers, at the end; SM id; leader MMA warp
 * cycles waiting for operands, its loop cycles, producer cycles waiting for free stages, MMA cycles
 * waiting for TMEM; epilogue cycles waiting for / folding accumulator chunks).  The buffer must hold
 * 12 x CTAs entries; NULL turns the stamps off (default).
 */
void ns_debug_mx_trace(void* device_buffer);
/* Diagnostics (builds with -DNS_SMALL_TRACE=1; else returns 0): the fused small-d kernel's clock64 stamps
 * of its last launch (block 0): [0] start, [1] X_0 formed, [2 + p] after product p, [100] loop end,
 * [128 + w] warp w's DMMA loop end in product 0.  Copies n <= 256 values to host memory and clears them. */
int ns_debug_small_trace(unsigned long long* out, int n);
/* Diagnostics (builds with -DNS_P64_TRACE=1; else returns -1): every CTA of the 64x64-tile FP64 product kernel
 * appends a record of 10 uint64 (SM id | mode << 16 | diagonal << 17; %globaltimer at start, first stage landed,
 * end; job << 32 | tile; K loop done in warps 0..3; 0) to `device_buffer` (1 + 10 x capacity uint64, element 0 = record counter,
 * zeroed by the caller) -- tools/p64_trace.py.  NULL turns the records off. */
int ns_debug_p64_trace(void* device_buffer, unsigned long long capacity);
const char* ns_status_string(ns_status_t st);
/* Thread-local message for the last non-NS_OK status on this thread ("" if none). */
const char* ns_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* NSREFLECTOR_H */
