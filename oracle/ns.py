"""Finite-step Newton–Schulz shifted-sign reflector, FP64 (oracle; test infrastructure).

The north_star loop, step by step, in the order and notation of BASELINE.json
north_star and the paper's eq:NS with the divide convention (reading C1):

    X_0     = (H - s I) / alpha
    for j = 0, 1, 2, ...
        Y_j = X_j X_j                                  (product 1)
        r_j = ||Y_j - I||_F                            (north_star residual)
        stop if rho_j < tol (rho = r or r/sqrt(d), C3/C4), or j == max_steps (C2, C5)
        X_{j+1} = 1.5 X_j - 0.5 X_j Y_j                (product 2; = 1/2 X(3I - X^2), eq:NS)
        X_{j+1} <- (X_{j+1} + X_{j+1}^T)/2             (re-symmetrise each step)
    R = X_steps, certificate = round((d - tr R)/2)     (prop:exact P:147-165; C7)

The matrix product is numpy's float64 matmul: a library primitive used as one
step, with no blocking or reordering of the algorithm around it.

Result flags (values are part of the C-ABI contract and
are restated here, not imported):
    CONVERGED=1  rho < tol
    MAX_STEPS=2  j reached max_steps without convergence
    INDEX_MISMATCH=4  certificate != k
    SCALING_SUSPECT=8  r_{j+1} > r_j (1 + 1e-12) + 1e-10 sqrt(d): with spec(X_0) in
                 [-1,1] every |1 - x^2| shrinks monotonically (prop:NSerr proof,
                 P:456-458), so a rise signals alpha < ||H - sI||_2 (cor:NS P:404-419)
    NONFINITE=16  r_j is NaN/Inf (stop at once, return X_j; certificate := -1, so
                 INDEX_MISMATCH is also set and SHIFT_ON_SPECTRUM is not evaluated)
    SHIFT_ON_SPECTRUM=32  |(d - tr R)/2 - cert| > 0.25 (C7)
"""
import math
import time

import numpy as np

CONVERGED = 1
MAX_STEPS = 2
INDEX_MISMATCH = 4
SCALING_SUSPECT = 8
NONFINITE = 16
SHIFT_ON_SPECTRUM = 32

TOL_ABS = 0
TOL_PER_SQRT_D = 1


def round_half_away(x):
    """Round half away from zero (reading C7)."""
    return int(math.floor(abs(x) + 0.5)) * (1 if x >= 0 else -1)


def initial_iterate(H, s, alpha):
    """X_0 = (H - s I)/alpha, elementwise divide (eq:NS P:379 with C1's divide convention)."""
    X = np.array(H, dtype=np.float64, copy=True)
    d = X.shape[0]
    idx = np.arange(d)
    X[idx, idx] = X[idx, idx] - s
    return X / alpha


def ns_reflector(H, s, alpha, k, max_steps, tol, tol_mode=TOL_ABS, trace_residuals=False):
    """Run the north_star loop on dense symmetric H (d x d, float64).

    Returns a dict with R, steps, residual, trace, cert, flags and optionally the
    per-step residual/trace history (j = 0..steps).
    """
    H = np.asarray(H, dtype=np.float64)
    d = H.shape[0]
    if H.shape != (d, d):
        raise ValueError("H must be square")
    if not (alpha > 0 and math.isfinite(alpha) and math.isfinite(s)):
        raise ValueError("alpha must be finite and > 0, s finite")
    X = initial_iterate(H, s, alpha)
    I = np.eye(d)
    flags = 0
    r_prev = None
    hist_r, hist_t = [], []
    j = 0
    while True:
        Y = X @ X                                       # product 1: Y_j = X_j^2
        r = math.sqrt(float(np.sum((Y - I) ** 2)))      # ||Y_j - I||_F
        hist_r.append(r)
        hist_t.append(float(np.trace(X)))
        if not math.isfinite(r):
            flags |= NONFINITE
            break
        if r_prev is not None and r > r_prev * (1.0 + 1e-12) + 1e-10 * math.sqrt(d):
            flags |= SCALING_SUSPECT
        rho = r / math.sqrt(d) if tol_mode == TOL_PER_SQRT_D else r
        if rho < tol:
            flags |= CONVERGED
            break
        if j == max_steps:
            flags |= MAX_STEPS
            break
        Z = X @ Y                                       # product 2: X_j (X_j^2)
        X = 1.5 * X - 0.5 * Z                           # X_{j+1}
        X = 0.5 * (X + X.T)                             # S:172 re-symmetrisation
        r_prev = r
        j += 1
    trace = float(np.trace(X))
    half = (d - trace) / 2.0
    if (flags & NONFINITE) or not math.isfinite(half):
        cert = -1                      # no certificate for a non-finite iterate (DESIGN.md flags)
    else:
        cert = round_half_away(half)
        if abs(half - cert) > 0.25:
            flags |= SHIFT_ON_SPECTRUM
    if cert != k:
        flags |= INDEX_MISMATCH
    out = dict(R=X, steps=j, residual=r, trace=trace, cert=cert, flags=flags)
    if trace_residuals:
        out["hist_residual"] = hist_r
        out["hist_trace"] = hist_t
    return out


def ns_fixed_depth(A, alpha, m):
    """X_m for X_0 = A/alpha and m NS updates, re-symmetrised each step (S:137-145 in
    the divide convention).  Used by the gapped-bound and mpmath pins."""
    X = np.asarray(A, dtype=np.float64) / alpha
    for _ in range(m):
        X = 1.5 * X - 0.5 * (X @ (X @ X))
        X = 0.5 * (X + X.T)
    return X


def timed_ns_steps(H, s, alpha, n_steps, return_iterate=False):
    """CPU-baseline helper (bench.py cpu_baseline / --impl reference): time exactly n_steps NS updates
    (2 products each) of the same loop as ns_reflector, without its stop test.  Returns (seconds,
    threads), plus X_{n_steps} when return_iterate (pinned in tests/test_oracle_ns.py: bitwise equal to
    ns_reflector's iterate after n_steps fixed steps).  The products are numpy/OpenBLAS FP64 matmuls,
    so the time is a "library CPU" number on the host's cores, not a hand-written-loop one."""
    import os
    X = initial_iterate(H, s, alpha)
    t0 = time.perf_counter()
    for _ in range(n_steps):
        Y = X @ X
        Z = X @ Y
        X = 1.5 * X - 0.5 * Z
        X = 0.5 * (X + X.T)
    t1 = time.perf_counter()
    threads = int(os.environ.get("OPENBLAS_NUM_THREADS", os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1)))
    if return_iterate:
        return t1 - t0, threads, X
    return t1 - t0, threads
