"""Shift/scale setup and filter variants (oracle; test infrastructure).

inf_norm_shifted   ||H - sI||_inf = max_i sum_j |H_ij - s delta_ij|: the cheap scaling surrogate of
                   the default realization and disc "scaling choice".
shift_certificate  prop:reuse_refresh, transcribed statement by statement.
inertia            #{i : lambda_i < s}, the plain definition from eigenvalues (the quantity the trace
                   certificate round((d - tr sgn(H - sI))/2) of prop:exact counts; alg:ssr step 3 realised
                   as an inertia probe).
shift_bisect       endpoint bisection with an inertia oracle until the estimated midpoint is admissible by
                   prop:reuse_refresh with eps <= rel_eps x estimated gap (the reference algorithm of the
                   C-ABI ns_shift_bisect: same probe order and the same floating-point formulas).
poly_filter_scalar / poly_filter_fixed_depth
                   the generic odd sign-preserving polynomial filter phi(t) = sum_i c_i t^(2i+1)
                   (eq:signpreserving P:278-289; the "low-degree odd polynomial filters" of P:513-518)
                   applied m times: X <- sum_i c_i X^(2i+1), the powers X^(2i+1) = X (X X)^i formed by
                   plain repeated products, re-symmetrised each step.
filter_step / filter_fixed_depth
                   an odd cubic sign-preserving filter phi(t) = a t + b t^3 (eq:signpreserving
                   P:278-289; Newton-Schulz is a = 3/2, b = -1/2, eq:NS) applied m times to
                   X_0 = (H - sI)/alpha: the fixed-depth filtered reflector phi_m(alpha(H - sI))
                   of eq:phi-reflector / alg:ssr step 6 (divide convention C1).
"""
import numpy as np


def inf_norm_shifted(H, s):
    A = np.array(H, dtype=np.float64, copy=True)
    A[np.diag_indices_from(A)] -= s
    return float(np.max(np.sum(np.abs(A), axis=1)))


def shift_certificate(lam_k_hat, lam_k1_hat, eps, s, delta=0.0):
    """prop:reuse_refresh: estimated margin, admissibility, reuse under drift delta, midpoint."""
    m_hat = min(s - lam_k_hat, lam_k1_hat - s)
    admissible = m_hat > eps                       # "If m_hat > eps, then s is admissible"
    margin_lb = m_hat - eps                        # "true margin at least m_hat - eps"
    reuse_ok = admissible and (delta < m_hat - eps)   # "Delta_n <= delta_n < m_hat - eps"
    reuse_margin_lb = m_hat - eps - delta          # "at least m_hat - eps - delta_n"
    midpoint = 0.5 * (lam_k_hat + lam_k1_hat)      # "estimated midpoint"
    midpoint_ok = 0.5 * (lam_k1_hat - lam_k_hat) > eps   # first claim applied to the midpoint
    return dict(margin_hat=m_hat, margin_lb=margin_lb, reuse_margin_lb=reuse_margin_lb, midpoint=midpoint,
                admissible=bool(admissible), reuse_ok=bool(reuse_ok), midpoint_ok=bool(midpoint_ok))


def filter_step_scalar(t, a, b):
    return a * t + b * t * t * t


def filter_scalar(t, m, a, b):
    x = np.asarray(t, dtype=np.float64)
    for _ in range(m):
        x = filter_step_scalar(x, a, b)
    return x


def filter_fixed_depth(H, s, alpha, m, a, b):
    """X_m with X_0 = (H - sI)/alpha and X <- a X + b X (X X), re-symmetrised each step."""
    X = np.array(H, dtype=np.float64, copy=True)
    X[np.diag_indices_from(X)] -= s
    X = X / alpha
    for _ in range(m):
        Y = X @ X
        X = a * X + b * (X @ Y)
        X = 0.5 * (X + X.T)
    return X


def inertia(w, s):
    """#{i : w_i < s} for the eigenvalues w of H (any order)."""
    return int(np.count_nonzero(np.asarray(w, dtype=np.float64) < s))


def shift_bisect(count, k, lo, hi, rel_eps, max_probes):
    """Bracket lambda_k in (a_k, b_k] and lambda_{k+1} in (a_k1, b_k1] with an inertia oracle count(s) =
    #{lambda < s} (count(lo) <= k-1, count(hi) >= k+1), bisecting the wider bracket (ties: lambda_k's), until
    the estimated midpoint passes prop:reuse_refresh's midpoint test -- half the estimated gap exceeds the
    estimate error eps ("eps_{n+1} < g_{n+1}/2") -- with eps <= rel_eps * estimated gap.
    Returns dict(s, lam_k_lo, lam_k_hi, lam_k1_lo, lam_k1_hi, eps, probes, ok)."""
    ak, bk, ak1, bk1 = lo, hi, lo, hi
    probes, ok = 0, False
    while True:
        lk, lk1 = 0.5 * (ak + bk), 0.5 * (ak1 + bk1)
        eps = 0.5 * max(bk - ak, bk1 - ak1)
        gap = lk1 - lk
        if gap > 0.0 and 0.5 * gap > eps and eps <= rel_eps * gap:
            ok = True
            break
        if probes >= max_probes:
            break
        refine_k = (bk - ak) >= (bk1 - ak1)
        a, b = (ak, bk) if refine_k else (ak1, bk1)
        sp = 0.5 * (a + b)
        c = count(sp)
        probes += 1
        if c <= k - 1:
            ak, ak1 = max(ak, sp), max(ak1, sp)
        elif c == k:
            bk, ak1 = min(bk, sp), max(ak1, sp)
        else:
            bk, bk1 = min(bk, sp), min(bk1, sp)
    return dict(s=0.5 * (0.5 * (ak + bk) + 0.5 * (ak1 + bk1)), lam_k_lo=ak, lam_k_hi=bk, lam_k1_lo=ak1,
                lam_k1_hi=bk1, eps=0.5 * max(bk - ak, bk1 - ak1), probes=probes, ok=ok)


def poly_filter_scalar(t, m, coeffs):
    """phi applied m times to scalars, phi(t) = sum_i coeffs[i] t^(2i+1)."""
    x = np.asarray(t, dtype=np.float64)
    for _ in range(m):
        x = sum(c * x ** (2 * i + 1) for i, c in enumerate(coeffs))
    return x


def poly_filter_fixed_depth(H, s, alpha, m, coeffs):
    """X_m with X_0 = (H - sI)/alpha and X <- sum_i coeffs[i] X^(2i+1) (odd powers by repeated products)."""
    X = np.array(H, dtype=np.float64, copy=True)
    X[np.diag_indices_from(X)] -= s
    X = X / alpha
    for _ in range(m):
        Y = X @ X
        P = X.copy()                      # X^(2i+1), i = 0
        acc = coeffs[0] * P
        for c in coeffs[1:]:
            P = P @ Y                     # X^(2i+1) = X^(2i-1) X^2
            acc = acc + c * P
        X = 0.5 * (acc + acc.T)
    return X
