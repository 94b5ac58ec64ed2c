"""Shift/scale setup and filter variants (oracle; test infrastructure).

inf_norm_shifted   ||H - sI||_inf = max_i sum_j |H_ij - s delta_ij|: the cheap scaling surrogate of
                   the default realization and disc "scaling choice".
shift_certificate  prop:reuse_refresh, transcribed statement by statement.
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
