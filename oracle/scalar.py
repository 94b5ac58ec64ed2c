"""Scalar Newton–Schulz polynomials and error recurrence (oracle; test infrastructure).

p_0(t)=t, p_{m+1}(t)=1/2 p_m(t)(3-p_m(t)^2)                 eq:pm
eps_{m+1}=1/2 eps_m^2 (3-eps_m),  eps_0 = 1-gamma           eq:ns_scalar_recurrence P:442-445
||p_m(A)-sgn A||_2 = max_i |p_m(mu_i)-sgn mu_i|             prop:spectralerr P:334-352
smallest m with eps_m(gamma) <= tol                          disc:spectral_compression P:478-508

For a symmetric X_0 = Q diag(mu) Q^T the NS iterate is X_m = Q diag(p_m(mu)) Q^T
(thm:generic proof P:308-312), so in exact arithmetic the residual
||X_m^2 - I||_F = sqrt(sum_i (p_m(mu_i)^2 - 1)^2) and the trace tr X_m = sum_i p_m(mu_i)
depend on the eigenvalues alone.  ``predict_run`` replays the north_star loop
(reading C2: check before update) on those scalars to predict the step count.
"""
import math

import numpy as np


def p_step(t):
    """One application of f(t) = 1/2 t (3 - t^2)  (eq:pm P:383)."""
    return 0.5 * t * (3.0 - t * t)


def p_m(t, m):
    """p_m(t) by m applications of f (eq:pm P:380-384). Works on scalars and arrays."""
    x = np.asarray(t, dtype=np.float64) if not isinstance(t, float) else t
    for _ in range(m):
        x = p_step(x)
    return x


def eps_m(gamma, m):
    """eps_m(gamma) = 1 - p_m(gamma) via the recurrence eq:ns_scalar_recurrence.

    eps_0 = 1 - gamma (prop:NSerr statement P:438-440), eps_{m+1} = 1/2 eps_m^2 (3 - eps_m).
    """
    if not (0.0 < gamma <= 1.0):
        raise ValueError("gamma must lie in (0,1] (prop:NSerr P:436)")
    e = 1.0 - gamma
    for _ in range(m):
        e = 0.5 * e * e * (3.0 - e)
    return e


def min_depth(gamma, tol, cap=64):
    """Smallest m with eps_m(gamma) <= tol (disc:spectral_compression P:491-494)."""
    for m in range(cap + 1):
        if eps_m(gamma, m) <= tol:
            return m
    raise ValueError(f"margin too small for polynomial filter: gamma={gamma}")


def spectral_operator_error(mu, m):
    """max_i |p_m(mu_i) - sgn(mu_i)|  (prop:spectralerr eq:spectralerr P:337-340)."""
    mu = np.asarray(mu, dtype=np.float64)
    return float(np.max(np.abs(p_m(mu, m) - np.sign(mu))))


def scaled_margin(lam, s, alpha):
    """gamma = min_i |lambda_i - s| / alpha  (disc:spectral_compression P:484-490, divide form C1)."""
    lam = np.asarray(lam, dtype=np.float64)
    return float(np.min(np.abs(lam - s)) / alpha)


def predict_run(mu, max_steps, tol, per_sqrt_d):
    """Exact-arithmetic replay of the north_star loop on the eigenvalues mu of X_0.

    Returns (steps, residual_sequence, trace_sequence).  residual_sequence[j] is
    ||X_j^2 - I||_F evaluated eigenvalue-wise; the loop checks before updating
    (reading C2) and stops when rho < tol (strict, C4) or j == max_steps.
    """
    mu = np.asarray(mu, dtype=np.float64)
    d = mu.size
    x = mu.copy()
    res, tr = [], []
    j = 0
    while True:
        r = math.sqrt(float(np.sum((x * x - 1.0) ** 2)))
        res.append(r)
        tr.append(float(np.sum(x)))
        rho = r / math.sqrt(d) if per_sqrt_d else r
        if rho < tol or j == max_steps:
            return j, res, tr
        x = p_step(x)
        j += 1
