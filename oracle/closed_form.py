"""Closed forms when the generator knows Q (oracle; test infrastructure).

For X_0 = (H - sI)/alpha = Q diag(mu) Q^T with mu_i = (lambda_i - s)/alpha:
    exact reflector      R   = Q diag(sgn(mu)) Q^T                  prop:exact P:155-163
    exact m-step iterate X_m = Q diag(p_m(mu)) Q^T                  thm:generic proof P:308-312,
                                                                     prop:spectralerr P:345-349
Q is either explicit (Haar, cfg0/cfg1) or a product of Householder reflectors
Q = H_1 H_2 ... H_n,  H_i = I - 2 v_i v_i^T / (v_i^T v_i)   (reading C13),
applied to a block of columns at O(n d c) cost, so columns of R can be formed at
any d (cfg3 d=16384, cfg4 d=49152) without materialising Q.
"""
import numpy as np

from .scalar import p_m


def spectral_matrix(Q, values):
    """Q diag(values) Q^T for explicit orthogonal Q."""
    Q = np.asarray(Q, dtype=np.float64)
    return (Q * np.asarray(values, dtype=np.float64)[None, :]) @ Q.T


def reflector_explicit_q(Q, lam, s):
    """R = Q diag(sgn(lambda - s)) Q^T (prop:exact)."""
    return spectral_matrix(Q, np.sign(np.asarray(lam) - s))


def iterate_explicit_q(Q, lam, s, alpha, m):
    """X_m = Q diag(p_m((lambda - s)/alpha)) Q^T (thm:generic proof P:308-312)."""
    mu = (np.asarray(lam, dtype=np.float64) - s) / alpha
    return spectral_matrix(Q, p_m(mu, m))


def householder_apply(Vh, B, transpose=False):
    """Q B (or Q^T B) for Q = H_1 ... H_n with reflector vectors Vh[i] (n x d).

    Q B = H_1 (H_2 (... (H_n B))) ; Q^T B = H_n (... (H_1 B)) since each H_i = H_i^T.
    """
    B = np.array(B, dtype=np.float64, copy=True)
    n = Vh.shape[0]
    order = range(n) if transpose else range(n - 1, -1, -1)
    for i in order:
        v = Vh[i]
        beta = 2.0 / float(v @ v)
        B -= np.outer(beta * v, v @ B)
    return B


def householder_spectral_columns(Vh, values, cols):
    """Columns `cols` of Q diag(values) Q^T, Q = H_1...H_n (reading C13)."""
    d = Vh.shape[1]
    cols = np.asarray(cols, dtype=np.int64)
    E = np.zeros((d, cols.size))
    E[cols, np.arange(cols.size)] = 1.0
    B = householder_apply(Vh, E, transpose=True)
    B *= np.asarray(values, dtype=np.float64)[:, None]
    return householder_apply(Vh, B, transpose=False)


def householder_reflector_columns(Vh, lam, s, cols):
    """Columns of R = Q diag(sgn(lambda - s)) Q^T."""
    return householder_spectral_columns(Vh, np.sign(np.asarray(lam) - s), cols)


def householder_iterate_columns(Vh, lam, s, alpha, m, cols):
    """Columns of X_m = Q diag(p_m(mu)) Q^T."""
    mu = (np.asarray(lam, dtype=np.float64) - s) / alpha
    return householder_spectral_columns(Vh, p_m(mu, m), cols)
