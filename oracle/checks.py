"""Reflector invariants (oracle; test infrastructure).

For the exact reflector R = sgn(H - sI) = I - 2P_k (prop:exact P:147-165):
    R^2 = I,  R^T = R,  R H = H R,  tr R = d - 2k
"""
import numpy as np


def reflector_invariants(R, H, k):
    """Return the four invariant defects (max-abs, except the trace which is absolute)."""
    R = np.asarray(R, dtype=np.float64)
    H = np.asarray(H, dtype=np.float64)
    d = R.shape[0]
    return dict(
        square=float(np.max(np.abs(R @ R - np.eye(d)))),
        symmetry=float(np.max(np.abs(R - R.T))),
        commutator=float(np.max(np.abs(R @ H - H @ R))),
        trace=float(abs(np.trace(R) - (d - 2 * k))),
    )


def frob_per_sqrt_d(A, B):
    """||A - B||_F / sqrt(d)  (the north_star parity metric)."""
    A = np.asarray(A, dtype=np.float64)
    return float(np.linalg.norm(A - np.asarray(B, dtype=np.float64)) / np.sqrt(A.shape[0]))
