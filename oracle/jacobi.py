"""Cyclic-Jacobi eigendecomposition and the exact reflector I - 2P_k (oracle; test infrastructure).

jacobi_eigh: plain C (oracle/jacobi.c), cyclic Jacobi with round-robin ordering,
             stop at off(A)_F <= 1e-13 ||A||_F, cap 60 sweeps.
exact_reflector: R_k = I - 2 P_k,  P_k = Q_k Q_k^T  (eq:Pk P:143-145; eq:Rk_intro P:43-45),
             which equals sgn(H - sI) for any s in (lambda_k, lambda_{k+1}) (prop:exact P:147-165).
"""
import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "jacobi.c")
_LIB = os.path.join(_HERE, "libjacobi.so")
_lib = None


_CMD = ["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fPIC", "-shared", "-o", _LIB, _SRC, "-lm"]


def build(force=False):
    """Compile oracle/jacobi.c -> oracle/libjacobi.so (gcc, OpenMP, no FMA contraction).
    Rebuilt whenever the sha256 of the source and command differs from the stamp next to the library."""
    import hashlib
    with open(_SRC, "rb") as f:
        digest = hashlib.sha256(f.read() + " ".join(_CMD).encode()).hexdigest()
    stamp = _LIB + ".sha256"
    if not force and os.path.exists(_LIB) and os.path.exists(stamp) and open(stamp).read().strip() == digest:
        return _LIB
    subprocess.check_call(_CMD)
    with open(stamp, "w") as f:
        f.write(digest + "\n")
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        lib.jacobi_eigh.restype = ctypes.c_int
        lib.jacobi_eigh.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                    ctypes.c_double, ctypes.c_int]
        _lib = lib
    return _lib


def jacobi_eigh(H, rel_tol=1e-13, max_sweeps=60):
    """Eigenvalues ascending and eigenvectors (columns of V) of symmetric H by cyclic Jacobi.

    Returns (w, V, sweeps).  Raises if not converged within max_sweeps (S:40 diagnostic).
    """
    A = np.array(H, dtype=np.float64, order="C", copy=True)
    d = A.shape[0]
    V = np.empty((d, d), dtype=np.float64)
    w = np.empty(d, dtype=np.float64)
    sweeps = _load().jacobi_eigh(d, A.ctypes.data, V.ctypes.data, w.ctypes.data, rel_tol, max_sweeps)
    if sweeps < 0:
        raise RuntimeError(f"cyclic Jacobi did not converge in {max_sweeps} sweeps")
    return w, V, sweeps


def exact_reflector_from_eig(V, k):
    """R_k = I - 2 V_k V_k^T with V_k the first k eigenvector columns (eq:Pk P:143-145)."""
    d = V.shape[0]
    Vk = V[:, :k]
    return np.eye(d) - 2.0 * (Vk @ Vk.T)


def exact_reflector(H, k):
    """I - 2P_k of H via cyclic Jacobi (SPEC exact_reflector S:294-302)."""
    w, V, _ = jacobi_eigh(H)
    return exact_reflector_from_eig(V, k), w


def midpoint_shift(w, k):
    """s = (lambda_k + lambda_{k+1})/2 (prop:mid eq:midpoint P:549-553); w ascending, k 1-based."""
    return 0.5 * (w[k - 1] + w[k])
