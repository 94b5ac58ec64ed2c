"""Full-size oracle runs for the GPU parity tests (test infrastructure; calls only oracle/).

The north_star's parity criterion is ||R_gpu - R_oracle||_F / sqrt(d) with R_oracle the oracle's own
Newton–Schulz output (reading C15), so the full-size tests run the oracle at full size on the GPU host's
CPU cores: configs[3] (d = 16384, 25 numpy FP64 products, ~4 min on 16 cores), configs[2] (d = 4096,
seeds 0-3), all 6144 problems of configs[1] (d = 256, in a process pool).

Results are cached under $NS_ORACLE_CACHE (default /tmp/nsr_oracle_cache), keyed by the sha256 of the
input matrix bytes and the run parameters, so a second run on the same box skips the CPU work.  Nothing
depends on the cache: a miss recomputes.
"""
import hashlib
import json
import os

import numpy as np

from oracle import ns as ons

CACHE = os.environ.get("NS_ORACLE_CACHE", "/tmp/nsr_oracle_cache")
_KEYS = ("steps", "residual", "trace", "cert", "flags")


def _key(H, *params):
    """sha256 of the input bytes (row block by row block, to bound memory at d = 16384) and the parameters."""
    h = hashlib.sha256()
    for r0 in range(0, H.shape[0], 1024):
        h.update(np.ascontiguousarray(H[r0:r0 + 1024]).tobytes())
    h.update(json.dumps(list(params)).encode())
    return h.hexdigest()[:32]


def ns_cached(H, s, alpha, k, max_steps, tol, tol_mode):
    """oracle/ns.py ns_reflector(..., trace_residuals=True) with a disk cache."""
    key = _key(H, s, alpha, k, max_steps, tol, tol_mode)
    base = os.path.join(CACHE, key)
    try:
        with open(base + ".json") as f:
            meta = json.load(f)
        R = np.load(base + ".npy", mmap_mode=None)
        meta["R"] = R
        return meta
    except (OSError, ValueError):
        pass
    out = ons.ns_reflector(H, s, alpha, k, max_steps, tol, tol_mode, trace_residuals=True)
    try:
        os.makedirs(CACHE, exist_ok=True)
        np.save(base + ".npy", out["R"])
        meta = {k_: out[k_] for k_ in _KEYS + ("hist_residual", "hist_trace")}
        with open(base + ".json", "w") as f:
            json.dump(meta, f)
    except OSError:
        pass
    return out


def _cfg1_worker(args):
    H, s, alpha, k = args
    o = ons.ns_reflector(H, s, alpha, k, 100, 1e-12, ons.TOL_ABS, trace_residuals=True)
    return o


def cfg1_all(probs, workers=None):
    """The oracle on every configs[1] problem (one process per core, single-threaded BLAS in each)."""
    import multiprocessing as mp
    h = hashlib.sha256()
    for p in probs:
        h.update(np.ascontiguousarray(p.H).tobytes())
        h.update(np.float64([p.s, p.alpha, p.k]).tobytes())
    key = h.hexdigest()[:32]
    path = os.path.join(CACHE, "cfg1_" + key + ".npz")
    try:
        with np.load(path) as z:
            Rs, st, rs, tr, ce, fl, hi = (z[n] for n in ("R", "steps", "residual", "trace", "cert", "flags", "hist"))
        return [dict(R=Rs[i], steps=int(st[i]), residual=float(rs[i]), trace=float(tr[i]), cert=int(ce[i]),
                     flags=int(fl[i]), hist_residual=[float(v) for v in hi[i][: int(st[i]) + 1]])
                for i in range(len(probs))]
    except (OSError, KeyError, ValueError):
        pass
    workers = workers or os.cpu_count() or 1
    env_prev = {v: os.environ.get(v) for v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS")}
    for v in env_prev:
        os.environ[v] = "1"
    try:
        ctx = mp.get_context("spawn")
        with ctx.Pool(workers) as pool:
            outs = pool.map(_cfg1_worker, [(p.H, p.s, p.alpha, p.k) for p in probs], chunksize=16)
    finally:
        for v, val in env_prev.items():
            if val is None:
                os.environ.pop(v, None)
            else:
                os.environ[v] = val
    try:
        os.makedirs(CACHE, exist_ok=True)
        hist = np.full((len(outs), 102), np.nan)
        for i, o in enumerate(outs):
            hist[i, : len(o["hist_residual"])] = o["hist_residual"]
        np.savez(path, R=np.stack([o["R"] for o in outs]), steps=[o["steps"] for o in outs],
                 residual=[o["residual"] for o in outs], trace=[o["trace"] for o in outs],
                 cert=[o["cert"] for o in outs], flags=[o["flags"] for o in outs], hist=hist)
    except OSError:
        pass
    return outs
