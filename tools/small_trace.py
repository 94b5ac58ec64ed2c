"""Phase timeline of the fused small-d kernel (configs[0]) from a -DNS_SMALL_TRACE=1 build.

    python tools/build_variant.py build_ab/small_trace.so -DNS_SMALL_TRACE=1
    python tools/small_trace.py build_ab/small_trace.so
"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_24840_b200 as nsr  # noqa: E402
import workloads  # noqa: E402

lib = nsr.load_library(os.path.abspath(sys.argv[1]))
lib.ns_debug_small_trace.restype = ctypes.c_int
lib.ns_debug_small_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
p = workloads.cfg0_controlled(0)
H = torch.from_numpy(p.H).cuda()
R = torch.empty_like(H)
ws = nsr.alloc_workspace(nsr.ns_workspace_bytes(p.d), H.device)
buf = (ctypes.c_ulonglong * 256)()
fixed = int(os.environ.get("FIXED", "0"))          # > 0: fixed step count (tol = 0), for timing experiments
steps, tol = (fixed, 0.0) if fixed else (100, 1e-12)
for _ in range(20):
    nsr.ns_reflector(H, p.s, p.alpha, p.k, steps, tol, R=R, ws=ws)
lib.ns_debug_small_trace(buf, 256)
_, res = nsr.ns_reflector(H, p.s, p.alpha, p.k, steps, tol, R=R, ws=ws)
torch.cuda.synchronize()
lib.ns_debug_small_trace(buf, 256)
t = list(buf)
t0 = t[0]
nprod = 2 * res["steps"] + 1
print(f"steps {res['steps']} products {nprod}; clock64 cycles since kernel start")
print(f"init (X_0 formed): {t[1] - t0}")
prev = t[1]
for q in range(nprod):
    print(f"product {q:2d} ({'square' if q % 2 == 0 else 'update'}): ends {t[2 + q] - t0:7d}  duration {t[2 + q] - prev:6d}")
    prev = t[2 + q]
print(f"loop end / copy-out start: {t[100] - t0}")
print("product 0 per-warp DMMA loop end (cycles after X_0):", [t[128 + w] - t[1] for w in range(20) if t[128 + w]])
print("product 1 per-warp DMMA loop end (cycles after product 0):", [t[160 + w] - t[2] for w in range(20) if t[160 + w]])
