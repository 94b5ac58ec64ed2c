"""Profile helper: cfg0 (d=64) reflector calls through the public API, for ncu / timing splits."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_24840_b200 as nsr  # noqa: E402
import workloads  # noqa: E402

p = workloads.cfg0_controlled(0)
H = torch.from_numpy(p.H).cuda()
R = torch.empty_like(H)
ws = nsr.alloc_workspace(nsr.ns_workspace_bytes(p.d), H.device)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
for _ in range(5):
    nsr.ns_reflector(H, p.s, p.alpha, p.k, 100, 1e-12, R=R, ws=ws)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(reps):
    nsr.ns_reflector(H, p.s, p.alpha, p.k, 100, 1e-12, R=R, ws=ws)
t1 = time.perf_counter()
print(f"wall per call {1e6 * (t1 - t0) / reps:.1f} us")
