"""cfg0 (d=64) reflector with a fixed step count m through the public API (for ncu launch timing).
usage: python tools/small_m.py m [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_24840_b200 as nsr  # noqa: E402
import workloads  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 0
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
p = workloads.cfg0_controlled(0)
H = torch.from_numpy(p.H).cuda()
R = torch.empty_like(H)
ws = nsr.alloc_workspace(nsr.ns_workspace_bytes(p.d), H.device)
for _ in range(reps):
    nsr.ns_reflector(H, p.s, p.alpha, p.k, m, 0.0, R=R, ws=ws)
torch.cuda.synchronize()
print("ok")
