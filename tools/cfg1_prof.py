"""Profile helper: one configs[1] batched call (6144 problems of d=256) through the public API."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_24840_b200 as nsr  # noqa: E402
import workloads  # noqa: E402

n_mat = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
probs = workloads.cfg1_batched(seed=0, n_matrices=n_mat, count=n_mat)
H = torch.stack([torch.from_numpy(p.H) for p in probs]).cuda()
s_ = [p.s for p in probs]
a_ = [p.alpha for p in probs]
k_ = [p.k for p in probs]
prec = int(sys.argv[2]) if len(sys.argv) > 2 else 0
ws = nsr.alloc_workspace(nsr.ns_workspace_bytes_batched(256, len(probs), prec), H.device)
R = torch.empty_like(H)
R, outs = nsr.ns_reflector_batched(H, s_, a_, k_, 100, 1e-12, R=R, ws=ws, prec=prec)
torch.cuda.synchronize()
print("steps sum", sum(o["steps"] for o in outs))
