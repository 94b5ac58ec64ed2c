"""configs[1] (6144 batched d = 256 problems): call time and the per-launch square / update split (library events)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_24840_b200 as nsr  # noqa: E402
import workloads  # noqa: E402

probs = workloads.cfg1_batched(seed=0, n_matrices=2048)
H = torch.stack([torch.from_numpy(p.H) for p in probs]).cuda()
s_, a_, k_ = [p.s for p in probs], [p.alpha for p in probs], [p.k for p in probs]
ws = nsr.alloc_workspace(nsr.ns_workspace_bytes_batched(256, len(probs), 0), H.device)
R = torch.empty_like(H)
for _ in range(2):
    nsr.ns_reflector_batched(H, s_, a_, k_, 100, 1e-12, R=R, ws=ws)
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    R, outs = nsr.ns_reflector_batched(H, s_, a_, k_, 100, 1e-12, R=R, ws=ws)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
nsr.ns_profile_enable(True)
nsr.ns_profile_reset()
nsr.ns_reflector_batched(H, s_, a_, k_, 100, 1e-12, R=R, ws=ws)
torch.cuda.synchronize()
pr = nsr.ns_profile_get()
print({"tag": os.environ.get("TAG", ""), "ms_median": sorted(ts)[2], "steps": sum(o["steps"] for o in outs), **pr})
