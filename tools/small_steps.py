"""Per-step cost of the fused small-d kernel: device time of ns_reflector(cfg0) vs the step count."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_24840_b200 as nsr  # noqa: E402
import workloads  # noqa: E402

p = workloads.cfg0_controlled(0)
for d in (64, 96, 32):
    Hn = p.H if d == 64 else __import__("numpy").pad(p.H, ((0, d - 64), (0, d - 64)))[:d, :d] if d > 64 else p.H[:d, :d]
    H = torch.from_numpy(Hn).cuda()
    R = torch.empty_like(H)
    ws = nsr.alloc_workspace(nsr.ns_workspace_bytes(d), H.device)
    s = torch.cuda.current_stream()
    for m in (0, 1, 2, 4, 8, 16):
        for _ in range(3):
            nsr.ns_reflector(H, p.s, p.alpha, p.k, m, 0.0, R=R, ws=ws)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 50
        torch.cuda.synchronize()
        e0.record(s)
        for _ in range(n):
            nsr.ns_reflector(H, p.s, p.alpha, p.k, m, 0.0, R=R, ws=ws)
        e1.record(s)
        torch.cuda.synchronize()
        print(f"d={d} max_steps={m}: {1e3 * e0.elapsed_time(e1) / n:.1f} us per call (incl. host)")
