"""Time one FP64 reflector (cfg3 recipe, fixed 10 steps) at several d; run under NS_TILE64_MAX=... to
compare the 64x64-tile and 128x128-tile product kernels."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_24840_b200 as nsr  # noqa: E402
import workloads  # noqa: E402

for d in (1024, 2048, 3000, 4096, 6144, 8192):
    p = workloads.cfg3_dense(d=d, k=d // 16, form=False)
    H = workloads.householder_form_fast(p.Vh, p.lam, device="cuda")
    R = torch.empty_like(H)
    ws = nsr.alloc_workspace(nsr.ns_workspace_bytes(d), H.device)
    f = lambda: nsr.ns_reflector(H, p.s, p.alpha, p.k, 10, 0.0, R=R, ws=ws)  # noqa: E731
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        f()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"d={d}: {ms:.2f} ms, {21 * d ** 3 / (ms * 1e-3) / 1e12:.2f} TFLOP/s", flush=True)
