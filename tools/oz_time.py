"""Time one symmetric product through ns_symm_product (CUDA events), e.g. for NS_OZ_DBG experiments.
usage: python tools/oz_time.py d [ozaki|mixed|fp64] [mode]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2605_24840_b200 as nsr  # noqa: E402

d = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
name = sys.argv[2] if len(sys.argv) > 2 else "ozaki"
prec = {"ozaki": nsr.NS_PREC_FP64_OZAKI, "mixed": nsr.NS_PREC_MIXED_BF16X3, "fp64": nsr.NS_PREC_FP64}[name]
mode = int(sys.argv[3]) if len(sys.argv) > 3 else 0
A = torch.randn(d, d, dtype=torch.float64, device="cuda")
A = (A + A.T) * (0.5 / d ** 0.5)
ws = nsr.alloc_workspace(nsr.ns_workspace_bytes(d, prec), A.device)
C = torch.empty_like(A)
for _ in range(2):
    nsr.ns_symm_product(A, A, mode=mode, C=C, ws=ws, prec=prec)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 5
e0.record()
for _ in range(n):
    nsr.ns_symm_product(A, A, mode=mode, C=C, ws=ws, prec=prec)
e1.record()
torch.cuda.synchronize()
print(f"d={d} {name} mode={mode}: {e0.elapsed_time(e1) / n:.2f} ms per ns_symm_product")
