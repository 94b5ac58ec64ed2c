"""Profile helper: a few Ozaki / BF16x3 / FP64 symmetric products at d (default 8192).
usage: python tools/oz_prof.py d [ozaki|mixed|fp64] [mode 0|1|2]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2605_24840_b200 as nsr  # noqa: E402

d = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
prec = {"ozaki": nsr.NS_PREC_FP64_OZAKI, "mixed": nsr.NS_PREC_MIXED_BF16X3, "fp64": nsr.NS_PREC_FP64}[
    sys.argv[2] if len(sys.argv) > 2 else "ozaki"]
mode = int(sys.argv[3]) if len(sys.argv) > 3 else 0
A = torch.randn(d, d, dtype=torch.float64, device="cuda")
A = (A + A.T) * (0.5 / d ** 0.5)
ws = nsr.alloc_workspace(nsr.ns_workspace_bytes(d, prec), A.device)
C = torch.empty_like(A)
for _ in range(3):
    nsr.ns_symm_product(A, A, mode=mode, C=C, ws=ws, prec=prec)
torch.cuda.synchronize()
print("ok")
