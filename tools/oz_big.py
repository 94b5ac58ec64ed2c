"""Ozaki square product at large d (kernel time via CUDA events): L2-locality experiments."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2605_24840_b200 as nsr  # noqa: E402

d = int(sys.argv[1]) if len(sys.argv) > 1 else 49152
A = torch.randn(d, d, dtype=torch.float64, device="cuda")
A = (A + A.T) * (0.5 / d ** 0.5)
ws = nsr.alloc_workspace(nsr.ns_workspace_bytes(d, nsr.NS_PREC_FP64_OZAKI), A.device)
C = torch.empty_like(A)
nsr.ns_symm_product(A, A, mode=0, C=C, ws=ws, prec=nsr.NS_PREC_FP64_OZAKI)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
nsr.ns_symm_product(A, A, mode=0, C=C, ws=ws, prec=nsr.NS_PREC_FP64_OZAKI)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(f"d={d}: {ms:.1f} ms per Ozaki symmetric product call ({d ** 3 / (ms * 1e-3) / 1e12:.1f} TFLOP/s FP64-equiv.)")
