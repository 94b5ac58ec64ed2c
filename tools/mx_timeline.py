"""Per-CTA timeline of the 2-SM split-precision product kernel (ns_debug_mx_trace): how long the
mainloop (start -> accumulators in registers) and the epilogue (-> end) take, and the idle gaps
between consecutive CTAs on an SM.  usage: python tools/mx_timeline.py [d] [mode]"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_24840_b200 as nsr  # noqa: E402

d = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
mode = int(sys.argv[2]) if len(sys.argv) > 2 else 0
A = torch.randn(d, d, dtype=torch.float64, device="cuda")
A = (A + A.T) * (0.5 / d ** 0.5)
ws = nsr.alloc_workspace(nsr.ns_workspace_bytes(d, nsr.NS_PREC_MIXED_BF16X3), A.device)
C = torch.empty_like(A)
nsr.ns_symm_product(A, A, mode=mode, C=C, ws=ws, prec=nsr.NS_PREC_MIXED_BF16X3)
n = (d + 127) // 128
buf = torch.zeros(12 * (2 * n * n + 16), dtype=torch.int64, device="cuda")
lib = nsr.load_library()
lib.ns_debug_mx_trace.argtypes = [ctypes.c_void_p]
lib.ns_debug_mx_trace(ctypes.c_void_p(buf.data_ptr()))
nsr.ns_symm_product(A, A, mode=mode, C=C, ws=ws, prec=nsr.NS_PREC_MIXED_BF16X3)
torch.cuda.synchronize()
lib.ns_debug_mx_trace(None)
t = buf.cpu().numpy().reshape(-1, 12)
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
start, acc, end, sm = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3, (t[:, 2] - t0) / 1e3, t[:, 3]
main, epi = acc - start, end - acc
print(f"CTAs {len(t)}  kernel span {end.max():.0f} us")
print(f"mainloop (start -> accumulators in registers): median {np.median(main):.1f} us, p10 {np.percentile(main, 10):.1f}, p90 {np.percentile(main, 90):.1f}")
print(f"epilogue (-> end): median {np.median(epi):.1f} us, p90 {np.percentile(epi, 90):.1f}")
gaps = []
for s in np.unique(sm):
    o = np.argsort(start[sm == s])
    st, en = start[sm == s][o], end[sm == s][o]
    gaps += list(st[1:] - en[:-1])
gaps = np.array(gaps)
print(f"gap between consecutive CTAs on an SM: median {np.median(gaps):.1f} us, p90 {np.percentile(gaps, 90):.1f}")
busy = np.sum(main) / (len(np.unique(sm)) * end.max())
print(f"mainloop share of SM time: {busy:.3f}")
lead = t[:, 5] > 0
print(f"leader MMA warp: waits on full {np.median(t[lead, 4] / t[lead, 5]):.3f} of its loop, on tempty "
      f"{np.median(t[lead, 7] / t[lead, 5]):.3f}")
print(f"producer waits on empty (cycles / mainloop cycles): {np.median(t[:, 6] / np.maximum(1, t[lead, 5].mean())):.3f}")
nch = max(1, (d // 64 + 7) // 8)
print(f"epilogue warp 2: waits on tfull {np.median(t[:, 8]) / nch:.0f} cycles per chunk, folds {np.median(t[:, 9]) / nch:.0f} "
      f"cycles per chunk (chunks per tile {nch})")
