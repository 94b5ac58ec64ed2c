"""Mixed path: final reflector error vs the re-anchor's CG iteration count (cfg3 recipe, d=16384 and 1024)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_24840_b200 as nsr  # noqa: E402
import workloads  # noqa: E402
from oracle import closed_form  # noqa: E402

for d, k in ((16384, 1024), (4096, 256)):
    p = workloads.cfg3_dense(d=d, k=k, form=False)
    H = workloads.householder_form_fast(p.Vh, p.lam, device="cuda")
    cols = np.array([0, 1, d // 2, d - 1])
    Rc = closed_form.householder_reflector_columns(p.Vh, p.lam, 0.0, cols)
    for it in (4, 8, 12, 16, 20, 24, 32):
        o = nsr.ns_options(cg_iters=it, polish=1)
        R, res = nsr.ns_reflector(H, p.s, p.alpha, p.k, p.max_steps, p.tol, p.tol_mode,
                                  prec=nsr.NS_PREC_MIXED_BF16X3, options=o)
        Rg = R[:, torch.as_tensor(cols, device="cuda")].cpu().numpy()
        err = float(np.sqrt(np.mean(np.sum((Rg - Rc) ** 2, axis=0))))
        print(f"d={d} cg_iters={it}: err {err:.3e} steps {res['steps']} cert {res['cert']}", flush=True)
