"""Residual floor of the FP64 and Ozaki paths on a converged iterate (fixed steps, tol 0)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_24840_b200 as nsr  # noqa: E402
import workloads  # noqa: E402

for d in (256, 1024, 2048, 4096):
    rng = np.random.default_rng(d)
    lam = np.concatenate([-rng.uniform(0.05, 1.0, d // 4), rng.uniform(0.05, 1.0, d - d // 4)])
    Q = workloads.haar_q(rng, d)
    H = 0.5 * (((Q * lam[None, :]) @ Q.T) + ((Q * lam[None, :]) @ Q.T).T)
    Hg = torch.from_numpy(H).cuda()
    out = [f"d={d}"]
    for prec in (0, 3):
        for m in (20, 24):
            R, r = nsr.ns_reflector(Hg, 0.0, 1.0, d // 4, m, 0.0, 0, prec=prec)
            out.append(f"prec={prec} m={m} r={r['residual']:.2e} r/d={r['residual'] / d:.2e}")
    print("  ".join(out), flush=True)
