"""Re-anchor CG stop tolerance sweep: final R error vs the oracle and CG iterations (NS_CG_DEBUG output)
on the random mixed-path problems.  usage: NS_CG_TOL=x NS_CG_DEBUG=1 python tools/cg_tol_sweep.py"""
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_24840_b200 as nsr  # noqa: E402
import workloads  # noqa: E402
from oracle import checks, ns as ons  # noqa: E402

worst = {1: 0.0, 2: 0.0}
for seed in range(6):
    rng = np.random.default_rng(2000 + seed)
    d = int(rng.choice([130, 200, 256, 300, 512]))
    k = int(rng.integers(1, d))
    g = 10.0 ** rng.uniform(-2, math.log10(0.3))
    lam = np.concatenate([-rng.uniform(g / 2, 1.0, k), rng.uniform(g / 2, 1.0, d - k)])
    Q = workloads.haar_q(rng, d)
    H = (Q * lam[None, :]) @ Q.T
    H = 0.5 * (H + H.T)
    s = float(rng.uniform(-0.3, 0.3) * g)
    alpha = float(np.linalg.norm(H - s * np.eye(d), 2)) * 1.02
    o = ons.ns_reflector(H, s, alpha, k, 100, 1e-10, 1)
    Hg = torch.from_numpy(H).cuda()
    for prec in (1, 2):
        R, r = nsr.ns_reflector(Hg, s, alpha, k, 100, 1e-10, 1, prec=prec)
        e = checks.frob_per_sqrt_d(R.cpu().numpy(), o["R"])
        worst[prec] = max(worst[prec], e)
        print(f"seed={seed} d={d} gap={g:.3g} prec={prec} steps={r['steps']}/{o['steps']} err={e:.2e}", flush=True)
print("worst", worst, "NS_CG_TOL", os.environ.get("NS_CG_TOL"))
