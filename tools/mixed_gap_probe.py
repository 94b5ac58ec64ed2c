"""Mixed path at small relative gaps: CG iterations, error vs the oracle.  usage: NS_CG_DEBUG=1 python ..."""
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_24840_b200 as nsr  # noqa: E402
import workloads  # noqa: E402
from oracle import checks, ns as ons  # noqa: E402

for seed, g in [(0, 1e-2), (1, 5e-3), (2, 3e-3), (3, 1e-3)]:
    rng = np.random.default_rng(3000 + seed)
    d = 256
    k = int(rng.integers(1, d))
    lam = np.concatenate([-rng.uniform(g / 2, 1.0, k), rng.uniform(g / 2, 1.0, d - k)])
    Q = workloads.haar_q(rng, d)
    H = (Q * lam[None, :]) @ Q.T
    H = 0.5 * (H + H.T)
    s = 0.0
    alpha = float(np.linalg.norm(H, 2)) * 1.02
    o = ons.ns_reflector(H, s, alpha, k, 100, 1e-10, 1)
    Hg = torch.from_numpy(H).cuda()
    for prec in (1, 2, 3):
        R, r = nsr.ns_reflector(Hg, s, alpha, k, 100, 1e-10, 1, prec=prec)
        print(f"gap={g:g} prec={prec} steps={r['steps']}/{o['steps']} sw={r['switch_step']} cert={r['cert']}/{k} "
              f"err={checks.frob_per_sqrt_d(R.cpu().numpy(), o['R']):.2e}", flush=True)
