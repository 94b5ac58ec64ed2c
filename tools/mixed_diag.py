"""Mixed-path diagnostics on the random-sweep problems: gap, steps, switch, pre-polish residual, error."""
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_24840_b200 as nsr  # noqa: E402
import workloads  # noqa: E402
from oracle import checks, ns as ons  # noqa: E402

seeds = [int(x) for x in sys.argv[1:]] or list(range(6))
for seed in seeds:
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
    Rf, rf = nsr.ns_reflector(Hg, s, alpha, k, 100, 1e-10, 1)
    line = [f"seed={seed} d={d} k={k} gap={g:.3g} min|lam-s|/alpha={np.min(np.abs(lam - s)) / alpha:.3g} "
            f"oracle_steps={o['steps']} fp64_err={checks.frob_per_sqrt_d(Rf.cpu().numpy(), o['R']):.2e}"]
    for prec in (1, 2, 3):
        for cg in (24, 48):
            opts = nsr.ns_options(cg_iters=cg) if prec != 3 else None
            R, r = nsr.ns_reflector(Hg, s, alpha, k, 100, 1e-10, 1, prec=prec, options=opts)
            line.append(f"  prec={prec} cg={cg} steps={r['steps']} sw={r['switch_step']} pre={r['pre_polish_residual']:.2e} "
                        f"err={checks.frob_per_sqrt_d(R.cpu().numpy(), o['R']):.2e}")
            if prec == 3:
                break
    print("\n".join(line), flush=True)
