"""Re-run chosen stress_sweep seeds on the mixed path with diagnostics (CG passes, residual histories)."""
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import paper_2605_24840_b200 as nsr  # noqa: E402
from oracle import checks, ns as ons  # noqa: E402
from stress_sweep import problem  # noqa: E402
for seed in [int(x) for x in sys.argv[1:]]:
    H, s, alpha, k, ms, tol, tm = problem(seed, int(os.environ.get("STRESS_DMAX", "600")))
    d = H.shape[0]
    alpha = max(alpha, float(np.linalg.norm(H - s * np.eye(d), 2)) * 1.01)
    ev = np.linalg.eigvalsh((H - s * np.eye(d)) / alpha)
    o = ons.ns_reflector(H, s, alpha, k, 100, 1e-10, 1, trace_residuals=True)
    print(f"seed={seed} d={d} min|x0|={np.min(np.abs(ev)):.3e} oracle steps={o['steps']} "
          f"hist/sqrt(d)={[f'{v / math.sqrt(d):.1e}' for v in o['hist_residual']]}", flush=True)
    for prec in (1, 2):
        R, r = nsr.ns_reflector(torch.from_numpy(H).cuda(), s, alpha, k, 100, 1e-10, 1, prec=prec)
        print(f"   prec={prec} steps={r['steps']} sw={r['switch_step']} pre={r['pre_polish_residual'] / math.sqrt(d):.2e} "
              f"res={r['residual'] / math.sqrt(d):.2e} err={checks.frob_per_sqrt_d(R.cpu().numpy(), o['R']):.2e}", flush=True)
