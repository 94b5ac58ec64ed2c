"""Diagnosis of the mixed path's late-switch problems (DESIGN reading C16b): the oracle's residual history next to
every precision path's steps, switch step, residuals and distance to the oracle's R, for the stress generator's
seeds 20000, 20022 (d < 600) and 20512 (d < 3000).  NS_MIXED_REDO=0 shows the behaviour before the redo step."""
import math, sys, os
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_24840_b200 as nsr
from oracle import ns as ons, checks
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import stress_sweep as ss
for seed, dm in ((20000, 600), (20022, 600), (20512, 3000)):
    H, s, alpha, k, ms, tol, tm = ss.problem(seed, dm)
    d = H.shape[0]
    ms, tol, tm = 100, 1e-10, 1
    alpha = max(alpha, float(np.linalg.norm(H - s * np.eye(d), 2)) * 1.01)
    o = ons.ns_reflector(H, s, alpha, k, ms, tol, tm, trace_residuals=True)
    t = tol if tm == 0 else tol * math.sqrt(d)
    print("seed", seed, "d", d, "k", k, "tol", tol, "tm", tm, "t", t, "oracle steps", o["steps"])
    print("  oracle hist", ["%.3e" % r for r in o["hist_residual"]])
    lam = np.linalg.eigvalsh(H)
    x = (lam - s) / alpha
    print("  min|x| %.3e max|x| %.6f" % (np.min(np.abs(x)), np.max(np.abs(x))))
    for prec in (0, 1, 2, 3):
        R, r = nsr.ns_reflector(torch.from_numpy(H).cuda(), s, alpha, k, ms, tol, tm, prec=prec)
        e = checks.frob_per_sqrt_d(R.cpu().numpy(), o["R"])
        print("  prec", prec, {kk: r[kk] for kk in ("steps", "flags", "residual", "switch_step", "pre_polish_residual", "cert")}, "err vs oracle R %.2e" % e)
