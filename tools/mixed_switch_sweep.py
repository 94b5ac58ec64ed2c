"""Mixed-path step-count experiment: switch threshold tau vs. step equality with the oracle.

For seeded random problems drawn like tests/test_gpu_parity.py::test_random_sweep_mixed (d 130..512, gaps
1e-3..0.3, run to ||X^2 - I||_F/sqrt(d) < 1e-10), run the mixed BF16x3 path with options.switch_tol = tau for
several tau and record the step difference to the oracle, the oracle's residual margins at its decision step
and the step before (r / threshold), and ||R - R_oracle||_F/sqrt(d).  Then time configs[3] at each tau.

usage: python tools/mixed_switch_sweep.py [n_problems] > gpurun_out/mixed_switch.jsonl
"""
import json
import math
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2605_24840_b200 as nsr  # noqa: E402
import workloads  # noqa: E402
from oracle import ns as ons  # noqa: E402

TAUS = [float(t) for t in os.environ.get("TAUS", "1e-4,1e-3,3e-3,1e-2,3e-2").split(",")]


def problem(seed):
    rng = np.random.default_rng(2000 + seed)
    d = int(rng.choice([130, 200, 256, 300, 512]))
    k = int(rng.integers(1, d))
    g = 10.0 ** rng.uniform(-3 if seed >= 6 else -2, math.log10(0.3))
    lam = np.concatenate([-rng.uniform(g / 2, 1.0, k), rng.uniform(g / 2, 1.0, d - k)])
    Q = workloads.haar_q(rng, d)
    H = (Q * lam[None, :]) @ Q.T
    H = 0.5 * (H + H.T)
    s = float(rng.uniform(-0.3, 0.3) * g)
    alpha = float(np.linalg.norm(H - s * np.eye(d), 2)) * 1.02
    return H, s, alpha, k


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    first = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    dev = torch.device("cuda:0")
    nsr.load_library()
    for seed in range(first, first + n):
        H, s, alpha, k = problem(seed)
        d = H.shape[0]
        thr = 1e-10 * math.sqrt(d)
        o = ons.ns_reflector(H, s, alpha, k, 100, 1e-10, 1, trace_residuals=True)
        h = o["hist_residual"]
        Hg = torch.from_numpy(H).to(dev)
        for tau in TAUS:
            R, r = nsr.ns_reflector(Hg, s, alpha, k, 100, 1e-10, 1, prec=nsr.NS_PREC_MIXED_BF16X3,
                                    options=nsr.ns_options(switch_tol=tau))
            err = float(np.linalg.norm(R.cpu().numpy() - o["R"]) / math.sqrt(d))
            print(json.dumps(dict(seed=seed, d=d, tau=tau, steps=r["steps"], oracle_steps=o["steps"],
                                  dsteps=r["steps"] - o["steps"], switch=r["switch_step"],
                                  margin_dec=h[o["steps"]] / thr, margin_prev=h[o["steps"] - 1] / thr,
                                  r_switch_oracle=(h[r["switch_step"]] / math.sqrt(d)) if 0 <= r["switch_step"] < len(h)
                                  else None, err=err, cert_ok=r["cert"] == k,
                                  res_ratio=(r["residual"] / o["residual"]) if r["steps"] == o["steps"] else None,
                                  res_ratio_prev=None)), flush=True)
    if os.environ.get("NO_CFG3"):
        return
    # configs[3] timing per tau
    p = workloads.cfg3_dense(form=False)
    Hc = workloads.householder_form_fast(p.Vh, p.lam, device=dev)
    ws = nsr.alloc_workspace(nsr.ns_workspace_bytes(p.d, nsr.NS_PREC_MIXED_BF16X3), dev)
    Rc = torch.empty_like(Hc)
    for tau in TAUS:
        for polish in (2, 1):
            opts = nsr.ns_options(switch_tol=tau, polish=polish)
            nsr.ns_reflector(Hc, p.s, p.alpha, p.k, p.max_steps, p.tol, p.tol_mode, R=Rc, ws=ws,
                             prec=nsr.NS_PREC_MIXED_BF16X3, options=opts)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            _, r = nsr.ns_reflector(Hc, p.s, p.alpha, p.k, p.max_steps, p.tol, p.tol_mode, R=Rc, ws=ws,
                                    prec=nsr.NS_PREC_MIXED_BF16X3, options=opts)
            e1.record()
            torch.cuda.synchronize()
            print(json.dumps(dict(cfg3=True, tau=tau, polish=polish, ms=e0.elapsed_time(e1), steps=r["steps"],
                                  switch=r["switch_step"], cert=r["cert"])), flush=True)


if __name__ == "__main__":
    main()
