"""Write tests/golden/cfg2_seed<N>.json (+ .npz of sampled columns) for configs[2].

Calls only oracle/ (cyclic Jacobi, NS loop) and workloads/ (the input recipe).
configs[2]: "s = midpoint of lambda_5 and lambda_6 computed by the oracle, alpha
from the Gershgorin bound".  Stored: the oracle's lowest 12 Jacobi eigenvalues,
s, alpha, gamma, the oracle NS result (steps, residual, trace, cert, flags) and a
few sampled columns of R_ns (oracle NS) and R_eig (Jacobi I - 2P_5).
Run:  OMP_NUM_THREADS=8 python tools/make_golden_cfg2.py <seed> [<seed> ...]
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import jacobi, ns, scalar  # noqa: E402
import workloads  # noqa: E402

GOLD = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")
COLS = [0, 1, 777, 2048, 4095]


def main(seeds):
    for seed in seeds:
        prob = workloads.cfg2_allen_cahn(seed=seed)
        t0 = time.time()
        w, V, sweeps = jacobi.jacobi_eigh(prob.H)
        t_jac = time.time() - t0
        s = jacobi.midpoint_shift(w, 5)
        alpha = workloads.configs.gershgorin_alpha(prob.H, s)
        t0 = time.time()
        out = ns.ns_reflector(prob.H, s, alpha, 5, 100, 1e-12, ns.TOL_ABS, trace_residuals=True)
        t_ns = time.time() - t0
        R_eig_cols = np.eye(prob.d)[:, COLS] - 2.0 * V[:, :5] @ V[COLS, :5].T
        gamma = scalar.scaled_margin(w, s, alpha)
        steps_pred = scalar.predict_run((w - s) / alpha, 100, 1e-12, False)[0]
        rec = dict(
            _source="tools/make_golden_cfg2.py (oracle/ only): cyclic Jacobi (S:79) + NS loop; configs[2] recipe C12",
            seed=seed, d=prob.d, k=5, lam_low=w[:12].tolist(), lam_max=float(w[-1]), s=s, alpha=alpha,
            gamma=gamma, jacobi_sweeps=sweeps, steps_pred_from_jacobi_lambda=steps_pred,
            ns=dict(steps=out["steps"], residual=out["residual"], trace=out["trace"], cert=out["cert"],
                    flags=out["flags"], hist_residual=out["hist_residual"]),
            cols=COLS, seconds=dict(jacobi=t_jac, ns=t_ns), threads=os.environ.get("OMP_NUM_THREADS"),
            ns_vs_eig_cols_max=float(np.max(np.abs(out["R"][:, COLS] - R_eig_cols))),
        )
        with open(os.path.join(GOLD, f"cfg2_seed{seed}.json"), "w") as f:
            json.dump(rec, f, indent=1)
        np.savez_compressed(os.path.join(GOLD, f"cfg2_seed{seed}_cols.npz"), cols=np.array(COLS),
                            R_ns=out["R"][:, COLS], R_eig=R_eig_cols)
        print(json.dumps({k: rec[k] for k in ("seed", "s", "alpha", "gamma", "jacobi_sweeps", "steps_pred_from_jacobi_lambda")}),
              rec["ns"]["steps"], rec["ns"]["cert"], rec["seconds"], rec["ns_vs_eig_cols_max"], flush=True)


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [0])
