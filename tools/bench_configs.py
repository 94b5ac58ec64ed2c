"""Measure every BASELINE config on one B200 (the bench.py line covers configs[3] only).

usage: python tools/bench_configs.py [cfg0 cfg1 cfg2 cfg3 cfg3mixed cfg3fixed cfg4 ...] > profiles/rNN_configs.jsonl

Every record: config, time (CUDA events on the launching stream, after warm-up), algorithmic
TFLOP/s ((2 steps + 1) d^3 per reflector), reflectors/s, steps, cert, flags and a correctness
check against something the oracle side fixes (closed forms / golden files / scalar replay).
The oracle itself is not run here except where noted.
"""
import json
import math
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2605_24840_b200 as nsr  # noqa: E402
import workloads  # noqa: E402
from oracle import closed_form, scalar  # noqa: E402

DEV = torch.device("cuda:0")
PEAK = 36.97


def timed(fn, reps, warm=1):
    for _ in range(warm):
        out = fn()
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    times = []
    for _ in range(reps):
        e0.record(s)
        out = fn()
        e1.record(s)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    return out, float(np.median(times)), times


def emit(rec):
    print(json.dumps(rec), flush=True)


def cfg0():
    for seed in range(5):
        p = workloads.cfg0_controlled(seed)
        H = torch.from_numpy(p.H).to(DEV)
        R = torch.empty_like(H)
        ws = nsr.alloc_workspace(nsr.ns_workspace_bytes(p.d), DEV)
        (R, res), ms, _ = timed(lambda: nsr.ns_reflector(H, p.s, p.alpha, p.k, 100, 1e-12, R=R, ws=ws), 100, 5)
        err = float(np.linalg.norm(R.cpu().numpy() - closed_form.reflector_explicit_q(p.Q, p.lam, p.s)) / 8)
        emit({"config": "cfg0", "seed": seed, "d": 64, "time_to_R_us": ms * 1e3, "steps": res["steps"],
              "cert": res["cert"], "flags": res["flags"], "err_vs_closed_form": err, "launches": res["launches"],
              "tflops": (2 * res["steps"] + 1) * 64 ** 3 / (ms * 1e-3) / 1e12})


def cfg1(n_mat=2048, prec=nsr.NS_PREC_FP64):
    t0 = time.time()
    probs = workloads.cfg1_batched(seed=0, n_matrices=2048, count=n_mat)
    gen_s = time.time() - t0
    H = torch.from_numpy(np.stack([p.H for p in probs])).to(DEV)
    ws = nsr.alloc_workspace(nsr.ns_workspace_bytes_batched(256, len(probs), prec), DEV)
    R = torch.empty_like(H)
    s_, a_, k_ = [p.s for p in probs], [p.alpha for p in probs], [p.k for p in probs]
    (R, outs), ms, _ = timed(lambda: nsr.ns_reflector_batched(H, s_, a_, k_, 100, 1e-12, R=R, ws=ws, prec=prec), 3, 1)
    steps = np.array([o["steps"] for o in outs])
    pred = np.array([scalar.predict_run((p.lam - p.s) / p.alpha, 100, 1e-12, False)[0] for p in probs])
    certs_ok = all(o["cert"] == p.k for o, p in zip(outs, probs))
    flops = float(np.sum(2 * steps + 1)) * 256.0 ** 3
    # direction error on a sample (closed form, prop:direrr)
    Rn = R.cpu().numpy()
    derr = max(float(np.linalg.norm((Rn[i] - closed_form.reflector_explicit_q(probs[i].Q, probs[i].lam, probs[i].s))
                                    @ probs[i].extra["probe"])) for i in range(0, len(probs), max(1, len(probs) // 64)))
    mid = steps[0::3]
    off = np.minimum(steps[1::3], steps[2::3])
    emit({"config": "cfg1", "prec": {0: "fp64", 3: "fp64_ozaki_int8"}[prec], "problems": len(probs), "d": 256,
          "time_ms": ms, "reflectors_per_s": len(probs) / (ms * 1e-3),
          "tflops": flops / (ms * 1e-3) / 1e12, "steps_sum": int(steps.sum()), "steps_min": int(steps.min()),
          "steps_max": int(steps.max()), "steps_equal_prediction": int(np.sum(steps == pred)),
          "steps_off_by_one": int(np.sum(np.abs(steps - pred) == 1)), "certs_ok": certs_ok,
          "midpoint_strictly_fewer": int(np.sum(mid < off)), "max_direction_error_sampled": derr,
          "launches": outs[0]["launches"], "host_generation_s": gen_s})


def cfg2(seed=0):
    g = json.load(open(os.path.join(ROOT, "tests", "golden", f"cfg2_seed{seed}.json")))
    prob = workloads.cfg2_allen_cahn(seed=seed, s=g["s"])
    H = torch.from_numpy(prob.H).to(DEV)
    R = torch.empty_like(H)
    ws = nsr.alloc_workspace(nsr.ns_workspace_bytes(4096), DEV)
    (R, res), ms, _ = timed(lambda: nsr.ns_reflector(H, g["s"], g["alpha"], 5, 100, 1e-12, R=R, ws=ws), 5, 1)
    cols = np.load(os.path.join(ROOT, "tests", "golden", f"cfg2_seed{seed}_cols.npz"))
    Rc = R[:, torch.as_tensor(cols["cols"], device=DEV)].cpu().numpy()
    err = float(np.sqrt(np.mean(np.sum((Rc - cols["R_ns"]) ** 2, axis=0))))
    emit({"config": "cfg2", "seed": seed, "d": 4096, "time_to_R_ms": ms, "steps": res["steps"],
          "oracle_steps": g["ns"]["steps"], "cert": res["cert"], "flags": res["flags"], "gamma": g["gamma"],
          "tflops": (2 * res["steps"] + 1) * 4096.0 ** 3 / (ms * 1e-3) / 1e12, "err_vs_oracle_cols": err})


def cfg3(mode="tol", prec=nsr.NS_PREC_FP64, reps=3, polish=0):
    p = workloads.cfg3_dense(form=False, mode=mode)
    H = workloads.householder_form_fast(p.Vh, p.lam, device=DEV)
    R = torch.empty_like(H)
    ws = nsr.alloc_workspace(nsr.ns_workspace_bytes(p.d, prec), DEV)
    opts = nsr.ns_options(polish=polish) if polish else None
    (R, res), ms, _ = timed(lambda: nsr.ns_reflector(H, p.s, p.alpha, p.k, p.max_steps, p.tol, p.tol_mode, R=R, ws=ws,
                                                     prec=prec, options=opts), reps, 1)
    cols = np.array([0, 1, 9999, 16383])
    Rc = closed_form.householder_reflector_columns(p.Vh, p.lam, 0.0, cols)
    Rg = R[:, torch.as_tensor(cols, device=DEV)].cpu().numpy()
    err = float(np.sqrt(np.mean(np.sum((Rg - Rc) ** 2, axis=0))))
    tf = (2 * res["steps"] + 1) * float(p.d) ** 3 / (ms * 1e-3) / 1e12
    emit({"config": "cfg3", "mode": mode, "prec": {0: "fp64", 1: "mixed_bf16x3", 2: "mixed_tf32x3",
                                                   3: "fp64_ozaki_int8"}[prec] + {0: "", 1: "+ozaki_polish", 2: "+ozaki_reanchor"}[polish],
          "d": p.d,
          "time_to_R_ms": ms, "steps": res["steps"], "cert": res["cert"], "flags": res["flags"],
          "switch_step": res["switch_step"], "tflops": tf, "frac_fp64_peak": tf / PEAK, "err_vs_closed_form": err,
          "launches": res["launches"]})
    del H, R, ws
    torch.cuda.empty_cache()


def cfg4(sharded=True, prec=nsr.NS_PREC_FP64):
    p = workloads.cfg4_sharded(form=False)
    H = workloads.householder_form_fast(p.Vh, p.lam, device=DEV)
    R = torch.empty_like(H)
    if sharded:
        uid = nsr.ns_comm_get_unique_id()
        comm = nsr.ns_comm_init(0, 1, uid)
        ws = nsr.alloc_workspace(nsr.ns_workspace_bytes_sharded(p.d, 1), DEV)
        fn = lambda: nsr.ns_reflector_sharded(comm, H, p.s, p.alpha, p.k, p.max_steps, p.tol, p.tol_mode, R=R, ws=ws)  # noqa: E731
    else:
        ws = nsr.alloc_workspace(nsr.ns_workspace_bytes(p.d, prec), DEV)
        fn = lambda: nsr.ns_reflector(H, p.s, p.alpha, p.k, p.max_steps, p.tol, p.tol_mode, R=R, ws=ws,  # noqa: E731
                                      prec=prec)
    (R, res), ms, _ = timed(fn, 1, 0)
    pred = scalar.predict_run((p.lam - p.s) / p.alpha, 100, 1e-10, True)[0]
    cols = np.array([0, 4095, 4096, 30000, 49151])
    Rc = closed_form.householder_reflector_columns(p.Vh, p.lam, 0.0, cols)
    Rg = R[:, torch.as_tensor(cols, device=DEV)].cpu().numpy()
    err = float(np.sqrt(np.mean(np.sum((Rg - Rc) ** 2, axis=0))))
    probe = torch.randn(p.d, dtype=torch.float64, device=DEV)
    inv = float(torch.linalg.vector_norm(R @ (R @ probe) - probe) / torch.linalg.vector_norm(probe))
    tf = (2 * res["steps"] + 1) * float(p.d) ** 3 / (ms * 1e-3) / 1e12
    emit({"config": "cfg4", "path": ("sharded P=1" if sharded else "single") + (" ozaki" if prec == 3 else ""),
          "d": p.d, "time_to_R_s": ms / 1e3,
          "steps": res["steps"], "predicted_steps": pred, "cert": res["cert"], "flags": res["flags"], "tflops": tf,
          "frac_fp64_peak": tf / PEAK, "err_vs_closed_form_cols": err, "probe_R2v_minus_v": inv,
          "trace_residual": abs(res["trace"] - (p.d - 2 * p.k)), "launches": res["launches"]})
    if sharded:
        nsr.ns_comm_destroy(comm)


def kscan():
    """§5.3 target-index scan (N2): d=64, k in {1,2,4,8,16}, 32 matched starts, m = exact/2/4/6."""
    Q, ks, starts = workloads.rotated_quartic_scan(d=64, n_starts=32)
    Qg = torch.from_numpy(Q).to(DEV)
    kk = [k for k in ks for _ in starts]
    x0 = torch.from_numpy(np.concatenate([starts for _ in ks])).to(DEV)
    for m in (0, 2, 4, 6):
        (xf, res), ms, _ = timed(lambda: nsr.ns_alg1_rotated_quartic(Qg, kk, x0, m, 0.2, 1000, 1e-10), 3, 1)
        per_k = {k: float(np.mean([r["success"] for r, kr in zip(res, kk) if kr == k])) for k in ks}
        emit({"config": "kscan", "m": m, "runs": len(kk), "time_ms": ms, "success_rate_by_k": per_k,
              "median_iters": float(np.median([r["iters"] for r in res]))})


def main():
    which = sys.argv[1:] or ["cfg0", "cfg1", "cfg2", "cfg3", "cfg3mixed", "cfg3fixed", "cfg3fixedmixed"]
    for w in which:
        if w == "cfg0":
            cfg0()
        elif w == "cfg1":
            cfg1()
        elif w == "cfg1small":
            cfg1(64)
        elif w == "cfg1ozaki":
            cfg1(prec=nsr.NS_PREC_FP64_OZAKI)
        elif w == "cfg2":
            cfg2(0)
            cfg2(1)
        elif w == "cfg3":
            cfg3("tol", nsr.NS_PREC_FP64)
        elif w == "cfg3mixed":
            cfg3("tol", nsr.NS_PREC_MIXED_BF16X3)
        elif w == "cfg3fixed":
            cfg3("fixed30", nsr.NS_PREC_FP64, reps=1)
        elif w == "cfg3fixedmixed":
            cfg3("fixed30", nsr.NS_PREC_MIXED_BF16X3, reps=1)
        elif w == "cfg3mixedoz":
            cfg3("tol", nsr.NS_PREC_MIXED_BF16X3, polish=1)
        elif w == "cfg3mixedoz2":
            cfg3("tol", nsr.NS_PREC_MIXED_BF16X3, polish=2)
        elif w == "cfg3fixedmixedoz":
            cfg3("fixed30", nsr.NS_PREC_MIXED_BF16X3, reps=1, polish=1)
        elif w == "cfg3tf32":
            cfg3("tol", nsr.NS_PREC_MIXED_TF32X3)
        elif w == "cfg3ozaki":
            cfg3("tol", nsr.NS_PREC_FP64_OZAKI)
        elif w == "cfg3fixedozaki":
            cfg3("fixed30", nsr.NS_PREC_FP64_OZAKI, reps=1)
        elif w == "cfg4":
            cfg4(True)
        elif w == "cfg4single":
            cfg4(False)
        elif w == "cfg4ozaki":
            cfg4(False, nsr.NS_PREC_FP64_OZAKI)
        elif w == "kscan":
            kscan()


if __name__ == "__main__":
    main()
