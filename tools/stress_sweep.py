"""Randomised stress of every path against the oracle (bug hunting; failures are printed with their seed).
usage: python tools/stress_sweep.py [n_fp64] [n_ozaki] [n_mixed] [seed0]"""
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_24840_b200 as nsr  # noqa: E402
import workloads  # noqa: E402
from oracle import checks, ns as ons  # noqa: E402

TOL_R = 1e-10


def tie(o, tol, tm, d):
    t = tol if tm == 0 else tol * math.sqrt(d)
    h = o["hist_residual"]
    cand = [h[o["steps"]]] + ([h[o["steps"] - 1]] if o["steps"] > 0 else [])
    return any(abs(r - t) <= 0.01 * t for r in cand)


def mixed_step_ok(r, o, tol, tm, d):
    """Reading C16b (round 2: switch at r/sqrt(d) < 1e-3): the mixed path must take the oracle's step count; a
    difference of one is not a failure only inside the predicate DESIGN C16b names: the oracle's residual at its
    decision step or the one before within 3% of the threshold (a late switch is handled by the library: the last
    low-precision step is redone in FP64-class arithmetic)."""
    t = tol if tm == 0 else tol * math.sqrt(d)
    h = o["hist_residual"]
    if abs(r["steps"] - o["steps"]) != 1:
        return False
    band = 0.03
    return any((1 - band) * t <= h[j] <= (1 + band) * t for j in (o["steps"] - 1, o["steps"]) if 0 <= j < len(h))


def problem(seed, dmax):
    rng = np.random.default_rng(seed)
    d = int(rng.integers(1, dmax))
    k = int(rng.integers(0, d + 1))
    g = 10.0 ** rng.uniform(-3.5, math.log10(0.5))
    cluster = rng.random() < 0.3
    neg = -rng.uniform(g / 2, 1.0, k) if not cluster else -(g / 2 + rng.exponential(0.01, k))
    pos = rng.uniform(g / 2, 1.0, d - k) if not cluster else g / 2 + rng.exponential(0.01, d - k)
    lam = np.concatenate([neg, pos]) * 10.0 ** rng.uniform(-2, 2)
    Q = workloads.haar_q(rng, d)
    H = (Q * lam[None, :]) @ Q.T
    H = 0.5 * (H + H.T)
    scale = float(np.max(np.abs(lam))) if d else 1.0
    s = float(rng.uniform(-0.4, 0.4) * g * scale)
    alpha = float(np.max(np.abs(lam - s))) * float(rng.choice([1.0, 1.001, 1.1, 2.0]))
    tm = int(rng.integers(0, 2))
    tol = float(rng.choice([1e-8, 1e-10, 1e-12]))
    ms = int(rng.choice([0, 1, 5, 30, 100]))
    return H, s, alpha, k, ms, tol, tm


def main():
    n64, noz, nmx, s0 = [int(x) for x in (sys.argv[1:] + ["120", "40", "30", "0"])[:4]]
    fails = 0
    dm = int(os.environ.get("STRESS_DMAX", "0"))   # larger sizes (2-SM split-precision kernel, 128-tile paths)
    for path, n, dmax, precs in (("fp64", n64, dm or 400, [0]), ("ozaki", noz, dm or 400, [3]),
                                 ("mixed", nmx, dm or 600, [1, 2])):
        for i in range(n):
            seed = 10_000 * (1 + precs[0]) + s0 + i
            H, s, alpha, k, ms, tol, tm = problem(seed, dmax)
            d = H.shape[0]
            if path == "mixed":
                ms, tol, tm = 100, 1e-10, 1
                alpha = max(alpha, float(np.linalg.norm(H - s * np.eye(d), 2)) * 1.01)
            o = ons.ns_reflector(H, s, alpha, k, ms, tol, tm, trace_residuals=True)
            for prec in precs:
                try:
                    R, r = nsr.ns_reflector(torch.from_numpy(H).cuda(), s, alpha, k, ms, tol, tm, prec=prec)
                except Exception as e:  # noqa: BLE001
                    print(f"FAIL {path} seed={seed} d={d} prec={prec}: exception {e}", flush=True)
                    fails += 1
                    continue
                Rn = R.cpu().numpy()
                msg = []
                if r["cert"] != o["cert"]:
                    msg.append(f"cert {r['cert']} vs {o['cert']}")
                # the Ozaki products' residual floor is ~1.5e-15 d (absolute; FP64 DMMA: ~3e-17 d, DESIGN Ozaki
                # section): tolerances within 10x of it are not expected to give the oracle's step count
                t_abs = tol if tm == 0 else tol * math.sqrt(d)
                below_floor = path == "ozaki" and tol > 0 and t_abs < 5e-16 * d   # 8-group floor ~4e-17 d
                if not (tol > 0 and tie(o, tol, tm, d)) and not below_floor:
                    ok_steps = r["steps"] == o["steps"] or (path == "mixed" and mixed_step_ok(r, o, tol, tm, d))
                    if not ok_steps:
                        msg.append(f"steps {r['steps']} vs {o['steps']}")
                    elif not (o["flags"] & (ons.SCALING_SUSPECT | ons.NONFINITE)) and r["steps"] == o["steps"]:
                        e = checks.frob_per_sqrt_d(Rn, o["R"])
                        if e > TOL_R:
                            msg.append(f"err {e:.2e}")
                if msg:
                    fails += 1
                    print(f"FAIL {path} seed={seed} d={d} k={k} s={s:.3g} alpha={alpha:.3g} ms={ms} tol={tol} tm={tm} "
                          f"prec={prec} flags={r['flags']}/{o['flags']}: {'; '.join(msg)}", flush=True)
    print(f"done: {fails} failures", flush=True)


if __name__ == "__main__":
    main()


def batched_stress(n, seed0=0):
    """Random batches (FP64 and Ozaki) and random emulated-rank counts against the oracle per problem."""
    fails = 0
    for i in range(n):
        rng = np.random.default_rng(90_000 + seed0 + i)
        seeds = [int(x) for x in rng.integers(0, 10**9, int(rng.integers(1, 24)))]
        first = problem(seeds[0], 400)
        d = first[0].shape[0]
        probs = [first]
        for sd in seeds[1:]:
            H, s, alpha, k, _, _, _ = problem(sd, 2)   # d = 1 placeholder, replaced below
            r2 = np.random.default_rng(sd)
            lam = np.sort(r2.uniform(-1, 1, d))
            lam[np.abs(lam) < 0.02] = 0.02
            Q = workloads.haar_q(r2, d)
            H = (Q * lam[None, :]) @ Q.T
            H = 0.5 * (H + H.T)
            k = int(np.sum(lam < 0))
            probs.append((H, 0.0, float(np.max(np.abs(lam))) * float(r2.choice([1.0, 1.2])), k, 0, 0, 0))
        ms, tol, tm = first[4], first[5], first[6]
        Hs = torch.from_numpy(np.stack([p[0] for p in probs])).cuda()
        for prec in (0, 3):
            R, outs = nsr.ns_reflector_batched(Hs, [p[1] for p in probs], [p[2] for p in probs],
                                               [p[3] for p in probs], ms, tol, tm, prec=prec)
            R = R.cpu().numpy()
            for b, p in enumerate(probs):
                o = ons.ns_reflector(p[0], p[1], p[2], p[3], ms, tol, tm, trace_residuals=True)
                msg = []
                if outs[b]["cert"] != o["cert"]:
                    msg.append(f"cert {outs[b]['cert']} vs {o['cert']}")
                if not (tol > 0 and tie(o, tol, tm, d)):
                    if outs[b]["steps"] != o["steps"]:
                        msg.append(f"steps {outs[b]['steps']} vs {o['steps']}")
                    elif not (o["flags"] & (ons.SCALING_SUSPECT | ons.NONFINITE)):
                        e = checks.frob_per_sqrt_d(R[b], o["R"])
                        if e > TOL_R:
                            msg.append(f"err {e:.2e}")
                if msg:
                    fails += 1
                    print(f"FAIL batched i={i} d={d} batch={len(probs)} b={b} prec={prec}: {'; '.join(msg)}", flush=True)
        # emulated ranks on the first problem
        H, s, alpha, k, ms, tol, tm = first
        P = int(rng.integers(2, 9))
        Re, re_ = nsr.ns_reflector_sharded_emulated(P, torch.from_numpy(H).cuda(), s, alpha, k, ms, tol, tm)
        Rd, rd = nsr.ns_reflector(torch.from_numpy(H).cuda(), s, alpha, k, ms, tol, tm)
        o = ons.ns_reflector(H, s, alpha, k, ms, tol, tm, trace_residuals=True)
        if re_["cert"] != o["cert"] or (not (tol > 0 and tie(o, tol, tm, d)) and re_["steps"] != o["steps"]):
            fails += 1
            print(f"FAIL emulated i={i} d={d} P={P}: steps {re_['steps']} vs {o['steps']}, cert {re_['cert']}", flush=True)
    print(f"batched/emulated done: {fails} failures", flush=True)


if __name__ == "__main__" and os.environ.get("STRESS_BATCHED"):
    batched_stress(int(os.environ["STRESS_BATCHED"]))


def graded_stress(n, seed0=0):
    """Graded matrices H = D A D (D log-uniform over 6 decades, A a random symmetric matrix): rows of very
    different magnitude (the Ozaki split scales per row); shift at the midpoint of a random spectral gap."""
    fails = 0
    for i in range(n):
        rng = np.random.default_rng(70_000 + seed0 + i)
        d = int(rng.integers(2, 400))
        Dg = 10.0 ** rng.uniform(-6, 0, d)
        A = rng.standard_normal((d, d))
        H = (Dg[:, None] * (0.5 * (A + A.T))) * Dg[None, :]
        lam = np.linalg.eigvalsh(H)
        k = int(rng.integers(1, d))
        s = 0.5 * (lam[k - 1] + lam[k])
        alpha = float(np.max(np.abs(lam - s))) * 1.01
        tol, tm = 1e-10, 1
        o = ons.ns_reflector(H, s, alpha, k, 200, tol, tm, trace_residuals=True)
        for prec in (0, 3):
            R, r = nsr.ns_reflector(torch.from_numpy(H).cuda(), s, alpha, k, 200, tol, tm, prec=prec)
            msg = []
            if r["cert"] != o["cert"]:
                msg.append(f"cert {r['cert']} vs {o['cert']}")
            if not tie(o, tol, tm, d):
                if r["steps"] != o["steps"]:
                    msg.append(f"steps {r['steps']} vs {o['steps']}")
                elif o["flags"] & ons.CONVERGED:
                    e = checks.frob_per_sqrt_d(R.cpu().numpy(), o["R"])
                    if e > TOL_R:
                        msg.append(f"err {e:.2e}")
            if msg:
                fails += 1
                print(f"FAIL graded i={i} d={d} k={k} prec={prec} flags={r['flags']}/{o['flags']}: {'; '.join(msg)}",
                      flush=True)
    print(f"graded done: {fails} failures", flush=True)


if __name__ == "__main__" and os.environ.get("STRESS_GRADED"):
    graded_stress(int(os.environ["STRESS_GRADED"]))


def host_stress(n, seed0=0):
    """Host entry (pinned: chunked staging + speculative copy; pageable: plain copies) vs the device entry,
    bitwise, on random problems of the chunked-path sizes."""
    fails = 0
    for i in range(n):
        rng = np.random.default_rng(80_000 + seed0 + i)
        H, s, alpha, k, ms, tol, tm = problem(80_000 + seed0 + i, 2)
        d = int(rng.integers(1024, 3000))
        lam = np.concatenate([-rng.uniform(0.01, 1.0, d // 4), rng.uniform(0.01, 1.0, d - d // 4)])
        Q = workloads.haar_q(rng, d)
        H = (Q * lam[None, :]) @ Q.T
        H = 0.5 * (H + H.T)
        s, alpha, k = 0.0, 1.0 * float(rng.choice([1.0, 1.3])), d // 4
        ms, tol, tm = int(rng.choice([5, 30, 100])), float(rng.choice([0.0, 1e-10, 1e-12])), int(rng.integers(0, 2))
        pinned = bool(rng.integers(0, 2))
        Hh = torch.from_numpy(H)
        Rh = torch.empty((d, d), dtype=torch.float64)
        if pinned:
            Hh, Rh = Hh.pin_memory(), Rh.pin_memory()
        prec = int(rng.choice([0, 0, 1, 3]))
        Rh, rh = nsr.ns_reflector_host(Hh, s, alpha, k, ms, tol, tm, R=Rh, prec=prec)
        Rd, rd = nsr.ns_reflector(torch.from_numpy(H).cuda(), s, alpha, k, ms, tol, tm, prec=prec)
        same = torch.equal(Rh, Rd.cpu()) and all(rh[q] == rd[q] for q in ("steps", "flags", "cert", "residual"))
        if not same:
            fails += 1
            print(f"FAIL host i={i} d={d} prec={prec} pinned={pinned} ms={ms} tol={tol}: {rh} vs {rd}", flush=True)
    print(f"host done: {fails} failures", flush=True)


if __name__ == "__main__" and os.environ.get("STRESS_HOST"):
    host_stress(int(os.environ["STRESS_HOST"]))
