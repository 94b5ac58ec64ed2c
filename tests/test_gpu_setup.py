"""N1 on the GPU: the device scale bound (alpha = 0), inertia probes from the trace certificate, and the
certified midpoint shift by inertia-probe bisection (alg:ssr steps 3-5; prop:reuse_refresh,
P:587-651) -- configs[2]'s shift produced on the device instead of by the oracle's Jacobi solve."""
import json
import math
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle import checks, ns as ons, setup  # noqa: E402
import workloads  # noqa: E402

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def nsr():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2605_24840_b200 as m
    m.load_library()
    return m


def _dev():
    return torch.device("cuda:0")


@pytest.mark.parametrize("prec_name", ["NS_PREC_FP64", "NS_PREC_FP64_OZAKI", "NS_PREC_MIXED_BF16X3"])
def test_alpha_zero_is_the_device_gershgorin_bound(nsr, prec_name):
    """alpha = 0: the library takes alpha = ||H - sI||_inf from the device; the run equals the run with that
    alpha passed explicitly, bit for bit, and the bound equals the oracle's (within summation-order rounding)."""
    prec = getattr(nsr, prec_name)
    p = workloads.cfg3_dense(d=700, k=40)
    Hg = torch.from_numpy(p.H).to(_dev())
    R0, r0 = nsr.ns_reflector(Hg, 0.013, 0.0, p.k, 100, 1e-10, 1, prec=prec)
    ref = setup.inf_norm_shifted(p.H, 0.013)
    assert abs(r0["alpha"] - ref) <= 1e-13 * ref
    R1, r1 = nsr.ns_reflector(Hg, 0.013, r0["alpha"], p.k, 100, 1e-10, 1, prec=prec)
    assert torch.equal(R0, R1) and r0 == r1


def test_alpha_zero_batched_and_device_arrays(nsr):
    """Batched: per-problem alpha = 0 entries get their own device bound; the device-array entry gives the
    host-array entry's results bitwise."""
    probs = workloads.cfg1_batched(seed=2, n_matrices=2048, count=12)
    H = torch.from_numpy(np.stack([q.H for q in probs])).to(_dev())
    s = [q.s for q in probs]
    a = [0.0 if i % 2 else q.alpha for i, q in enumerate(probs)]
    k = [q.k for q in probs]
    R, outs = nsr.ns_reflector_batched(H, s, a, k, 100, 1e-12)
    for i, q in enumerate(probs):
        want = setup.inf_norm_shifted(q.H, q.s) if i % 2 else q.alpha
        assert abs(outs[i]["alpha"] - want) <= 1e-13 * want
        assert outs[i]["cert"] == q.k
    Rd, outd = nsr.ns_reflector_batched_dev(H, torch.tensor(s, dtype=torch.float64, device=_dev()),
                                            torch.tensor(a, dtype=torch.float64, device=_dev()),
                                            torch.tensor(k, dtype=torch.int32, device=_dev()), 100, 1e-12)
    assert torch.equal(R, Rd) and outs == outd
    with pytest.raises(nsr.NsError, match="alpha"):
        nsr.ns_reflector_batched_dev(H, torch.tensor(s, dtype=torch.float64, device=_dev()),
                                     torch.full((len(s),), -1.0, dtype=torch.float64, device=_dev()),
                                     torch.tensor(k, dtype=torch.int32, device=_dev()), 100, 1e-12)


@pytest.mark.parametrize("prec_name", ["NS_PREC_FP64", "NS_PREC_FP64_OZAKI"])
@pytest.mark.parametrize("d", [50, 301, 1200])
def test_inertia_probe_counts(nsr, prec_name, d):
    """ns_inertia == #{lambda < s} (the oracle's definition on LAPACK eigenvalues) at shifts between
    eigenvalues, including shifts very close to one (tiny scaled margin: a long but resolved run)."""
    prec = getattr(nsr, prec_name)
    rng = np.random.default_rng(1000 + d)
    A = rng.standard_normal((d, d))
    A = 0.5 * (A + A.T) / math.sqrt(d)
    w = np.linalg.eigvalsh(A)
    Ag = torch.from_numpy(A).to(_dev())
    idx = sorted(set(rng.integers(1, d - 1, 5).tolist()) | {1, d // 2, d - 2})
    for i in idx:
        for frac in (0.5, 1e-3):
            s = w[i - 1] + frac * (w[i] - w[i - 1])
            c, resolved, res = nsr.ns_inertia(Ag, s, prec=prec)
            assert resolved and c == setup.inertia(w, s) == i, (i, frac, c, res)
            assert res["residual"] < 0.5 / math.sqrt(d)
    # outside the spectrum: 0 and d
    assert nsr.ns_inertia(Ag, w[0] - 1.0, prec=prec)[0] == 0
    assert nsr.ns_inertia(Ag, w[-1] + 1.0, prec=prec)[0] == d


@pytest.mark.parametrize("seed,prec_name", [(0, "NS_PREC_FP64"), (1, "NS_PREC_FP64_OZAKI"),
                                            (2, "NS_PREC_FP64_OZAKI"), (3, "NS_PREC_FP64")])
def test_cfg2_shift_from_device_bisection(nsr, seed, prec_name):
    """configs[2] (Allen-Cahn, d = 4096, k = 5) with the shift produced on the device: inertia-probe bisection
    from the bracket [-||H||_inf, ||H||_inf] to a prop:reuse_refresh-certified midpoint (rel_eps 0.05).  The
    probe sequence and the shift equal the reference algorithm's (oracle/setup.py shift_bisect on LAPACK
    eigenvalue counts) bit for bit; the shift lies in (lambda_5, lambda_6) of the oracle's Jacobi spectrum
    (tests/golden); the reflector at that shift, with the device Gershgorin alpha, matches the oracle's NS run
    (steps, certificate 5, flags, R within 1e-10)."""
    g = json.load(open(os.path.join(GOLD, f"cfg2_seed{seed}.json")))
    prob = workloads.cfg2_allen_cahn(seed=seed, s=g["s"])
    H = prob.H
    w = np.linalg.eigvalsh(H)
    assert np.max(np.abs(w[:12] - np.array(g["lam_low"]))) <= 1e-13 * np.max(np.abs(w))   # LAPACK vs the oracle's Jacobi
    hi = setup.inf_norm_shifted(H, 0.0) * (1.0 + 1e-12)
    ref = setup.shift_bisect(lambda s: setup.inertia(w, s), 5, -hi, hi, 0.05, 200)
    assert ref["ok"]
    Hg = torch.from_numpy(H).to(_dev())
    out = nsr.ns_shift_bisect(Hg, 5, -hi, hi, rel_eps=0.05, max_probes=200, prec=getattr(nsr, prec_name))
    assert out["ok"] and out["unresolved"] == 0
    assert out["probes"] == ref["probes"] and out["s"] == ref["s"]
    for key in ("lam_k_lo", "lam_k_hi", "lam_k1_lo", "lam_k1_hi", "eps"):
        assert out[key] == ref[key], key
    lam5, lam6 = g["lam_low"][4], g["lam_low"][5]
    assert lam5 < out["s"] < lam6
    assert abs(out["alpha"] - setup.inf_norm_shifted(H, out["s"])) <= 1e-13 * out["alpha"]
    R, res = nsr.ns_reflector(Hg, out["s"], 0.0, 5, 100, 1e-12, 0)
    assert res["alpha"] == out["alpha"]
    o = ons.ns_reflector(H, out["s"], res["alpha"], 5, 100, 1e-12, 0, trace_residuals=True)
    assert res["cert"] == o["cert"] == 5
    thr = 1e-12
    tie = any(abs(r_ - thr) <= 0.01 * thr for r_ in o["hist_residual"][max(0, o["steps"] - 1): o["steps"] + 1])
    if not tie:
        assert res["steps"] == o["steps"] and res["flags"] == o["flags"]
    assert checks.frob_per_sqrt_d(R.cpu().numpy(), o["R"]) <= 1e-10
