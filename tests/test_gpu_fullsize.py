"""Full-size parity: configs[1], configs[2] and configs[3] at their BASELINE sizes, every element of R
against the oracle's own Newton–Schulz output on the same input (north_star; reading C15).

For each run: identical step count (outside reading C9's +-1% tie band; inside it, +-1 and R compared
with the oracle's iterate at the GPU's step count), identical certificate and flags,
||R_gpu - R_oracle||_F / sqrt(d) <= 1e-10, and the reported residual and trace compared with the
oracle's values through bounds that follow from the measured difference of the returned iterates:

  | ||R_g^2 - I||_F - ||R_o^2 - I||_F |  <=  ||R_g^2 - R_o^2||_F + rounding
                                         <=  (||R_g||_2 + ||R_o||_2) ||R_g - R_o||_F + rounding
  | tr R_g - tr R_o |                    <=  sqrt(d) ||R_g - R_o||_F + rounding

with ||R||_2 <= 1 + 1e-6 for a converged iterate (its eigenvalues are p_m(mu) in [-1, 1] up to the
residual) and a rounding allowance of 64 u sqrt(d) for a residual (FP64 floor (2-4) u sqrt(d),
SURVEY EXP-1/EXP-10) and 8 u d for a trace.  Measured values are appended to $NS_PARITY_LOG (JSON lines)
when it is set; DESIGN.md §11 quotes them.

The oracle runs at full size on the host (tests/_oracle_runs.py; cached by input hash).
"""
import json
import math
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle import closed_form, ns as ons  # noqa: E402
import workloads  # noqa: E402
import _oracle_runs  # noqa: E402  (tests/ is on sys.path under pytest)

U = 2.0 ** -53
TOL_R = 1e-10
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


def _log(rec):
    path = os.environ.get("NS_PARITY_LOG")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(rec) + "\n")


def _tie(hist, thr, steps):
    cand = [hist[steps]] + ([hist[steps - 1]] if steps > 0 else [])
    return any(abs(r - thr) <= 0.01 * thr for r in cand)


def _frob_diff(A, B):
    """||A - B||_F in FP64, row block by row block (bounded memory at d = 16384)."""
    acc = 0.0
    for r0 in range(0, A.shape[0], 1024):
        D = A[r0:r0 + 1024] - B[r0:r0 + 1024]
        acc += float(np.sum(D * D))
    return math.sqrt(acc)


def check_run(label, Rg, res, o, d, thr, rerun=None, extra=None):
    """Element-by-element comparison of one GPU run with the oracle's run (see the module docstring).
    Rg: the GPU's R on the host (numpy); res: the C-ABI result; o: the oracle's result dict; thr: the
    absolute-equivalent stop threshold; rerun(steps): the oracle's iterate at a given fixed step count."""
    assert np.array_equal(Rg, Rg.T), f"{label}: R must be bitwise symmetric"
    tie = _tie(o["hist_residual"], thr, o["steps"])
    ref = o
    if res["steps"] != o["steps"]:
        assert tie and abs(res["steps"] - o["steps"]) == 1, (label, res["steps"], o["steps"])
        ref = rerun(res["steps"])      # the oracle's iterate at the GPU's step count
    else:
        assert res["flags"] == o["flags"], (label, res["flags"], o["flags"])
    assert res["cert"] == o["cert"], (label, res["cert"], o["cert"])
    dR = _frob_diff(Rg, ref["R"])
    err = dR / math.sqrt(d)
    assert err <= TOL_R, (label, err)
    nrm = 1.0 + 1e-6
    r_bound = 2.0 * nrm * dR + 64.0 * U * math.sqrt(d)
    assert abs(res["residual"] - ref["residual"]) <= r_bound, (label, res["residual"], ref["residual"], r_bound)
    t_bound = math.sqrt(d) * dR + 8.0 * U * d
    assert abs(res["trace"] - ref["trace"]) <= t_bound, (label, res["trace"], ref["trace"], t_bound)
    assert abs(res["trace"] - float(np.trace(Rg))) <= 8.0 * U * d, label
    rec = dict(test=label, d=d, steps=res["steps"], oracle_steps=o["steps"], tie_band=tie, cert=res["cert"],
               err_frob_per_sqrt_d=err, residual_gpu=res["residual"], residual_oracle=ref["residual"],
               trace_gpu=res["trace"], trace_oracle=ref["trace"])
    if extra:
        rec.update(extra)
    _log(rec)
    return rec


# --------------------------------------------------------------------------------------- configs[3]
@pytest.fixture(scope="module")
def cfg3_oracle():
    """configs[3] exactly as bench.py runs it (d = 16384, k = 1024, run to ||X^2 - I||_F/sqrt(d) < 1e-10),
    H formed on the host by the shared generator; the oracle's full NS run (~25 FP64 products)."""
    p = workloads.cfg3_dense(form=False)
    H = workloads.householder_form_fast(p.Vh, p.lam)
    o = _oracle_runs.ns_cached(H, p.s, p.alpha, p.k, p.max_steps, p.tol, p.tol_mode)
    return p, H, o


@pytest.mark.parametrize("prec_name", ["NS_PREC_FP64", "NS_PREC_MIXED_BF16X3", "NS_PREC_FP64_OZAKI"])
def test_cfg3_full_matrix_vs_oracle(nsr, cfg3_oracle, prec_name):
    p, H, o = cfg3_oracle
    prec = getattr(nsr, prec_name)
    Hg = torch.from_numpy(H).to(_dev())
    R, res = nsr.ns_reflector(Hg, p.s, p.alpha, p.k, p.max_steps, p.tol, p.tol_mode, prec=prec)
    Rg = R.cpu().numpy()
    del R, Hg
    torch.cuda.empty_cache()
    rec = check_run(f"cfg3[{prec_name}]", Rg, res, o, p.d, p.tol * math.sqrt(p.d),
                    extra=dict(switch_step=res["switch_step"], pre_polish_residual=res["pre_polish_residual"]))
    assert rec["steps"] == 12 and rec["cert"] == 1024
    # the oracle itself against the closed form R = Q sgn(Lambda) Q^T on sampled columns (prop:exact)
    cols = np.array([0, 1023, 1024, 8191, 16383])
    Rc = closed_form.householder_reflector_columns(p.Vh, p.lam, 0.0, cols)
    assert np.max(np.abs(o["R"][:, cols] - Rc)) <= 1e-12


# --------------------------------------------------------------------------------------- configs[2]
@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_cfg2_full_matrix_vs_oracle(nsr, seed):
    """configs[2] (Allen–Cahn, d = 4096) seeds 0-3: s and alpha from the oracle's Jacobi midpoint and
    Gershgorin bound (tests/golden/cfg2_seed<N>.json, tools/make_golden_cfg2.py); the FP64 path and the
    Ozaki path (8 digit-pair groups at this absolute tolerance) against the oracle's full R."""
    path = os.path.join(GOLD, f"cfg2_seed{seed}.json")
    if not os.path.exists(path):
        pytest.fail(f"missing golden file {path} (tools/make_golden_cfg2.py {seed})")
    g = json.load(open(path))
    prob = workloads.cfg2_allen_cahn(seed=seed, s=g["s"])
    assert abs(prob.alpha - g["alpha"]) <= 1e-12 * g["alpha"]
    o = _oracle_runs.ns_cached(prob.H, g["s"], g["alpha"], 5, 100, 1e-12, ons.TOL_ABS)
    assert o["steps"] == g["ns"]["steps"] and o["cert"] == 5

    def rerun(m):
        return ons.ns_reflector(prob.H, g["s"], g["alpha"], 5, m, 0.0, ons.TOL_ABS)

    Hg = torch.from_numpy(prob.H).to(_dev())
    for prec in (nsr.NS_PREC_FP64, nsr.NS_PREC_FP64_OZAKI):
        R, res = nsr.ns_reflector(Hg, g["s"], g["alpha"], 5, 100, 1e-12, 0, prec=prec)
        check_run(f"cfg2[seed={seed},prec={prec}]", R.cpu().numpy(), res, o, prob.d, 1e-12, rerun=rerun)


# --------------------------------------------------------------------------------------- configs[1]
@pytest.fixture(scope="module")
def cfg1_all():
    probs = workloads.cfg1_batched(seed=0, n_matrices=2048)
    assert len(probs) == 6144
    outs = _oracle_runs.cfg1_all(probs)
    return probs, outs


@pytest.mark.parametrize("prec_name", ["NS_PREC_FP64", "NS_PREC_FP64_OZAKI"])
def test_cfg1_all_problems_vs_oracle(nsr, cfg1_all, prec_name):
    """All 6144 configs[1] problems in one batched call (the launch configuration tools/bench_configs.py
    times), each against the oracle's NS run on the same input: steps, flags, certificate, full R,
    residual and trace (bounds in the module docstring); tie-band problems against the oracle's iterate
    at the GPU's step count and the closed form."""
    probs, outs = cfg1_all
    prec = getattr(nsr, prec_name)
    H = torch.from_numpy(np.stack([p_.H for p_ in probs])).to(_dev())
    R, res = nsr.ns_reflector_batched(H, [p_.s for p_ in probs], [p_.alpha for p_ in probs],
                                      [p_.k for p_ in probs], 100, 1e-12, prec=prec)
    Rn = R.cpu().numpy()
    del R, H
    torch.cuda.empty_cache()
    errs, ties, rdiff = [], 0, []
    for i, (p_, o) in enumerate(zip(probs, outs)):
        rec = _check_quiet(Rn[i], res[i], o, p_)
        errs.append(rec[0])
        ties += rec[1]
        rdiff.append(rec[2])
        if rec[1]:
            Rc = closed_form.reflector_explicit_q(p_.Q, p_.lam, p_.s)
            assert math.sqrt(np.sum((Rn[i] - Rc) ** 2) / p_.d) <= TOL_R, i
    _log(dict(test=f"cfg1_all[{prec_name}]", n=len(probs), max_err_frob_per_sqrt_d=float(np.max(errs)),
              median_err=float(np.median(errs)), tie_band_runs=ties, max_residual_diff=float(np.max(rdiff)),
              steps_total=int(sum(r_["steps"] for r_ in res))))
    assert np.max(errs) <= TOL_R


def _check_quiet(Rg, res, o, p_):
    """check_run without the per-problem log line (6144 problems): returns (err, in_tie_band, |dr|)."""
    d = p_.d
    assert np.array_equal(Rg, Rg.T)
    tie = _tie(o["hist_residual"], 1e-12, o["steps"])
    ref = o
    if res["steps"] != o["steps"]:
        assert tie and abs(res["steps"] - o["steps"]) == 1, (res["steps"], o["steps"])
        ref = ons.ns_reflector(p_.H, p_.s, p_.alpha, p_.k, res["steps"], 0.0, ons.TOL_ABS)
    else:
        assert res["flags"] == o["flags"], (res["flags"], o["flags"])
    assert res["cert"] == o["cert"] == p_.k
    dR = float(np.linalg.norm(Rg - ref["R"]))
    assert abs(res["residual"] - ref["residual"]) <= 2.0 * (1 + 1e-6) * dR + 64.0 * U * math.sqrt(d)
    assert abs(res["trace"] - ref["trace"]) <= math.sqrt(d) * dR + 8.0 * U * d
    return dR / math.sqrt(d), int(tie), abs(res["residual"] - ref["residual"])
