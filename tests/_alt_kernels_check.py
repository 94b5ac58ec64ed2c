"""Subprocess body for test_alternative_kernels (the kernel-selection knobs are read once per process):
run a few products / reflectors on the alternative kernels and print one JSON line of errors."""
import json
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_24840_b200 as nsr  # noqa: E402
import workloads  # noqa: E402
from oracle import ns as ons, checks  # noqa: E402

out = {}
rng = np.random.default_rng(7)
for d, mode in ((300, 0), (515, 1), (384, 2)):
    A = rng.standard_normal((d, d))
    A = 0.5 * (A + A.T) / math.sqrt(d)
    B = A @ A if mode != 2 else 0.5 * (lambda M: M + M.T)(rng.standard_normal((d, d)))
    ref = A @ B if mode != 1 else 1.5 * A - 0.5 * (A @ B)
    Ag, Bg = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    C = nsr.ns_symm_product(Ag, Bg, mode=mode, prec=nsr.NS_PREC_MIXED_BF16X3).cpu().numpy()
    out[f"mixed_{d}_{mode}"] = float(np.max(np.abs(C - ref)) / (np.max(np.abs(A)) * np.max(np.abs(B)) * d))
for d, k in ((1024, 64), (2048, 128)):
    p = workloads.cfg3_dense(d=d, k=k)
    o = ons.ns_reflector(p.H, p.s, p.alpha, p.k, p.max_steps, p.tol, p.tol_mode)
    R, res = nsr.ns_reflector(torch.from_numpy(p.H).cuda(), p.s, p.alpha, p.k, p.max_steps, p.tol, p.tol_mode)
    out[f"fp64_{d}"] = [checks.frob_per_sqrt_d(R.cpu().numpy(), o["R"]), res["steps"] == o["steps"]]
if os.environ.get("NS_SHARD_P2P") == "0":
    # the NCCL all-gather exchange of the sharded path on a one-rank communicator: = single path bitwise
    p = workloads.cfg3_dense(d=2048, k=128)
    Hg = torch.from_numpy(p.H).cuda()
    c = nsr.ns_comm_init(0, 1, nsr.ns_comm_get_unique_id())
    Rs, rs = nsr.ns_reflector_sharded(c, Hg, p.s, p.alpha, p.k, p.max_steps, p.tol, p.tol_mode)
    nsr.ns_comm_destroy(c)
    Rd, rd = nsr.ns_reflector(Hg, p.s, p.alpha, p.k, p.max_steps, p.tol, p.tol_mode)
    out["fp64_sharded_nccl"] = [0.0 if torch.equal(Rs, Rd) else 1.0, rs["steps"] == rd["steps"]]
print(json.dumps(out))
