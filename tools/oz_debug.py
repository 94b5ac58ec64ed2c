import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2605_24840_b200 as nsr, workloads
from oracle import ns as ons
for d,k in [(64,3),(128,8),(256,16),(1024,64)]:
    p = workloads.cfg0_controlled(seed=0, d=d, k=k) if d < 1024 else workloads.cfg3_dense(d=1024, k=64)
    H = torch.from_numpy(p.H).cuda()
    for m in range(0, 12):
        R1, r1 = nsr.ns_reflector(H, p.s, p.alpha, p.k, m, 0.0, p.tol_mode, prec=nsr.NS_PREC_FP64_OZAKI)
        R0, r0 = nsr.ns_reflector(H, p.s, p.alpha, p.k, m, 0.0, p.tol_mode)
        print(d, m, r1["residual"], r0["residual"], float((R1-R0).abs().max()), r1["trace"], r0["trace"])
