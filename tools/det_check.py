import sys, torch, numpy as np
sys.path.insert(0, ".")
import paper_2605_24840_b200 as nsr, workloads
probs = workloads.cfg1_batched(seed=0, n_matrices=2048, count=2048)
H = torch.stack([torch.from_numpy(p.H) for p in probs]).cuda()
s_ = [p.s for p in probs]; a_ = [p.alpha for p in probs]; k_ = [p.k for p in probs]
ws = nsr.alloc_workspace(nsr.ns_workspace_bytes_batched(256, len(probs)), H.device)
R1, o1 = nsr.ns_reflector_batched(H, s_, a_, k_, 100, 1e-12, ws=ws)
R1 = R1.clone()
R2, o2 = nsr.ns_reflector_batched(H, s_, a_, k_, 100, 1e-12, ws=ws)
print("bitwise equal:", torch.equal(R1, R2), "steps equal:", [a["steps"] for a in o1] == [b["steps"] for b in o2])
st = np.array([a["steps"] for a in o1])
print("steps sum", st.sum())
from oracle import scalar
pred = np.array([scalar.predict_run((p.lam - p.s) / p.alpha, 100, 1e-12, False)[0] for p in probs])
bad = np.nonzero(st != pred)[0]
print("off:", bad, st[bad], pred[bad], [o1[i]["residual"] for i in bad])
