"""configs[1] batch, every problem run for exactly 16 steps (tol = 0): 17 + 16 full-size product launches."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_24840_b200 as nsr  # noqa: E402
import workloads  # noqa: E402
probs = workloads.cfg1_batched(seed=0, n_matrices=2048)
H = torch.stack([torch.from_numpy(p.H) for p in probs]).cuda()
s_, a_, k_ = [p.s for p in probs], [p.alpha for p in probs], [p.k for p in probs]
ws = nsr.alloc_workspace(nsr.ns_workspace_bytes_batched(256, len(probs), 0), H.device)
R = torch.empty_like(H)
nsr.ns_reflector_batched(H, s_, a_, k_, 16, 0.0, R=R, ws=ws)
nsr.ns_profile_enable(True)
nsr.ns_profile_reset()
nsr.ns_reflector_batched(H, s_, a_, k_, 16, 0.0, R=R, ws=ws)
torch.cuda.synchronize()
pr = nsr.ns_profile_get()
print(os.environ.get("TAG", ""), "square ms/launch %.4f  update ms/launch %.4f" % (pr["ms_square"] / pr["n_square"], pr["ms_update"] / pr["n_update"]), pr["n_square"], pr["n_update"])
