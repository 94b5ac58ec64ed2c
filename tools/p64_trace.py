"""configs[1] (6144 batched d=256 problems) timing, and -- with a -DNS_P64_TRACE=1 build -- the per-CTA phase
timeline of the 64x64-tile product kernel: how much of each SM's time some co-resident CTA spends in its
K loop, prologue (start -> first stage landed) and epilogue (K loop done -> end).

    python tools/p64_trace.py [lib.so] [--trace] [--reps 5]
"""
import argparse
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2605_24840_b200 as nsr  # noqa: E402
import workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("lib", nargs="?", default=None)
ap.add_argument("--trace", action="store_true")
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--n", type=int, default=2048)
ap.add_argument("--fixed", type=int, default=0, help="run every problem for exactly this many steps (tol = 0)")
a = ap.parse_args()
if a.lib:
    nsr.load_library(os.path.abspath(a.lib))
lib = nsr.load_library()

probs = workloads.cfg1_batched(seed=0, n_matrices=2048, count=a.n)
H = torch.from_numpy(np.stack([p.H for p in probs])).cuda()
ws = nsr.alloc_workspace(nsr.ns_workspace_bytes_batched(256, len(probs), 0), H.device)
R = torch.empty_like(H)
s_, a_, k_ = [p.s for p in probs], [p.alpha for p in probs], [p.k for p in probs]
run = lambda: nsr.ns_reflector_batched(H, s_, a_, k_, a.fixed or 100, 0.0 if a.fixed else 1e-12, R=R, ws=ws)  # noqa: E731
run()
torch.cuda.synchronize()
ts = []
for _ in range(a.reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _, outs = run()
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
steps = sum(o["steps"] for o in outs)
flops = sum(2 * o["steps"] + 1 for o in outs) * 256.0 ** 3
import hashlib  # noqa: E402
rhash = hashlib.md5(R.cpu().numpy().tobytes()).hexdigest()[:12]
print(f"R md5 {rhash}")
print(f"cfg1 {len(probs)} problems: median {np.median(ts):.2f} ms (min {min(ts):.2f}), steps {steps}, "
      f"{flops / (np.median(ts) * 1e-3) / 1e12:.2f} TFLOP/s algorithmic; all: {[round(t, 2) for t in ts]}")

if a.trace:
    import ctypes
    cap = 3_000_000
    buf = torch.zeros(1 + 10 * cap, dtype=torch.int64, device="cuda")
    lib.ns_debug_p64_trace.restype = ctypes.c_int
    lib.ns_debug_p64_trace.argtypes = [ctypes.c_void_p, ctypes.c_ulonglong]
    rc = lib.ns_debug_p64_trace(ctypes.c_void_p(buf.data_ptr()), cap)
    if rc != 0:
        sys.exit(f"trace unavailable (rc {rc}): build with -DNS_P64_TRACE=1")
    run()
    torch.cuda.synchronize()
    lib.ns_debug_p64_trace(None, 0)
    n = min(int(buf[0].item()), cap)
    rec = buf[1:1 + 10 * n].view(n, 10).cpu().numpy().astype(np.uint64)
    sm = (rec[:, 0] & 0xffff).astype(np.int64)
    mode = ((rec[:, 0] >> 16) & 1).astype(np.int64)
    diag = ((rec[:, 0] >> 17) & 1).astype(np.int64)
    t0, t1, t3 = (rec[:, i].astype(np.int64) for i in (1, 2, 3))
    we = rec[:, 5:9].astype(np.int64)
    base = t0.min()
    t0, t1, t3, we = t0 - base, t1 - base, t3 - base, we - base
    t2 = we.max(1)                      # the CTA's K loop ends with its last warp
    t2f = we.min(1)
    tst = rec[:, 9].astype(np.int64) - base   # last warp's epilogue stores issued
    print(f"{n} CTAs traced; span {(t3.max()) / 1e6:.2f} ms")
    for m in (0, 1):
        for dg in (0, 1):
            k = (mode == m) & (diag == dg)
            if k.any():
                print(f"  mode {m} diag {dg}: n={k.sum():7d}  prologue {np.median(t1[k] - t0[k]) / 1e3:6.2f} us  "
                      f"K loop (first..last warp) {np.median(t2f[k] - t1[k]) / 1e3:6.2f}..{np.median(t2[k] - t1[k]) / 1e3:6.2f} us  "
                      f"epilogue {np.median(t3[k] - t2[k]) / 1e3:6.2f} us (stores issued +{np.median(tst[k] - t2[k]) / 1e3:5.2f})  total {np.median(t3[k] - t0[k]) / 1e3:6.2f} us; "
                      f"warp w ends last: {np.bincount(np.argmax(we[k], 1), minlength=4) / k.sum()}")
    # per SM: fraction of the busy span in which >= 1 CTA is inside its K loop
    res = [], []
    hist = np.zeros(8)
    for s in np.unique(sm):
        k = sm == s
        ev = np.concatenate([np.stack([t1[k], np.ones(k.sum())], 1), np.stack([t2[k], -np.ones(k.sum())], 1)])
        ev = ev[np.argsort(ev[:, 0], kind="stable")]
        cnt, last, inloop = 0, ev[0, 0], 0.0
        for t, dlt in ev:
            if cnt > 0:
                inloop += t - last
            hist[min(int(cnt), 7)] += t - last
            cnt += dlt
            last = t
        span = t3[k].max() - t0[k].min()
        occ = np.sum(t3[k] - t0[k]) / span
        res[0].append(inloop / span)
        res[1].append(occ)
    print(f"  per SM: some CTA in its K loop {100 * np.mean(res[0]):.1f}% of the SM's span "
          f"(min {100 * np.min(res[0]):.1f}%); mean resident CTAs {np.mean(res[1]):.2f}")
    hist /= hist.sum()
    print("  time share with n CTAs in their K loop: " + ", ".join(f"n={i}: {100 * h:.1f}%" for i, h in enumerate(hist) if h > 0.0005))
