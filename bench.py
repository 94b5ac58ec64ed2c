#!/usr/bin/env python
"""bench.py -- Newton–Schulz prescribed-index reflector on B200 (BASELINE.json metric).

One "step" = one full ns_reflector call (the whole hot path: X_0, every square +
residual + decision + update, R) on BASELINE configs[3]: d = 16384, k = 1024, Q = 64
Householders, s = 0, alpha = 1.05, FP64, run to ||X^2 - I||_F/sqrt(d) < 1e-10 (reading
C3; 12 NS updates = 25 symmetric products).  value = algorithmic TFLOP/s =
(2*steps + 1) * d^3 / time (symmetric product count), summed over ranks.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--mode tol|fixed30]

N > 1 (torchrun): configs[3] does not shard ("replicas only"), so
every rank computes its own reflector; value = all ranks' flops / max-over-ranks time.
--sharded (opt-in): ONE reflector sharded over the N ranks (ns_reflector_sharded, exchange fused
into the product epilogue over CUDA-IPC peer memory), "scaling": "strong"; --d 49152 = configs[4].
--impl reference times the CPU oracle (oracle/ns.py) on a bounded sample of the same
workload (one NS step per bench step) on the host cores; rank 0 only.
"""
import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Newton–Schulz reflector TFLOP/s & time-to-R_k at d=16384 FP64 (frac of peak)"
# FP64 peak: measured DMMA.8x8x4 throughput on this pool's B200 (tools/calib/fp64_calib.cu,
# profiles/r01_calib_fp64.log: 36.97 TFLOP/s at 1965 MHz = 148 SM x 64 FMA/clk); clocks stay at
# max under FP64 load (no power cap), so burst == sustained.  MEASURED_PEAKS.json has no FP64 entry.
FP64_PEAK_TFLOPS = 36.97
FP64_PEAK_SOURCE = "measured: DMMA.8x8x4 microbenchmark, profiles/r01_calib_fp64.log (cuBLAS DGEMM 36.15)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", default="tol", choices=["tol", "fixed30"])
    ap.add_argument("--prec", default="fp64", choices=["fp64", "mixed", "ozaki"],
                    help="fp64: DMMA path (headline); mixed: BF16x3 tcgen05 -> re-anchor -> FP64 (configs[3] mixed); "
                         "ozaki: FP64 products emulated on the INT8 tensor cores")
    ap.add_argument("--no-mixed", action="store_true", help="skip the secondary mixed / Ozaki measurements")
    ap.add_argument("--d", type=int, default=16384)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--sharded", action="store_true",
                    help="strong scaling: ONE reflector sharded over all ranks (ns_reflector_sharded, peer-memory "
                         "exchange) instead of one replica per rank; with --d 49152 this is configs[4]")
    return ap.parse_args()


def workload(args):
    import workloads
    if args.d == 49152:
        p = workloads.cfg4_sharded(form=False)
        return p, ("configs[4]: d=49152 k=4096 Q=32 Householders, lambda in [-1,-0.02]u[0.02,1], s=0, alpha=1.05, FP64, "
                   "run-to-tol ||X^2-I||_F/sqrt(d)<1e-10")
    k = 1024 if args.d == 16384 else max(1, args.d // 16)
    p = workloads.cfg3_dense(d=args.d, k=k, form=False, mode=args.mode)
    desc = (f"configs[3]: d={p.d} k={p.k} Q=64 Householders, lambda in [-1,-0.05]u[0.05,1], s=0, alpha=1.05, FP64, "
            + ("run-to-tol ||X^2-I||_F/sqrt(d)<1e-10" if args.mode == "tol" else "30 fixed steps"))
    return p, desc


class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region (B200_PROFILING.md clocks line)."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "200", "-i", str(self.gpu)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, power, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
                power.append(float(parts[3]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(smax), "power_w_max": max(power),
                "samples": len(sm), "reasons": sorted(reasons)}


def dist_setup():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ---------------------------------------------------------------------------------- reference arm
def run_reference(args):
    ws, rank, _ = dist_setup()
    if rank != 0:
        return 0  # the oracle runs on rank 0's host cores only
    from oracle import ns as ons
    import workloads
    p, desc = workload(args)
    H = workloads.householder_form_fast(p.Vh, p.lam)
    d = p.d
    flops_step = 2.0 * d ** 3          # one NS step = 2 symmetric products (algorithmic count)
    for _ in range(args.warmup):
        ons.timed_ns_steps(H, p.s, p.alpha, 1)
    times = []
    threads = None
    for _ in range(args.steps):
        t, threads = ons.timed_ns_steps(H, p.s, p.alpha, 1)
        times.append(t)
    T = float(np.sum(times))
    value = flops_step * args.steps / T / 1e12
    sample = f"one oracle NS step (2 numpy FP64 products + update) on the d={d} configs[3] matrix per bench step"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * T / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": desc, "d": d, "k": p.k, "sample": sample, "parallelism": "host cores"},
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": threads, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    ws, rank, local = dist_setup()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        pg = dist
    import paper_2605_24840_b200 as nsr
    import workloads
    nsr.load_library()

    p, desc = workload(args)
    d = p.d
    H = workloads.householder_form_fast(p.Vh, p.lam, device=dev)
    R = torch.empty_like(H)
    wsbuf = nsr.alloc_workspace(nsr.ns_workspace_bytes(d), dev)
    stream = torch.cuda.current_stream(dev)

    prec = {"fp64": nsr.NS_PREC_FP64, "mixed": nsr.NS_PREC_MIXED_BF16X3, "ozaki": nsr.NS_PREC_FP64_OZAKI}[args.prec]
    if prec != nsr.NS_PREC_FP64:
        wsbuf = nsr.alloc_workspace(nsr.ns_workspace_bytes(d, prec), dev)
    comm = None
    if args.sharded:
        if prec != nsr.NS_PREC_FP64:
            raise SystemExit("--sharded runs the FP64 path")
        uid = [nsr.ns_comm_get_unique_id() if rank == 0 else None]
        if pg:
            pg.broadcast_object_list(uid, src=0)
        comm = nsr.ns_comm_init(rank, ws, uid[0])
        del wsbuf
        wsbuf = nsr.alloc_workspace(nsr.ns_workspace_bytes_sharded(d, ws), dev)

    def call(pr=None, options=None):
        pr = prec if pr is None else pr
        if comm is not None and pr == nsr.NS_PREC_FP64 and options is None:
            return nsr.ns_reflector_sharded(comm, H, p.s, p.alpha, p.k, p.max_steps, p.tol, p.tol_mode, R=R,
                                            ws=wsbuf, stream=stream)
        return nsr.ns_reflector(H, p.s, p.alpha, p.k, p.max_steps, p.tol, p.tol_mode, R=R, ws=wsbuf, stream=stream,
                                prec=pr, options=options)

    for _ in range(max(3, args.warmup)):
        _, res = call()
    torch.cuda.synchronize(dev)

    # ---- timed region: K full reflector computations, CUDA events on the launching stream
    sampler = ClockSampler(local)
    nsr.ns_profile_reset()
    nsr.ns_profile_enable(True)
    if pg:
        pg.barrier()
    torch.cuda.synchronize(dev)
    sampler.start()
    time.sleep(0.3)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    results = []
    for _ in range(args.steps):
        _, res = call()
        results.append(res)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    clocks = sampler.stop()
    nsr.ns_profile_enable(False)
    prof = nsr.ns_profile_get()
    ms = e0.elapsed_time(e1)
    if pg:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        ms = float(t.item())
        pg.barrier()
    steps_ns = results[-1]["steps"]
    flops_call = (2 * steps_ns + 1) * float(d) ** 3
    n_refl = 1 if args.sharded else ws          # reflectors computed per bench step by all ranks together
    value = n_refl * args.steps * flops_call / (ms * 1e-3) / 1e12
    launches = int(sum(r["launches"] for r in results))

    # ---- roofline of the dominant kernel (the symmetric product): algorithmic d^3 flops per launch
    n_prod = prof["n_square"] + prof["n_update"]
    avg_ms = (prof["ms_square"] + prof["ms_update"]) / max(1, n_prod)
    achieved = float(d) ** 3 / (avg_ms * 1e-3) / 1e12 if n_prod else None
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            tj = json.load(f)
        traffic = tj.get(str(d), {}).get("bytes_per_launch")
    roofline = {"bound": "tensor", "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": (achieved / FP64_PEAK_TFLOPS) if achieved else None, "traffic": traffic,
                "kernel": "ns_product_kernel (FP64 DMMA, symmetric 128x128 tiles)",
                "flops_per_launch": float(d) ** 3, "avg_launch_ms": avg_ms, "launches_timed": n_prod,
                "square_ms": prof["ms_square"] / max(1, prof["n_square"]),
                "update_ms": prof["ms_update"] / max(1, prof["n_update"]),
                "kernel_share_of_step": (prof["ms_square"] + prof["ms_update"]) / ms if ms else None,
                "peak_source": FP64_PEAK_SOURCE}

    # ---- end to end through the public host-buffer entry (H2D + D2H inside the timed region)
    e2e = None
    if not args.no_e2e and not args.sharded:
        Hh = H.cpu().pin_memory()
        Rh = torch.empty((d, d), dtype=torch.float64).pin_memory()
        wsh = wsbuf
        nsr.ns_reflector_host(Hh, p.s, p.alpha, p.k, p.max_steps, p.tol, p.tol_mode, R=Rh, ws=wsh, stream=stream,
                              prec=prec)
        if pg:
            pg.barrier()
        torch.cuda.synchronize(dev)
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(args.steps):
            _, rh = nsr.ns_reflector_host(Hh, p.s, p.alpha, p.k, p.max_steps, p.tol, p.tol_mode, R=Rh, ws=wsh,
                                          stream=stream, prec=prec)
        f1.record(stream)
        torch.cuda.synchronize(dev)
        ems = f0.elapsed_time(f1)
        if pg:
            t = torch.tensor([ems], dtype=torch.float64, device=dev)
            pg.all_reduce(t, op=pg.ReduceOp.MAX)
            ems = float(t.item())
        e2e = {"value": ws * args.steps * (2 * rh["steps"] + 1) * float(d) ** 3 / (ems * 1e-3) / 1e12,
               "unit": "TFLOP/s", "h2d_bytes_per_step": d * d * 8, "d2h_bytes_per_step": d * d * 8,
               "ms_per_step": ems / args.steps, "entry": "ns_reflector_host (pinned host H, R)"}
        del Hh, Rh

    # ---- secondary: the same reflector through the mixed BF16x3 -> re-anchor -> FP64 mode and the
    # Ozaki-split FP64 emulation on the INT8 tensor cores (same metric, FP64-equivalent algorithmic flops)
    mixed = ozaki = None

    def secondary(pr, options=None):
        nonlocal wsbuf
        wsbuf = nsr.alloc_workspace(nsr.ns_workspace_bytes(d, pr), dev)
        _, rm = call(pr, options)
        torch.cuda.synchronize(dev)
        g0 = torch.cuda.Event(enable_timing=True)
        g1 = torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for _ in range(args.steps):
            _, rm = call(pr, options)
        g1.record(stream)
        torch.cuda.synchronize(dev)
        mms = g0.elapsed_time(g1) / args.steps
        return {"time_to_R_ms": mms, "value": (2 * rm["steps"] + 1) * float(d) ** 3 / (mms * 1e-3) / 1e12,
                "unit": "TFLOP/s (FP64-equivalent algorithmic)", "steps": rm["steps"], "switch_step": rm["switch_step"],
                "pre_polish_residual": rm["pre_polish_residual"], "cert": rm["cert"], "flags": rm["flags"],
                "speedup_vs_fp64": (ms / args.steps) / mms, "launches": rm["launches"]}

    mixed_oz = None
    if args.prec == "fp64" and not args.no_mixed and not args.sharded:
        mixed = secondary(nsr.NS_PREC_MIXED_BF16X3)
        # mixed_mode: the default (re-anchor products on the Ozaki INT8 cores, FP64 DMMA polishing steps);
        # the same mixed path with the polishing steps on the Ozaki INT8 products as well
        mixed_oz = secondary(nsr.NS_PREC_MIXED_BF16X3, nsr.ns_options(polish=1))
        if d <= 65536:
            ozaki = secondary(nsr.NS_PREC_FP64_OZAKI)

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline and not args.sharded:
        from oracle import ns as ons
        Hc = H.cpu().numpy()
        t, threads = ons.timed_ns_steps(Hc, p.s, p.alpha, 1)
        cpu = {"value": 2.0 * float(d) ** 3 / t / 1e12, "unit": "TFLOP/s", "cores": threads, "kind": "oracle",
               "sample": f"one oracle NS step (2 numpy FP64 products + update) on the same d={d} matrix, {t:.1f} s",
               "seconds": t}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if args.sharded else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": desc, "d": d, "k": p.k, "ns_steps": steps_ns, "products": 2 * steps_ns + 1,
                       "algorithmic_flops_per_reflector": flops_call, "l2": "inputs larger than L2 (3 x 2 GiB FP64 "
                       "matrices per step vs 126 MB L2)",
                       "parallelism": (f"sharded x{ws} (peer-memory exchange)" if args.sharded
                                       else (f"replicas x{ws}" if ws > 1 else "single")),
                       "frac_of_fp64_peak": value / ws / FP64_PEAK_TFLOPS},
            "time_to_R_ms": ms / args.steps, "reflectors_per_s": n_refl * args.steps / (ms * 1e-3),
            "result": {"steps": steps_ns, "cert": results[-1]["cert"], "flags": results[-1]["flags"],
                       "residual": results[-1]["residual"]},
            "gpu_launches": launches, "clocks": clocks, "roofline": roofline, "e2e": e2e, "cpu_baseline": cpu,
            "mixed_mode": mixed, "mixed_ozaki_polish_mode": mixed_oz, "ozaki_mode": ozaki, "precision": args.prec,
        }
        print(json.dumps(line), flush=True)
    if comm is not None:
        nsr.ns_comm_destroy(comm)
    if pg:
        pg.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
