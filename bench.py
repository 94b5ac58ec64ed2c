#!/usr/bin/env python
"""bench.py -- Newton–Schulz prescribed-index reflector on B200 (BASELINE.json metric).

One "step" = one full ns_reflector call (the whole hot path: X_0, every square +
residual + decision + update, R) on BASELINE configs[3]: d = 16384, k = 1024, Q = 64
Householders, s = 0, alpha = 1.05, FP64, run to ||X^2 - I||_F/sqrt(d) < 1e-10 (reading
C3; 12 NS updates = 25 symmetric products).  value = algorithmic TFLOP/s =
(2*steps + 1) * d^3 / time (symmetric product count), summed over ranks.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--mode tol|fixed30]

N > 1 (torchrun): ONE reflector sharded over the N ranks (strong scaling, "scaling": "strong"):
ns_reflector_sharded_rows, each rank holding only its block-row panel of H and receiving the same
rows of R; every rank computes 1/N of the upper 128x128 tiles of each symmetric product and its
product kernel's epilogue stores them into all ranks' buffers over NVLink (CUDA-IPC peer memory),
so N = 1 is the BENCH workload and N > 1 measures north_star's strong-scaling target on configs[3];
--d 49152 runs configs[4] (the sharded large-d case).  value = the one reflector's algorithmic
flops / max-over-ranks time.  --replicas: the old weak-scaling mode (one independent configs[3]
reflector per rank).
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
# B200 datasheet FP64 / FP64-tensor figure (NVIDIA HGX B200 specification, per GPU; not in B200_PROFILING.md,
# whose table lists no FP64 entry): reported as a second denominator next to the measured one.
FP64_DATASHEET_TFLOPS = 40.0


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
                    help="force the sharded rows entry also at N = 1 (N > 1 always runs it unless --replicas)")
    ap.add_argument("--per-config", action="store_true",
                    help="with --impl reference: time the CPU oracle on every BASELINE config (one JSON line each; "
                         "cfg0/cfg1/cfg2 NS in full, cfg3 one step extrapolated, cfg4 extrapolated and flagged, "
                         "Jacobi and closed-form verification timed separately)")
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: one independent reflector per rank (weak scaling) instead of one sharded reflector")
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
def _oracle_cfg1_worker(args):
    from oracle import ns as ons
    H, s, alpha, k = args
    return ons.ns_reflector(H, s, alpha, k, 100, 1e-12, ons.TOL_ABS)["steps"]


def run_reference_per_config(args):
    """The CPU oracle (numpy/OpenBLAS FP64 products: a "library CPU" number; plain-C cyclic Jacobi) timed on
    every BASELINE config on this host, one JSON line each -- reported next to the GPU numbers, not targeted."""
    import multiprocessing as mp
    from oracle import closed_form, jacobi, ns as ons
    import workloads
    cpu = _cpu_model()
    threads = int(os.environ.get("OPENBLAS_NUM_THREADS", os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1)))

    def emit(rec):
        rec.update({"impl": "reference", "kind": "oracle (numpy/OpenBLAS FP64 products; library CPU)", "cpu": cpu})
        print(json.dumps(rec), flush=True)

    # configs[0]: 5 seeds, full NS run each
    ts = []
    for seed in range(5):
        p = workloads.cfg0_controlled(seed)
        t0 = time.perf_counter()
        o = ons.ns_reflector(p.H, p.s, p.alpha, p.k, 100, 1e-12, 0)
        ts.append(time.perf_counter() - t0)
    emit({"config": "cfg0", "what": "NS run to 1e-12, 5 seeds", "ms_median": 1e3 * float(np.median(ts)),
          "steps": o["steps"], "cores": threads})
    # configs[1]: all 6144 problems, one process per core (single-threaded BLAS each)
    probs = workloads.cfg1_batched(seed=0, n_matrices=2048)
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    t0 = time.perf_counter()
    with mp.get_context("spawn").Pool(os.cpu_count()) as pool:
        steps = pool.map(_oracle_cfg1_worker, [(q.H, q.s, q.alpha, q.k) for q in probs], chunksize=16)
    t1 = time.perf_counter() - t0
    emit({"config": "cfg1", "what": "NS on all 6144 problems (process pool)", "seconds": t1,
          "reflectors_per_s": len(probs) / t1, "steps_total": int(sum(steps)), "cores": os.cpu_count(),
          "tflops": float(np.sum(2 * np.array(steps) + 1)) * 256.0 ** 3 / t1 / 1e12})
    del os.environ["OPENBLAS_NUM_THREADS"]
    t0 = time.perf_counter()
    for q in probs[:24:3]:
        jacobi.jacobi_eigh(q.H)
    tj = (time.perf_counter() - t0) / 8
    emit({"config": "cfg1", "what": "cyclic Jacobi (plain C, OpenMP) per d=256 matrix, 8 sampled; x2048 extrapolated",
          "seconds_per_matrix": tj, "seconds_2048_extrapolated": 2048 * tj, "extrapolated": True, "cores": threads})
    # configs[2]: seed 0 NS in full (s, alpha from the oracle's Jacobi, tests/golden)
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "cfg2_seed0.json")))
    prob = workloads.cfg2_allen_cahn(seed=0, s=g["s"])
    t0 = time.perf_counter()
    o = ons.ns_reflector(prob.H, g["s"], g["alpha"], 5, 100, 1e-12, 0)
    t2 = time.perf_counter() - t0
    emit({"config": "cfg2", "what": "NS run, seed 0 (d=4096)", "seconds": t2, "steps": o["steps"], "cores": threads,
          "tflops": (2 * o["steps"] + 1) * 4096.0 ** 3 / t2 / 1e12})
    emit({"config": "cfg2", "what": "cyclic Jacobi d=4096 (the shift's source), recorded by tools/make_golden_cfg2.py",
          "seconds": g["seconds"]["jacobi"], "threads": g.get("threads"), "recorded_not_rerun": True,
          "where": "the build container's CPU (not this host)"})
    # configs[3]: one NS step, extrapolated to the 12-step run and the 30-step fixed run
    p = workloads.cfg3_dense(form=False)
    H = workloads.householder_form_fast(p.Vh, p.lam)
    t, thr = ons.timed_ns_steps(H, p.s, p.alpha, 1)
    emit({"config": "cfg3", "what": "one NS step (2 products + update), d=16384", "seconds": t, "cores": thr,
          "tflops": 2.0 * 16384.0 ** 3 / t / 1e12, "seconds_run_to_tol_extrapolated": 12.5 * t,
          "seconds_fixed30_extrapolated": 30.5 * t, "extrapolated": True})
    t0 = time.perf_counter()
    closed_form.householder_reflector_columns(p.Vh, p.lam, 0.0, np.arange(0, 16384, 256))
    emit({"config": "cfg3", "what": "closed-form verification: 64 columns of Q sgn(Lambda) Q^T (64 Householders)",
          "seconds": time.perf_counter() - t0, "cores": threads})
    # configs[4]: extrapolated (d ratio 3: 27x per product; 29 products vs 25)
    emit({"config": "cfg4", "what": "NS run d=49152, extrapolated from the cfg3 step: 27 x per product, 29 products",
          "seconds_extrapolated": 27.0 * 14.5 * t, "extrapolated": True, "cores": thr})
    return 0


def run_reference(args):
    ws, rank, _ = dist_setup()
    if rank != 0:
        return 0  # the oracle runs on rank 0's host cores only
    if args.per_config:
        return run_reference_per_config(args)
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
def _timed(call, stream, steps, dev, pg):
    """K calls between CUDA events on the launching stream; barrier + synchronize on both sides; max over ranks."""
    import torch
    if pg:
        pg.barrier()
    torch.cuda.synchronize(dev)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    out = [call() for _ in range(steps)]
    e1.record(stream)
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1)
    if pg:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        ms = float(t.item())
        pg.barrier()
    return ms, out


def run_ours(args):
    import torch
    ws, rank, local = dist_setup()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    sharded = (ws > 1 and not args.replicas) or args.sharded
    if ws > 1:
        import torch.distributed as dist
        # communicator lines (NCCL INIT: nranks, NVLS / P2P transports) on stderr, so stdout keeps one JSON line
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        dist.init_process_group("nccl", device_id=dev)
        pg = dist
    import paper_2605_24840_b200 as nsr
    import workloads
    nsr.load_library()

    p, desc = workload(args)
    d = p.d
    H = workloads.householder_form_fast(p.Vh, p.lam, device=dev)
    stream = torch.cuda.current_stream(dev)
    prec = {"fp64": nsr.NS_PREC_FP64, "mixed": nsr.NS_PREC_MIXED_BF16X3, "ozaki": nsr.NS_PREC_FP64_OZAKI}[args.prec]

    comm = None
    if sharded:
        if prec != nsr.NS_PREC_FP64:
            raise SystemExit("the sharded path runs FP64")
        if d % ws:
            raise SystemExit(f"d = {d} is not divisible by the {ws} ranks")
        uid = [nsr.ns_comm_get_unique_id() if rank == 0 else None]
        if pg:
            pg.broadcast_object_list(uid, src=0)
        comm = nsr.ns_comm_init(rank, ws, uid[0])
        r0, r1 = nsr.ns_shard_rows(d, ws, rank)
        H_rows = H[r0:r1].clone()          # this rank's block-row panel of H: the only H it keeps
        del H
        torch.cuda.empty_cache()
        H = None
        R_rows = torch.empty_like(H_rows)
        wsbuf = nsr.alloc_workspace(nsr.ns_workspace_bytes_sharded(d, ws), dev)
    else:
        R = torch.empty_like(H)
        wsbuf = nsr.alloc_workspace(nsr.ns_workspace_bytes(d, prec), dev)

    def call(pr=None, options=None):
        pr = prec if pr is None else pr
        if comm is not None:
            return nsr.ns_reflector_sharded_rows(comm, H_rows, d, p.s, p.alpha, p.k, p.max_steps, p.tol, p.tol_mode,
                                                 R_rows=R_rows, ws=wsbuf, stream=stream, nranks=ws)
        return nsr.ns_reflector(H, p.s, p.alpha, p.k, p.max_steps, p.tol, p.tol_mode, R=R, ws=wsbuf, stream=stream,
                                prec=pr, options=options)

    for _ in range(max(3, args.warmup)):
        _, res = call()
    torch.cuda.synchronize(dev)

    # ---- timed region: K full reflector computations, CUDA events on the launching stream
    sampler = ClockSampler(local)
    nsr.ns_profile_reset()
    nsr.ns_profile_enable(True)
    sampler.start()
    time.sleep(0.3)
    ms, outs = _timed(call, stream, args.steps, dev, pg)
    results = [o[1] for o in outs]
    clocks = sampler.stop()
    nsr.ns_profile_enable(False)
    prof = nsr.ns_profile_get()
    steps_ns = results[-1]["steps"]
    flops_call = (2 * steps_ns + 1) * float(d) ** 3
    n_refl = 1 if sharded else ws          # reflectors computed per bench step by all ranks together
    value = n_refl * args.steps * flops_call / (ms * 1e-3) / 1e12
    launches = int(sum(r["launches"] for r in results))

    # ---- roofline of the dominant kernel (the symmetric product): algorithmic d^3 flops per launch, or its
    # 1/N share of the tiles on the sharded path (the kernel time excludes the barrier)
    n_prod = prof["n_square"] + prof["n_update"]
    avg_ms = (prof["ms_square"] + prof["ms_update"]) / max(1, n_prod)
    share = 1.0 / ws if sharded else 1.0
    achieved = share * float(d) ** 3 / (avg_ms * 1e-3) / 1e12 if n_prod else None
    if pg and achieved is not None:   # report the slowest rank's kernel
        t = torch.tensor([avg_ms], dtype=torch.float64, device=dev)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        avg_ms = float(t.item())
        achieved = share * float(d) ** 3 / (avg_ms * 1e-3) / 1e12
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath) and not sharded:
        with open(tpath) as f:
            tj = json.load(f)
        traffic = tj.get(str(d), {}).get("bytes_per_launch")
    roofline = {"bound": "tensor", "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": (achieved / FP64_PEAK_TFLOPS) if achieved else None, "traffic": traffic,
                "kernel": "ns_product_kernel (FP64 DMMA, symmetric 128x128 tiles"
                          + (f", 1/{ws} of the tiles per rank, peer-store epilogue)" if sharded else ")"),
                "flops_per_launch": share * float(d) ** 3, "avg_launch_ms": avg_ms, "launches_timed": n_prod,
                "square_ms": prof["ms_square"] / max(1, prof["n_square"]),
                "update_ms": prof["ms_update"] / max(1, prof["n_update"]),
                "kernel_share_of_step": (prof["ms_square"] + prof["ms_update"]) / ms if ms else None,
                "peak_source": FP64_PEAK_SOURCE,
                "frac_of_datasheet_fp64": (achieved / FP64_DATASHEET_TFLOPS) if achieved else None,
                "datasheet_fp64_tflops": FP64_DATASHEET_TFLOPS}

    # ---- end to end through the public entry with HOST buffers (H2D of the inputs and D2H of the result
    # inside the timed region)
    e2e = None
    if not args.no_e2e:
        if sharded:
            Hh = H_rows.cpu().pin_memory()
            Rh = torch.empty(tuple(H_rows.shape), dtype=torch.float64).pin_memory()

            def e2e_call():
                H_rows.copy_(Hh, non_blocking=True)
                out = call()
                Rh.copy_(R_rows, non_blocking=True)
                return out
            e2e_call()
            ems, eo = _timed(e2e_call, stream, args.steps, dev, pg)
            rh = eo[-1][1]
            e2e = {"value": args.steps * (2 * rh["steps"] + 1) * float(d) ** 3 / (ems * 1e-3) / 1e12,
                   "unit": "TFLOP/s", "h2d_bytes_per_step": d * d * 8, "d2h_bytes_per_step": d * d * 8,
                   "ms_per_step": ems / args.steps,
                   "entry": f"ns_reflector_sharded_rows with pinned host panels (each rank copies its {d // ws} "
                            f"rows of H in and of R out; bytes summed over ranks)"}
        else:
            Hh = H.cpu().pin_memory()
            Rh = torch.empty((d, d), dtype=torch.float64).pin_memory()
            nsr.ns_reflector_host(Hh, p.s, p.alpha, p.k, p.max_steps, p.tol, p.tol_mode, R=Rh, ws=wsbuf,
                                  stream=stream, prec=prec)
            ems, eo = _timed(lambda: nsr.ns_reflector_host(Hh, p.s, p.alpha, p.k, p.max_steps, p.tol, p.tol_mode,
                                                           R=Rh, ws=wsbuf, stream=stream, prec=prec),
                             stream, args.steps, dev, pg)
            rh = eo[-1][1]
            e2e = {"value": ws * args.steps * (2 * rh["steps"] + 1) * float(d) ** 3 / (ems * 1e-3) / 1e12,
                   "unit": "TFLOP/s", "h2d_bytes_per_step": ws * d * d * 8, "d2h_bytes_per_step": ws * d * d * 8,
                   "ms_per_step": ems / args.steps, "entry": "ns_reflector_host (pinned host H, R)"}
        del Hh, Rh

    # ---- secondary: the same reflector through the mixed BF16x3 -> re-anchor -> FP64 mode and the
    # Ozaki-split FP64 emulation on the INT8 tensor cores (same metric, FP64-equivalent algorithmic flops)
    mixed = ozaki = mixed_oz = None

    def secondary(pr, options=None):
        nonlocal wsbuf
        wsbuf = nsr.alloc_workspace(nsr.ns_workspace_bytes(d, pr), dev)
        call(pr, options)
        nsr.ns_profile_reset()
        nsr.ns_profile_enable(True)
        mms, mo = _timed(lambda: call(pr, options), stream, args.steps, dev, pg)
        nsr.ns_profile_enable(False)
        pf = nsr.ns_profile_get()
        rm = mo[-1][1]
        mms /= args.steps
        out = {"time_to_R_ms": mms, "value": (2 * rm["steps"] + 1) * float(d) ** 3 / (mms * 1e-3) / 1e12,
               "unit": "TFLOP/s (FP64-equivalent algorithmic)", "steps": rm["steps"], "switch_step": rm["switch_step"],
               "pre_polish_residual": rm["pre_polish_residual"], "cert": rm["cert"], "flags": rm["flags"],
               "speedup_vs_fp64": (ms / args.steps) / mms, "launches": rm["launches"]}
        out["executed_roofline"] = executed_roofline(pf, args.steps)
        return out

    if args.prec == "fp64" and not args.no_mixed and not sharded:
        mixed = secondary(nsr.NS_PREC_MIXED_BF16X3)
        # mixed_mode: the default (re-anchor products on the Ozaki INT8 cores, FP64 DMMA polishing steps);
        # the same mixed path with the polishing steps on the Ozaki INT8 products as well
        mixed_oz = secondary(nsr.NS_PREC_MIXED_BF16X3, nsr.ns_options(polish=1))
        if d <= 65536:
            ozaki = secondary(nsr.NS_PREC_FP64_OZAKI)

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline and not sharded:
        from oracle import ns as ons
        Hc = H.cpu().numpy()
        t, threads = ons.timed_ns_steps(Hc, p.s, p.alpha, 1)
        cpu = {"value": 2.0 * float(d) ** 3 / t / 1e12, "unit": "TFLOP/s", "cores": threads, "kind": "oracle",
               "sample": f"one oracle NS step (2 numpy/OpenBLAS FP64 products + update: a library-CPU number) on "
                         f"the same d={d} matrix, {t:.1f} s; {_cpu_model()}",
               "seconds": t}

    if rank == 0:
        nvlink = None
        if sharded and ws > 1:
            n_tiles = (-(-d // 128)) * (-(-d // 128) + 1) // 2
            n_my = -(-n_tiles // ws)
            per_product = n_my * 128 * 128 * 8 * (ws - 1)          # upper tiles only (receivers mirror)
            nvlink = {"bytes_out_per_rank_per_step": 2 * per_product,
                      "bytes_out_per_rank_per_reflector": (2 * steps_ns + 1) * per_product,
                      "note": "peer stores of each rank's upper tiles into the other ranks (receiver-side mirror)"}
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if sharded else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": desc, "d": d, "k": p.k, "ns_steps": steps_ns, "products": 2 * steps_ns + 1,
                       "algorithmic_flops_per_reflector": flops_call, "l2": "inputs larger than L2 (3 x 2 GiB FP64 "
                       "matrices per step vs 126 MB L2)",
                       "parallelism": (f"sharded x{ws} (block-row panels, upper tiles split, peer-memory exchange)"
                                       if sharded else (f"replicas x{ws}" if ws > 1 else "single")),
                       "frac_of_fp64_peak": value / ws / FP64_PEAK_TFLOPS,
                       "frac_of_datasheet_fp64": value / ws / FP64_DATASHEET_TFLOPS},
            "time_to_R_ms": ms / args.steps, "reflectors_per_s": n_refl * args.steps / (ms * 1e-3),
            "result": {"steps": steps_ns, "cert": results[-1]["cert"], "flags": results[-1]["flags"],
                       "residual": results[-1]["residual"]},
            "gpu_launches": launches, "clocks": clocks, "roofline": roofline, "e2e": e2e, "cpu_baseline": cpu,
            "nvlink": nvlink,
            "mixed_mode": mixed, "mixed_ozaki_polish_mode": mixed_oz, "ozaki_mode": ozaki, "precision": args.prec,
        }
        print(json.dumps(line), flush=True)
    if comm is not None:
        nsr.ns_comm_destroy(comm)
    if pg:
        pg.destroy_process_group()
    return 0


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return "CPU: " + ln.split(":", 1)[1].strip() + f", {os.cpu_count()} logical cores"
    except OSError:
        pass
    return f"{os.cpu_count()} logical cores"


def executed_roofline(pf, steps):
    """Roofline of the secondaries' tensor-core work in the arithmetic they EXECUTE (not FP64-equivalent):
    BF16 flops of the split products against MEASURED_PEAKS.json's bf16 figure, INT8 ops of the Ozaki digit
    products against the bf16 figure x 2 (the guide's nominal int8/fp8 : bf16 ratio, 4.5 : 2.25)."""
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mp = json.load(f)
        peaks = {"bf16": mp.get("bf16_tflops_sustained") or mp.get("bf16_tflops"), "bf16_burst": mp.get("bf16_tflops")}
    except (OSError, ValueError):
        peaks = {"bf16": None, "bf16_burst": None}
    out = {}
    if pf.get("n_lowp"):
        a = pf["lowp_flops"] / (pf["ms_lowp"] * 1e-3) / 1e12
        out["bf16"] = {"kernel": "ns_mx2_product_kernel (BF16x3 split, tcgen05 cta_group::2)", "launches": pf["n_lowp"],
                       "achieved": a, "unit": "TFLOP/s", "peak": peaks["bf16"],
                       "frac": a / peaks["bf16"] if peaks["bf16"] else None,
                       "frac_of_burst": a / peaks["bf16_burst"] if peaks["bf16_burst"] else None,
                       "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained (kernel timed inside a long step)"}
    if pf.get("n_oz"):
        a = pf["oz_ops"] / (pf["ms_oz"] * 1e-3) / 1e12
        # burst: the INT8 kernel exceeds 2 x the power-limited SUSTAINED bf16 GEMM rate (it draws less power
        # per op), so the sustained x 2 figure is no ceiling for it; the burst x 2 figure is
        pk = 2.0 * peaks["bf16_burst"] if peaks["bf16_burst"] else None
        pks = 2.0 * peaks["bf16"] if peaks["bf16"] else None
        out["int8"] = {"kernel": "ns_ozaki_product_kernel (INT8 digit pairs, tcgen05 kind::i8)", "launches": pf["n_oz"],
                       "achieved": a, "unit": "TOP/s", "peak": pk, "frac": a / pk if pk else None,
                       "frac_of_sustained_x2": a / pks if pks else None,
                       "peak_source": "MEASURED_PEAKS.json bf16_tflops (burst) x 2 (nominal int8 : bf16 = 4.5 : 2.25)"}
    return out


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
