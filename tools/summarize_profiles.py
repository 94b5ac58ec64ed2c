"""Summarise ncu outputs into profiles/ (launch-list shares, key full-set metrics, traffic.json).

usage: python tools/summarize_profiles.py <tag> [--launches gpurun_out/x.csv] [--rep gpurun_out/x.ncu-rep] [--d 16384]
"""
import argparse
import collections
import csv
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size",
        "sm__cycles_elapsed.avg.per_second", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "lts__t_sector_hit_rate.pct", "smsp__inst_executed.sum"]


def launches(path, tag):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    agg = collections.OrderedDict()
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        n = r[ki].split("(")[0]
        a = agg.setdefault(n, [0, 0.0])
        a[0] += 1
        a[1] += float(r[vi].replace(",", ""))
    tot = sum(a[1] for a in agg.values())
    out = [f"# ncu launch list ({os.path.basename(path)}): --metrics gpu__time_duration.sum --clock-control none",
           "# cold-cache, serialised: compare SHARES, not absolute times", f"{'kernel':70s} {'launches':>8s} {'total_ms':>12s} {'share':>7s}"]
    for n, (c, t) in agg.items():
        out.append(f"{n:70s} {c:8d} {t / 1e6:12.3f} {100 * t / tot:6.2f}%")
    dst = os.path.join(PROF, f"{tag}_launches.txt")
    open(dst, "w").write("\n".join(out) + "\n")
    print("\n".join(out))


def full(rep, tag, d):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out, traffic = [f"# ncu --set full summary of {os.path.basename(rep)}"], None
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        out.append(f"## {name}")
        vals = {}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                out.append(f"{k:75s} {r[i]:>20s} {units[i]}")
                vals[k] = (r[i], units[i])
        try:
            rd = float(vals["dram__bytes_read.sum"][0]) * (1e9 if vals["dram__bytes_read.sum"][1] == "Gbyte" else 1e6 if vals["dram__bytes_read.sum"][1] == "Mbyte" else 1)
            wr = float(vals["dram__bytes_write.sum"][0]) * (1e9 if vals["dram__bytes_write.sum"][1] == "Gbyte" else 1e6 if vals["dram__bytes_write.sum"][1] == "Mbyte" else 1)
            if traffic is None and rd == rd:
                traffic = rd + wr
        except (KeyError, ValueError):
            pass
    dst = os.path.join(PROF, f"{tag}_ncu_full.txt")
    open(dst, "w").write("\n".join(out) + "\n")
    print("\n".join(out))
    if traffic and d:
        tj = os.path.join(PROF, "traffic.json")
        cur = json.load(open(tj)) if os.path.exists(tj) else {}
        cur[str(d)] = {"bytes_per_launch": traffic, "source": f"profiles/{tag}_ncu_full.txt (dram read+write, first "
                                                               f"ns_product_kernel launch)"}
        json.dump(cur, open(tj, "w"), indent=1)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("tag")
    ap.add_argument("--launches")
    ap.add_argument("--rep")
    ap.add_argument("--d", type=int, default=0)
    a = ap.parse_args()
    if a.launches:
        launches(a.launches, a.tag)
    if a.rep:
        full(a.rep, a.tag, a.d)
