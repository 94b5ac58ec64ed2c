"""Aggregate a tools/ncu_launches.sh listing: launches, total ms and share per kernel (first N launches)."""
import collections
import sys

rows = [ln.rsplit(None, 2) for ln in open(sys.argv[1]) if ln.strip()]
n = int(sys.argv[2]) if len(sys.argv) > 2 else len(rows)
agg = collections.OrderedDict()
tot = 0.0
for r in rows[:n]:
    if len(r) < 3:
        continue
    try:
        v = float(r[1])
    except ValueError:
        continue
    k = r[0].split("(")[0].replace("void ", "").strip()[:48]
    a = agg.setdefault(k, [0, 0.0])
    a[0] += 1
    a[1] += v
    tot += v
for k, (c, v) in agg.items():
    print(f"{k:50s} {c:5d} {v / 1e6:10.2f} ms {100 * v / tot:6.2f}%")
print(f"total {tot / 1e6:.2f} ms over {n} launches")
