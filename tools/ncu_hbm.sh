# usage: bash tools/ncu_hbm.sh <count> <command...>: per-launch duration and DRAM bytes of the library's
# kernels (ncu, cold-cache, serialised), summed
n=$1; shift
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k "regex:ns_" \
  -c "$n" --csv "$@" 2>/dev/null | python3 -c "
import csv, sys, collections
rows = list(csv.reader(sys.stdin))
hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hi]; ki = h.index('ID'); mi = h.index('Metric Name'); vi = h.index('Metric Value'); ui = h.index('Metric Unit')
scale = {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9, 'ns': 1e-9, 'us': 1e-6, 'usecond': 1e-6, 'msecond': 1e-3, 'nsecond': 1e-9}
tot = collections.defaultdict(float); ids = set()
for r in rows[hi + 1:]:
    if len(r) != len(h): continue
    ids.add(r[ki]); tot[r[mi]] += float(r[vi].replace(',', '')) * scale.get(r[ui], 1)
t = tot['gpu__time_duration.sum']; rd = tot['dram__bytes_read.sum']; wr = tot['dram__bytes_write.sum']
print(f'{len(ids)} launches, {t*1e3:.1f} ms, read {rd/1e9:.1f} GB, write {wr/1e9:.1f} GB -> {(rd+wr)/t/1e12:.2f} TB/s average')
"
