# usage: bash tools/ncu_launches.sh <count> <kernel-regex> <command...>: per-launch kernel durations (ncu)
n=$1; shift; k=$1; shift
ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:$k" -c "$n" --csv "$@" 2>/dev/null | \
  python3 -c "
import csv,sys
rows=list(csv.reader(sys.stdin))
hi=next(i for i,r in enumerate(rows) if 'Kernel Name' in r)
h=rows[hi]; ki=h.index('Kernel Name'); vi=h.index('Metric Value'); ui=h.index('Metric Unit')
for r in rows[hi+1:]:
    if len(r)==len(h): print(r[ki][:60], r[vi], r[ui])
"
