# usage: bash tools/ncu_launches.sh <count> <kernel-regex> <command...>: per-launch kernel durations (ncu)
n=$1; shift; k=$1; shift
ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:$k" -c "$n" --csv "$@" 2>/dev/null | \
  python3 -c "
import csv,sys
rows=[r for r in csv.reader(sys.stdin) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value'); ui=h.index('Metric Unit')
for r in rows[1:]: print(r[ki][:60], r[vi], r[ui])
"
