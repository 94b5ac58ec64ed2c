# needs a second build: git worktree add build_ab/old <rev> && (cd build_ab/old && python paper_2605_24840_b200/build.py)
# alternate the in-tree library and build_ab/old's on the bench (FP64 cfg3), printing product kernel times
for v in new old new old; do
  if [ $v = new ]; then L=paper_2605_24840_b200/libnsreflector.so; else L=build_ab/old/paper_2605_24840_b200/libnsreflector.so; fi
  python tools/ab_lib.py $L bench.py --steps 3 --warmup 3 2>/dev/null > gpurun_out/ab_$v.json
  python -c "
import json; d=json.load(open('gpurun_out/ab_$v.json')); r=d['roofline']; print('$v', round(d['ms_per_step'],1), round(r['square_ms'],3), round(r['update_ms'],3), d['clocks']['sm_mhz'], d['clocks'].get('power_w_max'))"
done
