for v in 1 0 1 0; do
  NS_DIAG_TRI=$v python bench.py --steps 3 --warmup 3 2>/dev/null > gpurun_out/ab_$v.json
  python -c "
import json; d=json.load(open('gpurun_out/ab_$v.json')); r=d['roofline']; print('tri=$v', round(d['ms_per_step'],1), round(r['square_ms'],3), round(r['update_ms'],3), d['clocks']['sm_mhz'])"
  NS_DIAG_TRI=$v python tools/bench_configs.py cfg1 2>&1 | python -c "import sys,json; [print('tri=$v cfg1', round(json.loads(l)['time_ms'],2)) for l in sys.stdin if l.startswith('{')]"
done
