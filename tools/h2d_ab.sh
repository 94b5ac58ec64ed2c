# e2e A/B of the chunked H staging (ns_reflector_host): NS_H2D_CHUNKS=1 (default) vs 0
for v in 1 0 1 0; do
  NS_H2D_CHUNKS=$v python bench.py --steps 3 --warmup 3 --no-mixed --no-cpu-baseline 2>/dev/null > gpurun_out/h2d_$v.json
  python -c "
import json; d=json.load(open('gpurun_out/h2d_$v.json')); print('chunks=$v value', round(d['value'],3), 'e2e', round(d['e2e']['value'],3), round(d['e2e'].get('ms_per_step',0),1))"
done
