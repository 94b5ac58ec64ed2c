# Consolidated round-end evidence on one B200: GPU tests, the default bench line, every config,
# and the bench's kernel launch list (ncu, only after the same command exited 0 without ncu).
# usage: bash tools/final_run.sh <tag>   (outputs under gpurun_out/<tag>_*)
T=${1:-final}
python -m pytest tests -q -m gpu 2>&1 | tail -3 > gpurun_out/${T}_pytest.txt
python bench.py --steps 3 --warmup 3 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
python tools/bench_configs.py cfg0 cfg1 cfg1ozaki cfg2 cfg3 cfg3mixed cfg3mixedoz cfg3tf32 cfg3ozaki cfg3fixed \
  cfg3fixedmixed cfg3fixedmixedoz cfg3fixedozaki cfg4 cfg4single cfg4ozaki kscan 2>/dev/null | grep '^{' > gpurun_out/${T}_configs.jsonl
python bench.py --steps 1 --warmup 3 --no-mixed --no-cpu-baseline --no-e2e > /dev/null 2>&1 && \
  bash tools/ncu_launches.sh 400 "ns_" python bench.py --steps 1 --warmup 3 --no-mixed --no-cpu-baseline --no-e2e \
  > gpurun_out/${T}_launches.txt 2>&1
cat gpurun_out/${T}_pytest.txt
