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
# full ncu capture of one full-batch 64-tile launch (cfg1 square + update), after the same command ran clean
python tools/cfg1_prof.py > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on \
  -k "regex:ns_product64_kernel" -s 2 -c 2 -o gpurun_out/${T}_p64 python tools/cfg1_prof.py > gpurun_out/${T}_p64.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.txt 2>&1
python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/${T}_reference.json 2>/dev/null
