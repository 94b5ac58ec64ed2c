for v in new old new old; do
  if [ $v = new ]; then L=paper_2605_24840_b200/libnsreflector.so; else L=build_ab/small_v0.so; fi
  echo "$v $(python tools/ab_lib.py $L tools/small_prof.py 3000)"
done
for v in new old; do
  if [ $v = new ]; then L=paper_2605_24840_b200/libnsreflector.so; else L=build_ab/small_v0.so; fi
  echo "== $v kernel durations (ncu)"
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:ns_small -c 12 --csv python tools/ab_lib.py $L tools/small_prof.py 10 2>/dev/null | grep gpu__time | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' '; echo
done
python -m pytest tests/test_gpu_parity.py -q -k "cfg0 or ragged or small or boundaries or edge" 2>&1 | tail -2
