# needs a second build: git worktree add build_ab/old <rev> && (cd build_ab/old && python paper_2605_24840_b200/build.py)
# Ozaki product A/B: in-tree library vs build_ab/old, alternating
for v in new old new old; do
  if [ $v = new ]; then L=paper_2605_24840_b200/libnsreflector.so; else L=build_ab/old/paper_2605_24840_b200/libnsreflector.so; fi
  python tools/ab_lib.py $L tools/oz_time.py 16384 ozaki 0 | sed "s/^/$v /"
  python tools/ab_lib.py $L tools/oz_time.py 16384 ozaki 1 | sed "s/^/$v /"
done
