#!/bin/bash
# DRAM traffic of the FP64 square kernel at d=16384 vs the tile-order super-block edge (ncu, one launch each)
for G in 4 6 8 12 16 24; do
  NS_TILE_GROUP=$G timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none -k regex:ns_product_kernel -s 0 -c 1 --csv python tools/oz_prof.py 16384 fp64 2>/dev/null \
    | grep -E "dram__bytes|gpu__time" | awk -F'","' -v g=$G '{print "G=" g, $(NF-2), $(NF-1), $NF}'
done
