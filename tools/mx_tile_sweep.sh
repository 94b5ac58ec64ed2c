# L2-locality sweep of the BF16x3 product kernel: super-block edge of the tile order (mode 0: upper tiles,
# NS_TILE_GROUP; mode 2: all tiles, NS_TILE_GROUP_FULL).
for gu in 4 8 16; do
  echo "mode 0 G_upper=$gu"
  NS_TILE_GROUP=$gu ncu --metrics gpu__time_duration.sum,lts__t_sector_hit_rate.pct,dram__bytes_read.sum --clock-control none -k regex:ns_mx_product -c 1 python tools/oz_prof.py 16384 mixed 0 2>&1 | grep -E "duration|hit_rate|dram__bytes" | awk '{print $1, $(NF-1), $NF}'
done
for g in 4 6 8 12 16; do
  echo "mode 2 G_full=$g"
  NS_TILE_GROUP_FULL=$g ncu --metrics gpu__time_duration.sum,lts__t_sector_hit_rate.pct,dram__bytes_read.sum --clock-control none -k regex:ns_mx_product -c 1 python tools/oz_prof.py 16384 mixed 2 2>&1 | grep -E "duration|hit_rate|dram__bytes" | awk '{print $1, $(NF-1), $NF}'
done
