for mc in 1 0; do for dbg in 0 1; do
  NS_OZ_MC=$mc NS_OZ_DBG=$dbg python tools/oz_time.py 16384 ozaki 0
  NS_OZ_MC=$mc NS_OZ_DBG=$dbg bash tools/ncu_launches.sh 6 "ozaki_product" python tools/oz_time.py 16384 ozaki 0 | tail -2 | sed "s/^/mc=$mc dbg=$dbg /"
done; done
