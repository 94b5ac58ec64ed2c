for t in 1e-6 1e-7 1e-8 1e-9; do
  NS_CG_TOL=$t NS_CG_DEBUG=1 python tools/cg_tol_sweep.py 2>&1 | grep -E "worst|iterations" | sort | uniq -c | sort -rn | head -8
  NS_CG_TOL=$t NS_CG_DEBUG=1 python tools/bench_configs.py cfg3mixed 2>&1 | grep -E "iterations|^\{" | cut -c1-200
done
