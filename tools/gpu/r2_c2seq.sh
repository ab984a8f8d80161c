# C2 sequential (W=1) per mini-batch time under each latency switch
for rep in 1 2; do
  for v in "" "PIPESIM_DGRAD_CHAIN=0" "PIPESIM_FWD_CHAIN=0" "PIPESIM_SPARE_ACT=0" "PIPESIM_PRUNE_EDGES=0" "PIPESIM_DGRAD_CHAIN=0 PIPESIM_FWD_CHAIN=0 PIPESIM_SPARE_ACT=0 PIPESIM_PRUNE_EDGES=0"; do
    echo "== [$v] rep $rep: $(env $v timeout 300 python tools/c_timing.py --W 1 --mode sequential 2>&1 | tail -1)"
  done
done
