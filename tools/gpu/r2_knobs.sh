# latency knobs on the final C1 cycle
for rep in 1 2; do
  for v in "" "PIPESIM_SPLITK_MINKB=4" "PIPESIM_SPLITK_MINKB=6" "PIPESIM_CHAIN_BN=128" "PIPESIM_BN64=16" "PIPESIM_SMALL_TILES=0" "PIPESIM_PDL=0"; do
    echo "== [$v] rep $rep: $(env $v timeout 300 python tools/c_timing.py --W 2 | tail -1) | $(env $v timeout 300 python tools/c_timing.py --W 1 --mode sequential | tail -1)"
  done
done
