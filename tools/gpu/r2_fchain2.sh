# cluster forward chain: parity, then C1 / 1F1B / C2-sequential with and without
set -x
timeout 900 python -m pytest tests/test_gpu_dgrad_chain.py tests/test_gpu_pipeline.py -x -q 2>&1 | tail -3
for rep in 1 2; do
  for v in 0 1; do
    echo "== FWD_CHAIN=$v rep $rep"
    PIPESIM_FWD_CHAIN=$v timeout 300 python tools/c_timing.py --W 2 | tail -1
    PIPESIM_FWD_CHAIN=$v timeout 300 python tools/c_timing.py --W 2 --mode pipedream | tail -1
    PIPESIM_FWD_CHAIN=$v timeout 300 python tools/c_timing.py --W 1 --mode sequential | tail -1
  done
done
