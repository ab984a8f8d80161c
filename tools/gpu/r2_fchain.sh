# fused two-layer forward (PIPESIM_FWD_CHAIN): parity, then C1 / 1F1B / C2
# per mini-batch time with and without, alternating
set -x
timeout 900 python -m pytest tests/test_gpu_dgrad_chain.py -x -q 2>&1 | tail -15
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
for rep in 1 2; do
  for v in 0 1; do
    echo "== FWD_CHAIN=$v rep $rep"
    PIPESIM_FWD_CHAIN=$v timeout 300 python tools/c1_timeline.py 2>&1 | head -1
    PIPESIM_FWD_CHAIN=$v timeout 300 python tools/c1_trace.py --mode pipedream 2>&1 | head -1
  done
done
python tools/c1_trace.py > gpurun_out/c1_trace_fchain.log 2>&1; head -14 gpurun_out/c1_trace_fchain.log
