# fused two-layer dgrad (PIPESIM_DGRAD_CHAIN) and the spare activation slot
# of latency-bound networks (PIPESIM_SPARE_ACT): parity, then C1 / 1F1B per
# mini-batch time for each combination, alternating
set -x
timeout 900 python -m pytest tests/test_gpu_dgrad_chain.py -x -q 2>&1 | tail -3
timeout 1500 python -m pytest tests -m gpu -x -q -k "pipeline or configs or multiproc or verify or guard or capi" 2>&1 | tail -3
for rep in 1 2; do
  for v in "0 0" "1 0" "0 1" "1 1"; do
    set -- $v
    echo "== CHAIN=$1 SPARE=$2 rep $rep"
    PIPESIM_DGRAD_CHAIN=$1 PIPESIM_SPARE_ACT=$2 timeout 300 python tools/c1_timeline.py 2>&1 | head -1
  done
done
python tools/c1_trace.py > gpurun_out/c1_trace_chain.log 2>&1; head -3 gpurun_out/c1_trace_chain.log
python tools/c1_trace.py --mode pipedream > gpurun_out/c1_trace_chain_pd.log 2>&1; head -1 gpurun_out/c1_trace_chain_pd.log
