# dgrad chain as a cluster (PIPESIM_CHAIN_CLUSTER): parity, sanitizer, C1 / 1F1B A/B
set -x
timeout 900 python -m pytest tests/test_gpu_dgrad_chain.py tests/test_gpu_pipeline.py tests/test_gpu_configs.py -x -q 2>&1 | tail -2
for rep in 1 2; do
  for v in 0 1; do
    echo "== CHAIN_CLUSTER=$v rep $rep"
    PIPESIM_CHAIN_CLUSTER=$v timeout 300 python tools/c_timing.py --W 2 | tail -1
    PIPESIM_CHAIN_CLUSTER=$v timeout 300 python tools/c_timing.py --W 2 --mode pipedream | tail -1
  done
done
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 900 $CS --tool $tool --target-processes all --print-limit 20 python tools/sanitize_run.py timeprest > gpurun_out/san_cc_$tool.log 2>&1; echo $tool rc=$?; tail -1 gpurun_out/san_cc_$tool.log
done
