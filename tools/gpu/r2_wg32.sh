# 32-wide single-CTA wgrad (64-byte-swizzle MN-major B) on latency-bound nets
set -x
PIPESIM_WGRAD_SINGLE=32 timeout 600 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_dgrad_chain.py -x -q 2>&1 | tail -2
for rep in 1 2; do
  for v in 64 32; do
    echo "== WGRAD_SINGLE=$v rep $rep"
    PIPESIM_WGRAD_SINGLE=$v timeout 300 python tools/c_timing.py --W 2 | tail -1
    PIPESIM_WGRAD_SINGLE=$v timeout 300 python tools/c_timing.py --W 2 --mode pipedream | tail -1
    PIPESIM_WGRAD_SINGLE=$v timeout 300 python tools/c_timing.py --W 1 --mode sequential | tail -1
  done
done
