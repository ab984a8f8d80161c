for r in 1 2 3; do
PIPESIM_SPLIT_MASTER=0 timeout 300 python -m pytest tests/test_gpu_pipeline.py -q -x -k "coalescing_is_bit" 2>&1 | grep -E "passed|failed|Max rel" | head -3
done
