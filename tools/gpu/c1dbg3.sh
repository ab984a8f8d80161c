for v in 0 1; do for r in 1 2 3; do
echo "== split=$v run $r"
PIPESIM_SPLIT_MASTER=$v timeout 300 python -m pytest tests/test_gpu_pipeline.py -q -x -k "coalescing_is_bit" 2>&1 | grep -E "passed|failed|Mismatch|Max abs|Max rel|Mismatched" | head -5
done; done
