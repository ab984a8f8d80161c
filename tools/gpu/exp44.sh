mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_verify.py -q -x -k full_width -s 2>&1 | tail -5
