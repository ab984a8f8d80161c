python tools/c1_timeline.py 2>&1 | head -1
PIPESIM_SPLITK_MINKB=8 python tools/c1_timeline.py 2>&1 | head -1
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_pipeline.py tests/test_gpu_configs.py -q -x -p no:cacheprovider 2>&1 | tail -1
