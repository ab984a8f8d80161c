PIPESIM_SPLIT_MASTER=0 timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
timeout 900 python -m pytest tests/test_export.py tests/test_gpu_pipeline.py -q -m gpu -x 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_multiproc.py tests/test_gpu_pipeline.py -q -m gpu -x 2>&1 | tail -3
