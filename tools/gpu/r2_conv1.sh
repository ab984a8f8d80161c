mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_convnet.py tests/test_gpu_pipeline.py tests/test_gpu_multiproc.py -x -q -p no:cacheprovider > gpurun_out/r2_conv1.log 2>&1; echo rc=$?; tail -30 gpurun_out/r2_conv1.log
