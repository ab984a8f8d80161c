mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_multiproc.py -q -x > gpurun_out/mp.log 2>&1; echo mp rc=$?; tail -30 gpurun_out/mp.log
