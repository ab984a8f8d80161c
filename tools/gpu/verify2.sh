mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_verify.py -q -x > gpurun_out/verify.log 2>&1; echo verify rc=$?; tail -25 gpurun_out/verify.log
timeout 600 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo all rc=$?; tail -3 gpurun_out/pytest_gpu.log
