timeout 240 python -m pytest tests/test_gpu_kernels.py -q -x > gpurun_out/kern.log 2>&1; echo kern rc=$?; tail -5 gpurun_out/kern.log
timeout 240 python -m pytest tests/test_gpu_pipeline.py -q -x > gpurun_out/pipe.log 2>&1; echo pipe rc=$?; tail -5 gpurun_out/pipe.log
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench2.log 2>&1; echo bench rc=$?; tail -1 gpurun_out/bench2.log | cut -c1-1500
