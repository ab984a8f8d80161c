set -x
timeout 600 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -3 gpurun_out/smoke.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_m32.log 2>&1; echo bench rc=$?; tail -3 gpurun_out/bench_m32.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --mini-batches 8 --no-cpu-baseline > gpurun_out/ncu_list.log 2>&1; echo ncu rc=$?; tail -3 gpurun_out/ncu_list.log
