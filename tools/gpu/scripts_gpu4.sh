timeout 300 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu4.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu4.log
timeout 400 ncu --set full --clock-control none --import-source on -k regex:gemm -c 3 -o gpurun_out/prof_gemm_r1 python tools/prof_gemm.py all 1 > gpurun_out/prof_gemm_r1.log 2>&1; echo ncu-full rc=$?
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv python tools/prof_step.py 4 > gpurun_out/prof_step_r1.log 2>&1; echo ncu-list rc=$?
timeout 600 python bench.py > gpurun_out/bench_r1.json 2> gpurun_out/bench_r1.err; echo bench rc=$?; tail -c 1500 gpurun_out/bench_r1.json
