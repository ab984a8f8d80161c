mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo bench rc=$?; tail -c 4000 gpurun_out/bench_full.json
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1b.csv python tools/prof_step.py 4 > gpurun_out/prof_step.log 2>&1; echo ncu-list rc=$?
python tools/launch_summary.py gpurun_out/launches_r1b.csv > gpurun_out/launch_summary.txt 2>&1; cat gpurun_out/launch_summary.txt
timeout 400 ncu --set full --clock-control none --import-source on -k regex:gemm -c 3 -o gpurun_out/prof_r1b python tools/prof_gemm.py fwd256,dgrad,wgrad 1 > gpurun_out/prof_r1b.log 2>&1; echo ncu-full rc=$?
