mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo bench rc=$?; python -c "import json;d=json.load(open('gpurun_out/bench_full.json'));print(d['value'],d['ms_per_step'],d['e2e']['value'],d['roofline']['step_gemm_tflops'],d['clocks'])"
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1j.csv python tools/prof_step.py 4 > gpurun_out/prof_step.log 2>&1; echo ncu-list rc=$?
python tools/launch_summary.py gpurun_out/launches_r1j.csv
PIPESIM_SPLITK=0 timeout 400 ncu --set full --clock-control none --import-source on -k regex:gemm -c 3 -o gpurun_out/prof_r1j python tools/prof_gemm.py fwd1024,dgrad,wgrad 1 > gpurun_out/prof_r1j.log 2>&1; echo ncu-full rc=$?
timeout 900 python tools/sweep.py --out gpurun_out/sweep_r1.json > gpurun_out/sweep_r1.md 2> gpurun_out/sweep_r1.err; echo sweep rc=$?
timeout 600 python tools/configs.py --out gpurun_out/configs_r1.json > gpurun_out/configs_r1.md 2> gpurun_out/configs_r1.err; echo configs rc=$?
timeout 600 python tools/timeline.py --out-json gpurun_out/timeline_r1.json --trace gpurun_out/trace_r1.json > gpurun_out/timeline_r1.txt 2>&1; echo tl rc=$?
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref_r1j.json 2> gpurun_out/bench_ref_r1j.err; echo ref rc=$?
