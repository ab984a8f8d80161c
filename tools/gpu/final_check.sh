mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_final.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/pytest_final.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/bench_final2.json 2> gpurun_out/bench_final2.err; echo bench rc=$?
python -c "import json;d=json.load(open('gpurun_out/bench_final2.json'));print(round(d['value']), round(d['ms_per_step'],2), round(d['e2e']['value']), round(d['roofline']['step_frac_of_sustained'],3), d['clocks'], d['cpu_baseline']['value'])"
