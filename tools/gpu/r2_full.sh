mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/r2g_pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/r2g_pytest.log
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/r2g_bench.json 2> gpurun_out/r2g_bench.err; echo bench rc=$?
python -c "import json;d=json.load(open('gpurun_out/r2g_bench.json'));print(round(d['value']), round(d['ms_per_step'],2), d['e2e']['value'], d['roofline']['frac'], d['clocks']); print(json.dumps(d.get('e2e_dropin'))[:1500])"
