# after the latency changes: the whole GPU suite, smoke, the small-network
# configs table and the default bench line (profiles/round2/)
O=gpurun_out/r2f; mkdir -p $O
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -1 $O/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$?; tail -1 $O/smoke.log
for rep in 1 2; do timeout 300 python tools/c_timing.py --W 1 --mode sequential | tail -1; timeout 300 python tools/c_timing.py --W 2 | tail -1; done
timeout 600 python tools/configs.py --out $O/configs_r2.json > $O/configs_r2.md 2> $O/configs.err; echo configs rc=$?
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo bench rc=$?
python -c "import json;d=json.load(open('$O/bench.json'));print(round(d['value']), round(d['ms_per_step'],2), round(d['e2e']['value']), d['roofline']['frac'], d['clocks'])"
timeout 600 python tools/vgg_bench.py --W 4 8 --M 16 --profile --out $O/vgg16_bench.json > /dev/null 2> $O/vgg.err; echo vgg rc=$?
