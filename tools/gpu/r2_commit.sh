timeout 900 python -m pytest tests -q -x -m gpu -p no:cacheprovider > gpurun_out/ce_pytest.log 2>&1; tail -1 gpurun_out/ce_pytest.log
export PIPESIM_SESSION_SPLIT=0
for sp in 1,1,1,2 2,1,2; do python tools/conv_determinism.py $sp 2>&1 | tail -3; done
unset PIPESIM_SESSION_SPLIT
python tools/mlp_determinism.py 2>&1 | tail -5
python tools/c1_timeline.py 2>&1 | head -1
PIPESIM_COMMIT_EDGES=0 python tools/c1_timeline.py 2>&1 | head -1
for i in 1 2; do
PIPESIM_BENCH_VGG=0 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-dropin > gpurun_out/ce_on_$i.json 2>/dev/null
PIPESIM_BENCH_VGG=0 PIPESIM_COMMIT_EDGES=0 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-dropin > gpurun_out/ce_off_$i.json 2>/dev/null
done
for f in ce_on_1 ce_off_1 ce_on_2 ce_off_2; do python -c "
import json;d=json.load(open('gpurun_out/$f.json'));print('$f', round(d['value']), round(d['e2e']['value']), d['clocks']['sm_mhz'], {k: round(v.get('us_per_mini_batch', 0),1) for k,v in d['other_configs'].items()})"; done
