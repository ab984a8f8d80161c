timeout 900 python -m pytest tests -q -x -m gpu -p no:cacheprovider > gpurun_out/st_pytest.log 2>&1; tail -1 gpurun_out/st_pytest.log
python tools/configs.py 2>/dev/null | head -8
for i in 1 2; do
PIPESIM_BENCH_VGG=0 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-dropin > gpurun_out/st_on_$i.json 2>/dev/null
PIPESIM_BENCH_VGG=0 PIPESIM_SMALL_TILES=0 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-dropin > gpurun_out/st_off_$i.json 2>/dev/null
done
for f in st_on_1 st_off_1 st_on_2 st_off_2; do python -c "
import json;d=json.load(open('gpurun_out/$f.json'));print('$f', round(d['value']), round(d['e2e']['value']), d['clocks']['sm_mhz'], {k: round(v.get('us_per_mini_batch', 0),1) for k,v in d['other_configs'].items()})"; done
