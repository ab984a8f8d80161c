timeout 900 python -m pytest tests -q -x -m gpu -p no:cacheprovider > gpurun_out/pdl_pytest.log 2>&1; tail -1 gpurun_out/pdl_pytest.log
python tools/c1_timeline.py 2>&1 | head -1
PIPESIM_PDL=0 python tools/c1_timeline.py 2>&1 | head -1
for i in 1 2; do
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-dropin > gpurun_out/pdl_on_$i.json 2>/dev/null
done
for f in pdl_on_1 pdl_on_2; do python -c "
import json;d=json.load(open('gpurun_out/$f.json'));print('$f', round(d['value']), round(d['e2e']['value']), d['clocks']['sm_mhz'], d['other_configs'])"; done
