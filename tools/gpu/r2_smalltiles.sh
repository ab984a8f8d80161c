# 256-row forwards of the 16x4096 step on 128-wide tiles (PIPESIM_SMALL_TILES=17)
for rep in 1 2; do
  for v in 16 17; do
    PIPESIM_SMALL_TILES=$v PIPESIM_BENCH_VGG=0 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-dropin 2>/dev/null | python -c "
import sys,json;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);r=d['roofline']
print('SMALL_TILES=$v', round(d['value']), d['clocks']['sm_mhz'], 'frac', round(r['frac'],3), {k: round(v['us'],1) for k,v in r['kinds']['fwd']['shapes'].items()})"
  done
done
