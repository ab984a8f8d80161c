# stream priorities re-check: 0 (none), 3 (dgrad chain first), 4 (commits first)
mkdir -p gpurun_out; o=gpurun_out/exp62.txt; : > $o
for r in 1 2; do for v in 0 3 4; do
  PIPESIM_PRIO=$v timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/b62.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/b62.json'));print('prio=$v', round(d['value']), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']), d['clocks']['sm_mhz'])" >> $o
done; done
cat $o
