# second wgrad stream per stage (PIPESIM_SIDE2=1)
mkdir -p gpurun_out; o=gpurun_out/exp61.txt; : > $o
PIPESIM_SIDE2=1 timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -2 >> $o
for r in 1 2 3; do for v in 1 0; do
  PIPESIM_SIDE2=$v timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/b61.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/b61.json'));print('side2=$v', round(d['value']), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']), d['clocks']['sm_mhz'])" >> $o
done; done
cat $o
