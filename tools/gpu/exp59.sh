# dgrad tile width on the critical backward chain
mkdir -p gpurun_out; o=gpurun_out/exp59.txt; : > $o
for r in 1 2 3; do for v in 1 0; do
  PIPESIM_BN512_DGRAD=$v timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/b59.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/b59.json'));print('dgrad512=$v', round(d['value']), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']), d['clocks']['sm_mhz'])" >> $o
done; done
cat $o
