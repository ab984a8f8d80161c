# knob re-check with split masters (one box, alternating)
mkdir -p gpurun_out; o=gpurun_out/exp57.txt; : > $o
for r in 1 2; do
for cfg in "X=0" "PIPESIM_BN512_ROWS=1024" "PIPESIM_BN512=0" "PIPESIM_MAXPAIRS=64" "PIPESIM_BIAS_STREAM=0"; do
  env $cfg timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/b57.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/b57.json'));print('$cfg', round(d['value']), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']), d['clocks']['sm_mhz'])" >> $o
done; done
cat $o
