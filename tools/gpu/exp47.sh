# step sensitivity (timing only): bf16 copy stores skipped (8)
mkdir -p gpurun_out; o=gpurun_out/exp47.txt; : > $o
for r in 1 2; do for v in 0 8; do
  PIPESIM_DBG_EPI=$v timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/b47.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/b47.json'));print('dbg=$v', round(d['value']), round(d['ms_per_step'],2), d['clocks']['sm_mhz'])" >> $o
done; done
cat $o
