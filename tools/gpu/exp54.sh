# L2 evict_last hint on forward weight loads (PIPESIM_DBG_EPI=64)
mkdir -p gpurun_out; o=gpurun_out/exp54.txt; : > $o
PIPESIM_DBG_EPI=64 timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k fwd 2>&1 | tail -1 >> $o
for r in 1 2 3; do for v in 0 64; do
  PIPESIM_DBG_EPI=$v timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/b54.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/b54.json'));print('dbg=$v', round(d['value']), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']), d['clocks']['sm_mhz'])" >> $o
done; done
cat $o
