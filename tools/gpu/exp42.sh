# fill/drain mini-batches on 256-wide tiles (PIPESIM_EDGE_NARROW)
mkdir -p gpurun_out; o=gpurun_out/exp42.txt; : > $o
timeout 600 python -m pytest tests/test_gpu_pipeline.py -q -x 2>&1 | tail -1 >> $o
for r in 1 2 3; do for v in 1 0; do
  PIPESIM_EDGE_NARROW=$v timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/b42.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/b42.json'));print('edge_narrow=$v', round(d['value']), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']), d['clocks']['sm_mhz'])" >> $o
done; done
cat $o
