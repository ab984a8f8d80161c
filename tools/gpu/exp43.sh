# wgrad master loads by cp.async (32) vs TMA (0)
mkdir -p gpurun_out; o=gpurun_out/exp43.txt; : > $o
PIPESIM_DBG_EPI=32 timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "dw_sgd" 2>&1 | tail -1 >> $o
PIPESIM_DBG_EPI=32 timeout 600 python -m pytest tests/test_gpu_pipeline.py -q -x 2>&1 | tail -1 >> $o
for v in 0 32 0 32; do PIPESIM_DBG_EPI=$v PIPESIM_SPLITK=0 python tools/gemm_exp.py >> $o 2>&1; done
for r in 1 2; do for v in 0 32; do
  PIPESIM_DBG_EPI=$v timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/b43.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/b43.json'));print('epi=$v', round(d['value']), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']), d['clocks']['sm_mhz'])" >> $o
done; done
cat $o
