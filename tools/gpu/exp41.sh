# bf16 copy as 32x64 TMA boxes (3 stores per 64 columns)
mkdir -p gpurun_out; o=gpurun_out/exp41.txt; : > $o
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_pipeline.py tests/test_gpu_verify.py -q -x 2>&1 | tail -2 >> $o
for v in 0 8 0; do PIPESIM_DBG_EPI=$v PIPESIM_SPLITK=0 python tools/gemm_exp.py >> $o 2>&1; done
for r in 1 2; do
  timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/b41.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/b41.json'));print('bench', round(d['value']), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']), d['clocks']['sm_mhz'])" >> $o
done
cat $o
