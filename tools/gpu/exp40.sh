# wgrad store cost: all stores (4) vs bf16 stores only (8)
mkdir -p gpurun_out; o=gpurun_out/exp40.txt; : > $o
for v in 0 8 4 0 8; do PIPESIM_DBG_EPI=$v PIPESIM_SPLITK=0 python tools/gemm_exp.py >> $o 2>&1; done
timeout 300 python bench.py --steps 8 --warmup 3 > gpurun_out/b40.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/b40.json'));print('bench', round(d['value']), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']), d['clocks']['sm_mhz'], d['roofline']['traffic'])" >> $o
cat $o
