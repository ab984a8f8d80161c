# forward epilogue: TMEM load of the next step in flight during the stores
mkdir -p gpurun_out; o=gpurun_out/exp64.txt; : > $o
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -1 >> $o
PIPESIM_SPLITK=0 python tools/gemm_exp.py >> $o 2>&1
for r in 1 2; do
  timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/b64.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/b64.json'));print('bench', round(d['value']), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']), d['clocks']['sm_mhz'])" >> $o
done
cat $o
