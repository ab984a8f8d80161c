# interleaved hi|lo slots, one 3-D TMA box per chunk
mkdir -p gpurun_out; o=gpurun_out/exp53.txt; : > $o
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -2 >> $o
PIPESIM_SPLITK=0 python tools/gemm_exp.py >> $o 2>&1
for v in 4 2; do PIPESIM_DBG_EPI=$v PIPESIM_SPLITK=0 python tools/gemm_exp.py 2>&1 | sed "s/^/dbg=$v /" >> $o; done
for r in 1 2; do
  timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/b53.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/b53.json'));print('bench', round(d['value']), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']), d['clocks']['sm_mhz'], round(d['roofline']['in_step']['wgrad']['mean_us'],1))" >> $o
done
cat $o
