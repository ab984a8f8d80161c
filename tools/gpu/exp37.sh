# vector epilogue interior fast path (fwd/dgrad), bias kernel v2, 2-buffer SGD
mkdir -p gpurun_out; o=gpurun_out/exp37.txt; : > $o
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -2 >> $o
for r in 1 2; do
  PIPESIM_SPLITK=0 python tools/gemm_exp.py >> $o 2>&1
  timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/b37.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/b37.json'));print('bench', round(d['value']), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']), d['clocks']['sm_mhz'])" >> $o
done
PIPESIM_SPLITK=0 timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm -c 2 -o gpurun_out/prof_37 python tools/prof_gemm.py fwd1024,dgrad 1 > /dev/null 2>&1
cat $o
