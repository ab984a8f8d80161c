# ReLU sign masks: full GPU suite + bench A/B (PIPESIM_RELU_MASK=0)
mkdir -p gpurun_out; o=gpurun_out/exp55.txt; : > $o
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3 >> $o
PIPESIM_SPLITK=0 python tools/gemm_exp.py >> $o 2>&1
for r in 1 2; do for v in 1 0; do
  PIPESIM_RELU_MASK=$v timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/b55.json 2>gpurun_out/b55.err
  python -c "import json;d=json.load(open('gpurun_out/b55.json'));print('mask=$v', round(d['value']), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']), d['clocks']['sm_mhz'], round(d['roofline']['in_step']['dgrad']['mean_us'],1))" >> $o 2>&1
done; done
cat $o
