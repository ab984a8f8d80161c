# split fp32 masters: full GPU tests + bench A/B
mkdir -p gpurun_out; o=gpurun_out/exp48.txt; : > $o
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -15 >> $o
for r in 1 2; do for v in 1 0; do
  PIPESIM_SPLIT_MASTER=$v timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/b48.json 2>gpurun_out/b48.err
  python -c "import json;d=json.load(open('gpurun_out/b48.json'));print('split=$v', round(d['value']), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']), d['clocks']['sm_mhz'], round(d['roofline']['in_step']['wgrad']['mean_us'],1))" >> $o 2>&1
done; done
cat $o
