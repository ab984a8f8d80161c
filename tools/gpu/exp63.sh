# steady state: more mini-batches per step (fill/drain amortised)
mkdir -p gpurun_out; o=gpurun_out/exp63.txt; : > $o
for m in 32 64 128; do
  timeout 600 python bench.py --steps 4 --warmup 3 --mini-batches $m --no-cpu-baseline > gpurun_out/b63.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/b63.json'));print('M=$m', round(d['value']), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']), round(d['roofline']['step_frac_of_sustained'],3), d['clocks']['sm_mhz'])" >> $o
done
cat $o
