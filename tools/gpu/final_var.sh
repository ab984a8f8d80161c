# run-to-run spread of the default bench on one box
mkdir -p gpurun_out; o=gpurun_out/final_var.txt; : > $o
for r in 1 2 3; do
  timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/bv.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/bv.json'));print('run $r', round(d['value']), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']), 'step_frac', round(d['roofline']['step_frac_of_sustained'],3), d['clocks'])" >> $o
done
cat $o
