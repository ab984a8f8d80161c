# wgrad wave quantisation: 256 tiles on 64 pairs (4 full waves) vs 74 pairs (3.46 waves)
mkdir -p gpurun_out; o=gpurun_out/exp45.txt; : > $o
for v in 74 64; do PIPESIM_MAXPAIRS=$v PIPESIM_SPLITK=0 python tools/gemm_exp.py >> $o 2>&1; done
for r in 1 2 3; do for v in 74 64; do
  PIPESIM_MAXPAIRS=$v timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/b45.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/b45.json'));print('maxpairs=$v', round(d['value']), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']), d['clocks']['sm_mhz'])" >> $o
done; done
cat $o
