# BN=512 row threshold A/B (uninstrumented timed step) + reference arm
mkdir -p gpurun_out
for r in 0 512 1024 0; do
  for rep in 1 2; do
    PIPESIM_BN512_ROWS=$r timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/b33.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/b33.json'));print('rows>=$r', round(d['value']), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']), 'fwd', round(d['roofline']['in_step']['fwd']['tflops']), d['clocks']['sm_mhz'])" >> gpurun_out/exp33.txt
  done
done
PIPESIM_BN512=0 timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/b33.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/b33.json'));print('bn512 off', round(d['value']), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']), d['clocks']['sm_mhz'])" >> gpurun_out/exp33.txt
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref33.json 2> gpurun_out/bench_ref33.err
nproc >> gpurun_out/exp33.txt; free -g >> gpurun_out/exp33.txt
cat gpurun_out/exp33.txt gpurun_out/bench_ref33.json
