# bias prefetch + tiles-per-pair A/B for fwd/dgrad
mkdir -p gpurun_out; o=gpurun_out/exp34.txt; : > $o
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x 2>&1 | tail -1 >> $o
for cfg in "1 1" "0 2" "0 1" "1 2" "1 1" "0 2"; do
  set -- $cfg
  PIPESIM_SPLITK=0 PIPESIM_BN512=$1 PIPESIM_TILES_PER_PAIR=$2 python tools/gemm_exp.py 2>&1 | sed "s/^/bn512=$1 tpp=$2 /" >> $o
  PIPESIM_BN512=$1 PIPESIM_TILES_PER_PAIR=$2 timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/b34.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/b34.json'));print('bn512=$1 tpp=$2', round(d['value']), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']), d['clocks']['sm_mhz'])" >> $o
done
cat $o
