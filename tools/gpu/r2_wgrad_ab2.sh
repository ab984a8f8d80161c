# A/B: L2 tensor prefetch of the next tile's masters in the split SGD epilogue
mkdir -p gpurun_out
for v in base pf1 pf1b4; do
  if [ $v = base ]; then unset PIPESIM_LIB; else export PIPESIM_LIB=$PWD/paper_2410_14312_b200/lib/variants/libpipesim_b200_$v.so; fi
  timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_pipeline.py -q -m gpu -x -p no:cacheprovider -k "split or wgrad or c3" > gpurun_out/ab2_$v.test.log 2>&1; echo $v tests rc=$? $(tail -1 gpurun_out/ab2_$v.test.log)
  for rep in 1 2; do
  timeout 600 python bench.py --no-cpu-baseline --no-dropin > gpurun_out/ab2_$v.json 2> gpurun_out/ab2_$v.err
  python -c "
import json;d=json.load(open('gpurun_out/ab2_$v.json'));k=d['roofline']['kinds']
print('$v', round(d['value']), round(d['ms_per_step'],2), d['clocks']['sm_mhz'], 'wgrad', {s:round(v['us'],1) for s,v in k['wgrad']['shapes'].items()}, 'hbm', round(k['wgrad']['shapes']['1024x4096x4096']['hbm_gbs']))"
  done
done
