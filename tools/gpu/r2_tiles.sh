mkdir -p gpurun_out
PIPESIM_FWD_FIX=1 timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "linear_fwd" 2>&1 | tail -1
for i in 1 2; do
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-dropin > gpurun_out/t512_$i.json 2>/dev/null
PIPESIM_BN512=0 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-dropin > gpurun_out/t256_$i.json 2>/dev/null
done
for f in t512_1 t256_1 t512_2 t256_2; do python -c "
import json;d=json.load(open('gpurun_out/$f.json'));r=d['roofline'];print('$f', round(d['value']), round(d['e2e']['value']), r['frac'], d['clocks']['sm_mhz'], r['kinds']['fwd']['shapes'])"; done
