# A/B with the order reversed (working tree first), to expose order/thermal bias
mkdir -p gpurun_out
for i in 1 2 3; do
PIPESIM_BENCH_VGG=0 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-dropin > gpurun_out/ab_new_$i.json 2>/dev/null
(cd ab_old && PIPESIM_SPLITK=0 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-dropin > ../gpurun_out/ab_old_$i.json 2>/dev/null)
done
for f in ab_new_1 ab_old_1 ab_new_2 ab_old_2 ab_new_3 ab_old_3; do python -c "
import json;d=json.load(open('gpurun_out/$f.json'));print('$f', round(d['value']), round(d['ms_per_step'],2), d['clocks']['sm_mhz'])"; done
