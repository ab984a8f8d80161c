mkdir -p gpurun_out; o=gpurun_out/exp27.txt; : > $o
for r in 1 2; do for v in 0 3 1; do
PIPESIM_PRIO=$v timeout 300 python bench.py --no-cpu-baseline --steps 8 > gpurun_out/b.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/b.json'));print('prio $v bench',d['value'],d['ms_per_step'])" >> $o 2>&1
done; done
cat $o
