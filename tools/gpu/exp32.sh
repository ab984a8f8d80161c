mkdir -p gpurun_out; o=gpurun_out/exp32.txt; : > $o
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x 2>&1 | tail -1 >> $o
PIPESIM_SPLITK=0 python tools/gemm_exp.py >> $o 2>&1
for r in 1 2; do timeout 300 python bench.py --no-cpu-baseline --steps 8 > gpurun_out/b.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/b.json'));print('bench',d['value'],d['ms_per_step'],'e2e',d['e2e']['value'])" >> $o 2>&1; done
cat $o
