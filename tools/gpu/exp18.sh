mkdir -p gpurun_out; o=gpurun_out/exp18.txt; : > $o
PIPESIM_SPLITK=0 python tools/gemm_exp.py >> $o 2>&1
PIPESIM_SPLITK=0 timeout 300 python bench.py --no-cpu-baseline > gpurun_out/b.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/b.json'));print('bench',d['value'],d['ms_per_step'], d['roofline']['in_step'])" >> $o 2>&1
cat $o
