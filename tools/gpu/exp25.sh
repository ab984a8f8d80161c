mkdir -p gpurun_out; o=gpurun_out/exp25.txt; : > $o
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -2 >> $o
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/b.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/b.json'));print('bench',d['value'],d['ms_per_step'],'e2e',d['e2e']['value'])" >> $o 2>&1
cat $o
