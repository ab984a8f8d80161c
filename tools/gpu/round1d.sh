mkdir -p gpurun_out
timeout 600 python tools/timeline.py --out-json gpurun_out/timeline_r1.json --trace gpurun_out/trace_r1.json > gpurun_out/timeline_r1.txt 2>&1; echo tl rc=$?; cat gpurun_out/timeline_r1.txt
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/b.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/b.json'));print('bench',d['value'],d['ms_per_step'],'e2e',d['e2e']['value'], d['other_configs'])"
