mkdir -p gpurun_out; o=gpurun_out/exp22.txt; : > $o
timeout 600 python -m pytest tests/test_gpu_pipeline.py -q -x -k "streamed or small or c1" 2>&1 | tail -3 >> $o
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/b.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/b.json'));print('bench',d['value'],d['ms_per_step'], 'e2e', d['e2e'])" >> $o 2>&1
cat $o
