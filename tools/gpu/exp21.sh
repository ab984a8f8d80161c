mkdir -p gpurun_out; o=gpurun_out/exp21.txt; : > $o
PIPESIM_SPLIT_FB=1 timeout 600 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_multiproc.py tests/test_gpu_verify.py tests/test_export.py -q -x 2>&1 | tail -3 >> $o
for v in 0 1; do
PIPESIM_SPLIT_FB=$v timeout 300 python bench.py --no-cpu-baseline > gpurun_out/b.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/b.json'));print('split_fb $v bench',d['value'],d['ms_per_step'], d['roofline']['in_step']['fwd'])" >> $o 2>&1
done
cat $o
