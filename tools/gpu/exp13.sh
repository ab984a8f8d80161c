mkdir -p gpurun_out; o=gpurun_out/exp13.txt; : > $o
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x 2>&1 | tail -3 >> $o
PIPESIM_SPLITK=0 python tools/gemm_exp.py >> $o 2>&1
PIPESIM_SPLITK=0 PIPESIM_EPI=vec python tools/gemm_exp.py >> $o 2>&1
timeout 300 python -m pytest tests/test_gpu_pipeline.py -q -x 2>&1 | tail -2 >> $o
PIPESIM_SPLITK=0 timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$? >> $o; python -c "import json;d=json.load(open('gpurun_out/bench.json'));print(d['value'],d['ms_per_step'],d['e2e']['value'])" >> $o 2>&1
cat $o
