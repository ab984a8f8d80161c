mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x > gpurun_out/kern.log 2>&1; echo kern rc=$?; tail -3 gpurun_out/kern.log
timeout 300 python -m pytest tests/test_gpu_pipeline.py -q -x > gpurun_out/pipe.log 2>&1; echo pipe rc=$?; tail -3 gpurun_out/pipe.log
python tools/gemm_yardstick.py > gpurun_out/yard1.txt 2>&1; cat gpurun_out/yard1.txt
PIPESIM_SPLITK=0 python tools/gemm_yardstick.py > gpurun_out/yard1_nosplit.txt 2>&1; head -4 gpurun_out/yard1_nosplit.txt
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?; python -c "import json;d=json.load(open('gpurun_out/bench.json'));print(d['value'],d['ms_per_step'],d['e2e']['value'])"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm -c 4 -o gpurun_out/prof_fd python tools/prof_gemm.py fwd128,fwd1024,dgrad 1 > gpurun_out/prof_fd.log 2>&1; echo ncu rc=$?
