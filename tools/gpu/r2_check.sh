# Round-2 validation: the full -m gpu suite, smoke, default bench, reference arm.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2_gpu.txt
timeout 1500 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/r2_pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/r2_pytest.log
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/r2_smoke.log
timeout 900 python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo bench rc=$?
cat gpurun_out/r2_bench.json | head -c 3000
