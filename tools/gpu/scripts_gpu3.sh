timeout 300 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu3.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu3.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench rc=$?; tail -c 3000 gpurun_out/bench_default.json
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc=$?; cat gpurun_out/bench_ref.json
nproc; lscpu | grep "Model name"
