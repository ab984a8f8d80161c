mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_digest.py tests/test_gpu_multiproc.py -q -m gpu -x -p no:cacheprovider > gpurun_out/r2f_digest.log 2>&1; echo digest+ipc tests rc=$?; tail -3 gpurun_out/r2f_digest.log
for c in c1 c3; do timeout 600 tools/bin/dropin_bench $c 3 auto > gpurun_out/r2f_dropin_${c}_auto.json 2> gpurun_out/r2f_dropin_${c}_auto.err; echo dropin $c rc=$?; cat gpurun_out/r2f_dropin_${c}_auto.json; done
timeout 1500 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/r2f_pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/r2f_pytest.log
