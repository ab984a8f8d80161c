mkdir -p gpurun_out; o=gpurun_out/exp20.txt; : > $o
timeout 300 python -m pytest tests/test_export.py tests/test_gpu_multiproc.py -q -x 2>&1 | tail -2 >> $o
for d in 0 2 4 6 1; do PIPESIM_SPLITK=0 PIPESIM_DBG_EPI=$d python tools/gemm_exp.py >> $o 2>&1; done
cat $o
