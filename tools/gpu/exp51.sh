mkdir -p gpurun_out; o=gpurun_out/exp51.txt; : > $o
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x 2>&1 | tail -3 >> $o
PIPESIM_SPLITK=0 python tools/gemm_exp.py >> $o 2>&1
for v in 0 4 2; do PIPESIM_DBG_EPI=$v PIPESIM_SPLITK=0 python tools/gemm_exp.py 2>&1 | sed "s/^/dbg=$v /" >> $o; done
cat $o
