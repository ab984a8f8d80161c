mkdir -p gpurun_out; o=gpurun_out/exp3.txt; : > $o
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x 2>&1 | tail -2 >> $o
python tools/gemm_exp.py >> $o 2>&1
PIPESIM_DBG_EPI=1 python tools/gemm_exp.py >> $o 2>&1
PIPESIM_SPLITK=0 python tools/gemm_exp.py >> $o 2>&1
PIPESIM_SPLITK=2 python tools/gemm_exp.py >> $o 2>&1
python tools/gemm_overhead.py >> $o 2>&1
PIPESIM_DBG_EPI=1 python tools/gemm_overhead.py >> $o 2>&1
PIPESIM_DBG_EPI=1 PIPESIM_SPLITK=0 python tools/gemm_overhead.py >> $o 2>&1
cat $o
