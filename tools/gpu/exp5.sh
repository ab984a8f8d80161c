mkdir -p gpurun_out; o=gpurun_out/exp5.txt; : > $o
python tools/gemm_exp.py >> $o 2>&1
PIPESIM_DBG_EPI=1 python tools/gemm_exp.py >> $o 2>&1
PIPESIM_SPLITK=2 python tools/gemm_exp.py >> $o 2>&1
PIPESIM_SPLITK=0 python tools/gemm_exp.py >> $o 2>&1
cat $o
