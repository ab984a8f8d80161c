mkdir -p gpurun_out; o=gpurun_out/exp8.txt; : > $o
PIPESIM_SPLITK=0 python tools/gemm_exp.py >> $o 2>&1
PIPESIM_SPLITK=0 PIPESIM_EPI=rows python tools/gemm_exp.py >> $o 2>&1
cat $o
