mkdir -p gpurun_out; o=gpurun_out/exp9.txt; : > $o
for d in 0 1 2 4 8 12 14; do PIPESIM_SPLITK=0 PIPESIM_DBG_EPI=$d python tools/gemm_exp.py >> $o 2>&1; done
PIPESIM_SPLITK=0 PIPESIM_EPI=rows python tools/gemm_exp.py >> $o 2>&1
cat $o
