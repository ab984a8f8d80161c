mkdir -p gpurun_out; o=gpurun_out/exp14.txt; : > $o
PIPESIM_SPLITK=0 PIPESIM_WG_BN=128 python tools/gemm_exp.py >> $o 2>&1
PIPESIM_SPLITK=0 PIPESIM_DBG_EPI=1 python tools/gemm_exp.py >> $o 2>&1
PIPESIM_SPLITK=0 PIPESIM_DBG_EPI=1 PIPESIM_WG_BN=128 python tools/gemm_exp.py >> $o 2>&1
cat $o
