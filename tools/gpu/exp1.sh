mkdir -p gpurun_out; o=gpurun_out/exp1.txt; : > $o
python tools/gemm_exp.py >> $o 2>&1
PIPESIM_DBG_EPI=1 python tools/gemm_exp.py >> $o 2>&1
PIPESIM_SPLITK=0 python tools/gemm_exp.py >> $o 2>&1
PIPESIM_SPLITK=0 PIPESIM_DBG_EPI=1 python tools/gemm_exp.py >> $o 2>&1
for s in 2 8; do PIPESIM_SPLITK=$s python tools/gemm_exp.py >> $o 2>&1; done
PIPESIM_SPLITK=0 PIPESIM_EPI=tile python tools/gemm_exp.py >> $o 2>&1
PIPESIM_SPLITK=0 PIPESIM_GEMM=single python tools/gemm_exp.py >> $o 2>&1
cat $o
