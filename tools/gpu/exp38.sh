# wgrad SGD epilogue decomposition: skip loads (2), stores (4), both (6), all (1)
mkdir -p gpurun_out; o=gpurun_out/exp38.txt; : > $o
for v in 0 1 2 4 6; do PIPESIM_DBG_EPI=$v PIPESIM_SPLITK=0 python tools/gemm_exp.py >> $o 2>&1; done
cat $o
