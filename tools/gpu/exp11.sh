mkdir -p gpurun_out; o=gpurun_out/exp11.txt; : > $o
for p in 74 56 48 37 24 16; do PIPESIM_SPLITK=0 PIPESIM_MAXPAIRS=$p python tools/gemm_exp.py >> $o 2>&1; done
cat $o
