mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm -c 3 -o gpurun_out/prof_e python tools/prof_gemm.py fwd128,dgrad,wgrad 1 > gpurun_out/prof_e.log 2>&1; echo ncu rc=$?
python tools/gemm_exp.py > gpurun_out/exp7.txt 2>&1; cat gpurun_out/exp7.txt
