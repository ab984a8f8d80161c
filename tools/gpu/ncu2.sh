mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm -c 1 -o gpurun_out/prof_wg python tools/prof_gemm.py wgrad 1 > gpurun_out/prof_wg.log 2>&1; echo ncu rc=$?
