mkdir -p gpurun_out
PIPESIM_SPLITK=0 timeout 400 ncu --set full --clock-control none --import-source on -k regex:gemm -c 3 -o gpurun_out/prof_r1c python tools/prof_gemm.py fwd256,dgrad,wgrad 1 > gpurun_out/prof_r1c.log 2>&1; echo ncu-full rc=$?
timeout 900 python tools/sweep.py --out gpurun_out/sweep_r1.json > gpurun_out/sweep_r1.md 2> gpurun_out/sweep_r1.err; echo sweep rc=$?; cat gpurun_out/sweep_r1.md | head -60; tail -3 gpurun_out/sweep_r1.err
