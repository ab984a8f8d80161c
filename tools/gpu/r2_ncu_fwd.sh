mkdir -p gpurun_out
ncu --set full --clock-control none -k regex:gemm -c 4 -o gpurun_out/ncu_convfwd -f python tools/conv_fwd_probe.py 224:64:64 28:512:512 > gpurun_out/ncu_convfwd.log 2>&1
tail -2 gpurun_out/ncu_convfwd.log
