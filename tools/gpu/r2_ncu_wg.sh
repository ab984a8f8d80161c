mkdir -p gpurun_out
ncu --set full --clock-control none -k regex:gemm -c 2 -o gpurun_out/ncu_convwg -f python tools/conv_wgrad_probe.py 28:512:512 224:64:64 > gpurun_out/ncu_convwg.log 2>&1
tail -3 gpurun_out/ncu_convwg.log
