mkdir -p gpurun_out
./tools/tma_probe > gpurun_out/tma_probe.txt 2>&1; cat gpurun_out/tma_probe.txt
timeout 900 python tools/configs.py --out gpurun_out/configs_r1.json > gpurun_out/configs_r1.md 2> gpurun_out/configs_r1.err; echo configs rc=$?; cat gpurun_out/configs_r1.md; tail -3 gpurun_out/configs_r1.err
