mkdir -p gpurun_out
timeout 120 python tools/conv_kernel_diag.py halo 2>&1 | tail -5
timeout 300 python -m pytest tests/test_gpu_conv.py -q -x -p no:cacheprovider 2>&1 | tail -3
timeout 300 python tools/vgg_layers.py --out gpurun_out/vgg_layers3.json 2>&1 | head -3
