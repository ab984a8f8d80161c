mkdir -p gpurun_out
python tools/conv_kernel_diag.py 2>&1 | tail -9
timeout 600 python -m pytest tests/test_gpu_conv.py tests/test_gpu_convnet.py -x -q -p no:cacheprovider 2>&1 | tail -3
timeout 600 python tools/vgg_layers.py --out gpurun_out/vgg_layers2.json 2>&1 | tail -12
