timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_conv.py tests/test_gpu_convnet.py -q -x -p no:cacheprovider 2>&1 | tail -1
PIPESIM_FWD_FIX=1 timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k linear_fwd 2>&1 | tail -1
PIPESIM_CONV_HALO=1 timeout 300 python -m pytest tests/test_gpu_conv.py -q -x -p no:cacheprovider 2>&1 | tail -1
bash tools/gpu/r2_ab_start.sh
