mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "linear_fwd" 2>&1 | tail -2
python tools/fwd_shapes.py
PIPESIM_FWD_FIX=0 python tools/fwd_shapes.py
PIPESIM_FWD_FIX=0 PIPESIM_SPLITK=0 python tools/fwd_shapes.py
PIPESIM_BN512=0 python tools/fwd_shapes.py
