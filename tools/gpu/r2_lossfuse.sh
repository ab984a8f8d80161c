timeout 900 python -m pytest tests -q -x -m gpu -p no:cacheprovider > gpurun_out/lf_pytest.log 2>&1; tail -1 gpurun_out/lf_pytest.log
python tools/c1_timeline.py 2>&1 | head -1
PIPESIM_LOSS_FUSE=0 python tools/c1_timeline.py 2>&1 | head -1
