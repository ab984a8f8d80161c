export PIPESIM_SESSION_SPLIT=0
CFG=64,M,64,128 TAG=unpooled python tools/conv_determinism.py 1,1,1,2 2>&1 | tail -3
FCL=3 TAG=fc3 python tools/conv_determinism.py 1,1,1,3 2>&1 | tail -3
FCL=3 TAG=fc3b python tools/conv_determinism.py 3,1,2 2>&1 | tail -3
