python tools/diag_e2e.py 2>&1 | sed -n 2,6p
PIPESIM_H2D_SIDE=1 python tools/diag_e2e.py 2>&1 | sed -n 2,3p
timeout 600 python -m pytest tests -q -x -p no:cacheprovider -m gpu -k "e2e or host or stream or train_epoch" 2>&1 | tail -2
