PIPESIM_DBG_NOUPLOAD=1 python tools/diag_e2e.py 2>&1 | grep streamed | tail -2
PIPESIM_DBG_COPYONLY=1 python tools/diag_e2e.py 2>&1 | grep streamed | tail -2
