timeout 300 python tools/vgg_layers.py 2>&1 | head -1 | cut -c1-200
PIPESIM_DBG_EPI=16 timeout 300 python tools/vgg_layers.py 2>&1 | head -1 | cut -c1-200
PIPESIM_CONV_HALO=0 timeout 300 python tools/vgg_layers.py 2>&1 | head -1 | cut -c1-200
