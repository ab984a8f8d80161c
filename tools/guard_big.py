"""PIPESIM_GUARD=1 over the benchmark configurations (one epoch each)."""
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_2410_14312_b200 import convnet as CN
from paper_2410_14312_b200 import pipesim as P
net = CN.vgg16()
x, lab = CN.synthetic_images(4 * 64, net, seed=7)
for W in (4, 8):
    s = P.Session(net, W, 4, 64, 4, 1e-4)
    s.load_params(CN.init_params(net, 1))
    s.upload(x, lab, y_labels=True)
    s.run_epoch()
    s.close()
    print("vgg16 W", W, "guards intact")
net = P.NetworkSpec([4096] * 17, ["relu"] * 15 + ["linear"], "softmax_cross_entropy")
x, lab = P.make_classification_task(8 * 1024, 4096, 4096, seed=7, as_labels=True, dtype=np.float32)
for W, mode in ((8, "timeprest"), (8, "pipedream"), (2, "timeprest")):
    s = P.Session(net, W, 8, 1024, 8, 0.05, mode=mode)
    s.load_params(P.init_network_params(net, 1))
    s.upload(x, lab, y_labels=True)
    s.run_epoch()
    s.close()
    print("mlp16x4096 W", W, mode, "guards intact")
