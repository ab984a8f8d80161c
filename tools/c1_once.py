"""One C1 epoch (784-512-256-10, W=2, N=4, B=256, M=12), graph: ncu target."""
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_2410_14312_b200 import pipesim as P
net = P.NetworkSpec([784, 512, 256, 10], ["relu", "relu", "linear"], "softmax_cross_entropy")
s = P.Session(net, 2, 4, 256, 12, 0.05, "timeprest")
s.load_params(P.init_network_params(net, 1))
x, lab = P.make_classification_task(12 * 256, 784, 10, seed=7, as_labels=True, dtype=np.float32)
s.upload(x, lab, y_labels=True)
print(s.run_epoch()["device_ms"])
