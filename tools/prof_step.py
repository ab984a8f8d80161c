"""One small pipeline session epoch (C3 shapes, M mini-batches) for ncu launch lists."""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2410_14312_b200 import pipesim as P
M = int(sys.argv[1]) if len(sys.argv) > 1 else 2
graph = (sys.argv[2] != "eager") if len(sys.argv) > 2 else True
net = P.NetworkSpec([4096] * 17, ["relu"] * 15 + ["linear"], "softmax_cross_entropy")
s = P.Session(net, 8, 8, 1024, M, 0.05, "timeprest", use_graph=graph)
s.load_params(P.init_network_params(net, 1))
x, lab = P.make_classification_task(M * 1024, 4096, 4096, seed=7, as_labels=True, dtype=np.float32)
s.upload(x, lab, y_labels=True)
for _ in range(2):
    r = s.run_epoch()
print("epoch ms", r["device_ms"], "kernels/epoch", s.kernels_per_epoch)
