"""Per-mini-batch graph time of a small-network config (C1 / C2 shapes):
python tools/c_timing.py --W 1 --mode sequential [--M 12]"""
import argparse
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2410_14312_b200 import pipesim as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--W", type=int, default=2)
ap.add_argument("--N", type=int, default=4)
ap.add_argument("--B", type=int, default=256)
ap.add_argument("--M", type=int, default=12)
ap.add_argument("--mode", default="timeprest")
a = ap.parse_args()
net = P.NetworkSpec([784, 512, 256, 10], ["relu", "relu", "linear"], "softmax_cross_entropy")
s = P.Session(net, a.W, a.N, a.B, a.M, 0.05, a.mode)
s.load_params(P.init_network_params(net, 1))
x, lab = P.make_classification_task(a.M * a.B, 784, 10, seed=7, as_labels=True, dtype=np.float32)
s.upload(x, lab, y_labels=True)
for _ in range(3):
    s.run_epoch()
ms = [s.run_epoch()["device_ms"] for _ in range(9)]
print(f"W={a.W} {a.mode} us/mini {1000 * np.median(ms) / a.M:.2f} kernels/epoch {s.kernels_per_epoch}")
