"""C1 (784-512-256-10, W=2, N=4, B=256) per-node device timeline of one
epoch: where the per-mini-batch time goes.  GPU box: python tools/c1_timeline.py"""
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_2410_14312_b200 import pipesim as P
widths, acts = [784, 512, 256, 10], ["relu", "relu", "linear"]
net = P.NetworkSpec(widths, acts, "softmax_cross_entropy")
W, N, B, M = 2, 4, 256, 32
s = P.Session(net, W, N, B, M, 0.05, "timeprest")
s.load_params(P.init_network_params(net, 1))
x, lab = P.make_classification_task(M * B, 784, 10, seed=7, as_labels=True, dtype=np.float32)
s.upload(x, lab, y_labels=True)
for _ in range(3):
    r = s.run_epoch()
ms = [s.run_epoch()["device_ms"] for _ in range(5)]
print("graph epoch ms", np.median(ms), "us/mini", 1000 * np.median(ms) / M, "kernels/epoch", s.kernels_per_epoch)
pr = s.profile_epoch()["profile"]
print("profile makespan", pr["makespan_ms"], "busy", pr["busy_ms"])
nodes = sorted(pr["nodes"], key=lambda n: n["start_ms"])
for n in nodes[:40]:
    print("%6.1f %6.1f us  stage %d %s mini %d micro %s" % (1000 * n["start_ms"], 1000 * (n["end_ms"] - n["start_ms"]), n["stage"], "F" if n["fwd"] else "B", n["mini"], n["micro"]))
