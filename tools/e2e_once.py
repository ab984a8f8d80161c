"""One streamed (host-input) epoch of the bench workload (ncu target)."""
import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2410_14312_b200 import pipesim as P
net = P.NetworkSpec([4096] * 17, ["relu"] * 15 + ["linear"], "softmax_cross_entropy")
W, N, B, M = 8, 8, 1024, int(sys.argv[1]) if len(sys.argv) > 1 else 4
s = P.Session(net, W, N, B, M, 0.05, "timeprest")
s.load_params(P.init_network_params(net, 1))
x, lab = P.make_classification_task(M * B, 4096, 4096, seed=7, as_labels=True, dtype=np.float32)
xh = torch.from_numpy(x).pin_memory(); yh = torch.from_numpy(lab).pin_memory()
r = s.train_epoch_host(xh.data_ptr(), "f32", yh.data_ptr(), "labels")
print(r["device_ms"])
