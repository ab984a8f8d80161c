import sys, time, numpy as np, torch
sys.path.insert(0, "/root/repo")
from paper_2410_14312_b200 import pipesim as P
net = P.NetworkSpec([4096] * 17, ["relu"] * 15 + ["linear"], "softmax_cross_entropy")
W, N, B, M = 8, 8, 1024, 32
import os
s = P.Session(net, W, N, B, M, 0.05, "timeprest", use_graph=os.environ.get("NOGRAPH") is None)
s.load_params(P.init_network_params(net, 1))
x, lab = P.make_classification_task(M * B, 4096, 4096, seed=7, as_labels=True, dtype=np.float32)
xh = torch.from_numpy(x).pin_memory(); yh = torch.from_numpy(lab).pin_memory()
xb = torch.from_numpy(x).to(torch.bfloat16).pin_memory()
for name, xx, dt in (("f32", xh, "f32"), ("bf16", xb, "bf16")):
    for i in range(3):
        t = time.perf_counter()
        r = s.train_epoch_host(xx.data_ptr(), dt, yh.data_ptr(), "labels")
        print("streamed %s: wall ms %.2f device ms %.2f loss0 %.6f" % (name, 1000 * (time.perf_counter() - t), r["device_ms"], r["mini_loss"][0]))
s.upload(x, lab, y_labels=True)
for i in range(2):
    r = s.run_epoch(); print("resident device ms %.2f loss0 %.6f" % (r["device_ms"], r["mini_loss"][0]))
