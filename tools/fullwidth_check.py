"""Full-width precision check: the bf16 tensor-core session against the fp32
FFMA verify session at the benchmark's width (4096, B=1024, N=8; 4 layers on
2 stages, M=3), printing the relative loss / weight / weight-delta errors
(tests/test_gpu_verify.py::test_full_width_bf16_against_fp32_verify asserts
them).   python tools/fullwidth_check.py"""
import numpy as np, sys
sys.path.insert(0, '.')
from paper_2410_14312_b200 import pipesim as P
net = P.NetworkSpec([4096] * 5, ["relu"] * 3 + ["linear"], "softmax_cross_entropy")
W, N, B, M = 2, 8, 1024, 3
p0 = P.init_network_params(net, 1)
x, lab = P.make_classification_task(M * B, 4096, 4096, seed=7, as_labels=True, dtype=np.float32)
res = {}
for prec in ("bf16", "fp32"):
    s = P.Session(net, W, N, B, M, 0.05, "timeprest", precision=prec)
    s.load_params(p0); s.upload(x, lab, y_labels=True)
    r = s.run_epoch()
    res[prec] = (np.asarray(r["mini_loss"]), s.read_params()); s.close()
(l16, w16), (l32, w32) = res["bf16"], res["fp32"]
print("loss", l16, l32, np.abs(l16 - l32).max() / np.abs(l32).max())
print("w", np.linalg.norm(w16 - w32) / np.linalg.norm(w32))
print("dw", np.linalg.norm((w16 - p0) - (w32 - p0)) / np.linalg.norm(w32 - p0))
