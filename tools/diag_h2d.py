"""Why the f32-input e2e epoch is slower than bf16: raw H2D bandwidth, and the
resident epoch with an unrelated concurrent H2D copy of the same bytes."""
import sys, time, numpy as np, torch
sys.path.insert(0, ".")
from paper_2410_14312_b200 import pipesim as P
net = P.NetworkSpec([4096] * 17, ["relu"] * 15 + ["linear"], "softmax_cross_entropy")
W, N, B, M = 8, 8, 1024, 32
s = P.Session(net, W, N, B, M, 0.05, "timeprest")
s.load_params(P.init_network_params(net, 1))
x, lab = P.make_classification_task(M * B, 4096, 4096, seed=7, as_labels=True, dtype=np.float32)
s.upload(x, lab, y_labels=True)
xh = torch.from_numpy(x).pin_memory()
dev = torch.empty(xh.numel(), dtype=torch.float32, device="cuda")
st = torch.cuda.Stream()
for _ in range(3):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(st); dev.copy_(xh.view(-1), non_blocking=True) if False else None
    with torch.cuda.stream(st):
        e0.record(); dev.copy_(xh.view(-1), non_blocking=True); e1.record()
    torch.cuda.synchronize()
    print("H2D %d MB: %.2f ms = %.1f GB/s" % (xh.numel() * 4 >> 20, e0.elapsed_time(e1), xh.numel() * 4 / e0.elapsed_time(e1) / 1e6))
for _ in range(2):
    r = s.run_epoch(); print("resident alone %.2f" % r["device_ms"])
for _ in range(3):
    with torch.cuda.stream(st):
        dev.copy_(xh.view(-1), non_blocking=True)
    r = s.run_epoch(); torch.cuda.synchronize(); print("resident + concurrent H2D %.2f" % r["device_ms"])
xb = torch.from_numpy(x).to(torch.bfloat16).pin_memory()
devb = torch.empty(xb.numel(), dtype=torch.bfloat16, device="cuda")
for _ in range(2):
    with torch.cuda.stream(st):
        devb.copy_(xb.view(-1), non_blocking=True)
    r = s.run_epoch(); torch.cuda.synchronize(); print("resident + concurrent bf16 H2D %.2f" % r["device_ms"])
