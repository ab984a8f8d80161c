import sys, pathlib, torch
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
from paper_2410_14312_b200 import kernels as K
m = 1024; n = k = 4096
dz = K.padded_bf16(m, k); dz.normal_(); xx = K.padded_bf16(m, n); xx.normal_()
w32 = torch.zeros(k, n, device="cuda"); w32b = torch.zeros(k, n, device="cuda"); w16 = K.padded_bf16(k, n)
def t(fn, reps=30):
    for _ in range(3): fn()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(reps): fn()
    e1.record(); e1.synchronize()
    return e0.elapsed_time(e1) * 1000 / reps
print("sgd+w16 out-of-place", round(t(lambda: K.linear_bwd_dw_sgd(dz, xx, w32, w32b, w16, 0.0)), 1))
print("sgd+w16 in-place    ", round(t(lambda: K.linear_bwd_dw_sgd(dz, xx, w32, w32, w16, 0.0)), 1))
print("sgd no w16          ", round(t(lambda: K.linear_bwd_dw_sgd(dz, xx, w32, w32b, None, 0.0)), 1))
big = torch.empty(256 * 1024 * 1024 // 4, device="cuda")
print("copy 168MB (rd 67MB wr 101MB)", round(t(lambda: w32b.copy_(w32)), 1), "us for 134MB fp32 copy")
