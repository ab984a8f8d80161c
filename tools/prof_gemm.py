"""Launch layer-GEMM shapes of the C3 workload a few times (for ncu).

  python tools/prof_gemm.py <which[,which...]|all> [reps]
  which: fwd128 fwd256 fwd1024 dgrad wgrad   (fwd = fwd128)
"""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
from paper_2410_14312_b200 import kernels as K

arg = sys.argv[1] if len(sys.argv) > 1 else "all"
which = {"fwd128", "dgrad", "wgrad"} if arg == "all" else set(arg.replace("fwd,", "fwd128,").split(","))
if arg == "fwd":
    which = {"fwd128"}
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
torch.manual_seed(0)
m = 1024; n = k = 4096
for rows in (128, 256, 512, 1024):
    if f"fwd{rows}" in which:
        x = K.padded_bf16(rows, k); x.normal_(); w = K.padded_bf16(n, k); w.normal_()
        b = torch.zeros(n, device="cuda"); y = K.padded_bf16(rows, n)
        for _ in range(reps): K.linear_fwd(x, w, b, "relu", y16=y)
if "dgrad" in which:
    dz = K.padded_bf16(m, k); dz.normal_(); w = K.padded_bf16(k, n); w.normal_()
    xin = K.padded_bf16(m, n); xin.normal_(); d = K.padded_bf16(m, n)
    for _ in range(reps): K.linear_bwd_dx(dz, w, xin, "relu", d)
if "wgrad" in which:  # split fp32 masters, as in the session
    dz = K.padded_bf16(m, k); dz.normal_(); xx = K.padded_bf16(m, n); xx.normal_()
    hi = K.padded_bf16(k, n); lo = torch.zeros(k, n, dtype=torch.int16, device="cuda")
    for _ in range(reps): K.linear_bwd_dw_sgd_split(dz, xx, hi, lo, hi, lo, 0.0)
if "wgrad32" in which:  # fp32 masters + bf16 copy
    dz = K.padded_bf16(m, k); dz.normal_(); xx = K.padded_bf16(m, n); xx.normal_()
    w32 = torch.zeros(k, n, device="cuda"); w16 = K.padded_bf16(k, n)
    for _ in range(reps): K.linear_bwd_dw_sgd(dz, xx, w32, w32, w16, 0.0)
torch.cuda.synchronize()
print("done")
