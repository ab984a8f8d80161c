"""Launch each layer-GEMM shape of the C3 workload a few times (for ncu)."""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
from paper_2410_14312_b200 import kernels as K

which = sys.argv[1] if len(sys.argv) > 1 else "all"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
torch.manual_seed(0)
m = 1024; n = k = 4096
if which in ("all", "fwd"):
    x = K.padded_bf16(128, k); x.normal_(); w = K.padded_bf16(n, k); w.normal_()
    b = torch.zeros(n, device="cuda"); y = K.padded_bf16(128, n)
    for _ in range(reps): K.linear_fwd(x, w, b, "relu", y16=y)
if which in ("all", "dgrad"):
    dz = K.padded_bf16(m, k); dz.normal_(); w = K.padded_bf16(k, n); w.normal_()
    xin = K.padded_bf16(m, n); xin.normal_(); d = K.padded_bf16(m, n)
    for _ in range(reps): K.linear_bwd_dx(dz, w, xin, "relu", d)
if which in ("all", "wgrad"):
    dz = K.padded_bf16(m, k); dz.normal_(); xx = K.padded_bf16(m, n); xx.normal_()
    w32 = torch.zeros(k, n, device="cuda"); w16 = K.padded_bf16(k, n)
    for _ in range(reps): K.linear_bwd_dw_sgd(dz, xx, w32, w32, w16, 0.0)
torch.cuda.synchronize()
print("done")
