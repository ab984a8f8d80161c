"""Times our layer GEMMs on the benchmark shapes, graph-captured, cycling
through enough operand copies that every launch reads its weights from HBM
(as in the pipeline).  Env knobs select variants (PIPESIM_SPLITK,
PIPESIM_DBG_EPI, PIPESIM_EPI, PIPESIM_GEMM).  One JSON line; --cublas adds
torch.mm on the same shapes."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_14312_b200 import kernels as K

n = 4096
COPIES = 6  # 6 x 32 MiB weights > L2
cub = "--cublas" in sys.argv
res = {}
ws = [K.padded_bf16(n, n).normal_() for _ in range(COPIES)]
for m in (128, 256, 512, 1024):
    x = K.padded_bf16(m, n); x.normal_()
    b = torch.zeros(n, device="cuda"); y = K.padded_bf16(m, n)
    res[f"fwd{m}"] = K.graph_time_us([lambda w=w: K.linear_fwd(x, w, b, "relu", y16=y) for w in ws])
    if cub:
        res[f"cublas_fwd{m}"] = K.graph_time_us([lambda w=w: torch.mm(x, w.t()) for w in ws])
dz = K.padded_bf16(1024, n); dz.normal_()
xin = K.padded_bf16(1024, n); xin.normal_(); d = K.padded_bf16(1024, n)
res["dgrad"] = K.graph_time_us([lambda w=w: K.linear_bwd_dx(dz, w, xin, "relu", d) for w in ws])
if cub:
    res["cublas_dgrad"] = K.graph_time_us([lambda w=w: torch.mm(dz, w) for w in ws])
xx = K.padded_bf16(1024, n); xx.normal_()
w32s = [torch.zeros(n, n, device="cuda") for _ in range(2)]
w16 = K.padded_bf16(n, n)
res["wgrad32"] = K.graph_time_us([lambda w=w: K.linear_bwd_dw_sgd(dz, xx, w, w, w16, 0.0) for w in w32s])
his = [K.padded_bf16(n, n) for _ in range(2)]
los = [torch.zeros(n, n, dtype=torch.int16, device="cuda") for _ in range(2)]
res["wgrad"] = K.graph_time_us([lambda i=i: K.linear_bwd_dw_sgd_split(dz, xx, his[i], los[i], his[i], los[i], 0.0)
                                for i in range(2)])
if cub:
    res["cublas_wgrad"] = K.graph_time_us(lambda: torch.mm(dz.t(), xx))
env = {k: v for k, v in os.environ.items() if k.startswith("PIPESIM_")}
print(json.dumps({"env": env, **{k: round(v, 2) for k, v in res.items()}}))
