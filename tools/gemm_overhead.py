"""Fixed cost of one layer-GEMM launch: forward of 128 rows, N=4096, over
K = 64..4096 (PIPESIM_DBG_EPI=1 isolates the mainloop)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_14312_b200 import kernels as K
from tools.gemm_yardstick import timeit
out = {}
for n in (256, 4096):
    for k in (64, 256, 1024, 4096):
        x = K.padded_bf16(128, k); x.normal_(); w = K.padded_bf16(n, k); w.normal_()
        b = torch.zeros(n, device="cuda"); y = K.padded_bf16(128, n)
        out[f"n{n}_k{k}"] = round(timeit(lambda: K.linear_fwd(x, w, b, "relu", y16=y), 50), 2)
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("PIPESIM_")}, **out}))
