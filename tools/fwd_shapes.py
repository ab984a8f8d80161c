"""Alone timings of the 4096 x 4096 forward GEMM at the pipeline's row counts
(CUDA graph, 6 rotated weight copies so weights stream from HBM), TFLOP/s
and fraction of the burst bf16 peak.  PIPESIM_FWD_FIX / PIPESIM_SPLITK /
PIPESIM_BN512 select the variant.  GPU box: python tools/fwd_shapes.py"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_14312_b200 import kernels as K  # noqa: E402

BURST = 1634.8


def main():
    rows_list = [int(v) for v in sys.argv[1:]] or [128, 256, 512, 768, 1024]
    n = 4096
    ws = []
    for _ in range(6):
        w = K.padded_bf16(n, n)
        w.copy_((torch.rand(n, n, device="cuda") * 2 - 1) / 64)
        ws.append(w)
    b = torch.zeros(n, device="cuda")
    out = {}
    for rows in rows_list:
        x = K.padded_bf16(rows, n)
        x.copy_(torch.rand(rows, n, device="cuda"))
        y = K.padded_bf16(rows, n)
        fns = [lambda w=w: K.linear_fwd(x, w, b, "relu", y16=y) for w in ws]
        us = K.graph_time_us(fns, reps=60)
        tf = 2.0 * rows * n * n / us / 1e6
        out[rows] = {"us": round(us, 2), "tflops": round(tf, 1), "frac": round(tf / BURST, 3)}
    env = {k: os.environ.get(k) for k in ("PIPESIM_FWD_FIX", "PIPESIM_SPLITK", "PIPESIM_BN512")}
    print(json.dumps({"env": env, "shapes": out}))


if __name__ == "__main__":
    main()
