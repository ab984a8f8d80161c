"""Per-layer kernel timings of VGG-16's conv layers alone (graph-captured,
CUDA events): implicit-GEMM forward, dgrad and wgrad (+ reduce-SGD) at a
given image count, TFLOP/s and the fraction of the burst bf16 peak, plus
the pooling / im2col kernels' GB/s.  GPU box: python tools/vgg_layers.py"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_14312_b200 import convnet as CN  # noqa: E402
from paper_2410_14312_b200 import kernels as K  # noqa: E402

BURST = 1634.8
HBM = 6515.1


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=64)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    n = args.n
    rows = []
    for i, l in enumerate(CN.vgg16().layers):
        if l.kind != "conv" or l.in_ % 64:
            continue
        h, w, cin, cout = l.h, l.w, l.in_, l.out
        x = torch.randn(n, h, w, cin, device="cuda").relu().bfloat16()
        wt = (torch.randn(cout, 9 * cin, device="cuda") * 0.02).bfloat16()
        b = torch.zeros(cout, device="cuda")
        y = torch.empty(n, h, w, cout, device="cuda", dtype=torch.bfloat16)
        dz = torch.randn(n, h, w, cout, device="cuda").bfloat16()
        d = torch.empty_like(x)
        w0 = torch.zeros(cout, 9 * cin, device="cuda")
        w1 = torch.empty_like(w0)
        w16 = torch.empty(cout, 9 * cin, device="cuda", dtype=torch.bfloat16)
        fl = 2.0 * n * h * w * cout * 9 * cin
        t_f = K.graph_time_us(lambda: K.conv_fwd(x, wt, b, "relu", y), reps=20)
        t_d = K.graph_time_us(lambda: K.conv_bwd_dx(dz, wt, x, "relu", d), reps=20)
        t_w = K.graph_time_us(lambda: K.conv_bwd_dw_sgd(dz, x, w0, w1, w16, 0.01), reps=20)
        r = {"layer": i, "h": h, "cin": cin, "cout": cout, "n": n, "gflop": fl / 1e9,
             "fwd_us": t_f, "dgrad_us": t_d, "wgrad_us": t_w,
             "fwd_frac": fl / t_f / 1e6 / BURST, "dgrad_frac": fl / t_d / 1e6 / BURST,
             "wgrad_frac": fl / t_w / 1e6 / BURST}
        if l.pool:
            yp = torch.empty(n, h // 2, w // 2, cout, device="cuda", dtype=torch.bfloat16)
            t_p = K.graph_time_us(lambda: K.maxpool2_fwd(y, yp), reps=20)
            gp = torch.empty_like(yp)
            dp = torch.empty_like(y)
            t_pb = K.graph_time_us(lambda: K.maxpool2_bwd(gp, y, yp, dp), reps=20)
            by = y.numel() * 2 * 1.25
            r.update(pool_fwd_us=t_p, pool_fwd_gbs=by / t_p / 1e3, pool_bwd_us=t_pb,
                     pool_bwd_gbs=(y.numel() * 4 + yp.numel() * 4) / t_pb / 1e3)
        print(json.dumps({k: (round(v, 3) if isinstance(v, float) else v) for k, v in r.items()}),
              flush=True)
        rows.append(r)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
