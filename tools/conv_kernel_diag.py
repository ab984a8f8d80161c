"""Relative error of the conv GEMM kernels against float64 torch on the same
bf16 operands, per shape (GPU box: python tools/conv_kernel_diag.py)."""
import sys

import torch
import torch.nn.functional as F

sys.path.insert(0, ".")
from paper_2410_14312_b200 import kernels as K  # noqa: E402


def w_krsc(w):
    return w.permute(0, 2, 3, 1).reshape(w.shape[0], -1).contiguous()


def rel(a, b):
    return ((a.double() - b.double()).norm() / b.double().norm()).item()


def main():
    shapes = [(8, 8, 8, 64, 64), (8, 4, 4, 64, 128), (2, 8, 8, 64, 64), (1, 8, 8, 64, 64),
              (4, 16, 16, 64, 64), (3, 14, 14, 64, 128), (2, 7, 9, 128, 256), (8, 2, 2, 128, 128),
              (1, 3, 112, 64, 64), (2, 5, 224, 64, 128), (1, 12, 112, 128, 64), (4, 224, 224, 64, 64)]
    for n, h, w, cin, cout in (shapes if len(sys.argv) < 2 else shapes[-4:]):
        torch.manual_seed(0)
        x = torch.randn(n, h, w, cin, device="cuda").relu().bfloat16()
        wt = (torch.randn(cout, cin, 3, 3, device="cuda") / (3 * cin ** 0.5)).bfloat16()
        dz = torch.randn(n, h, w, cout, device="cuda").bfloat16()
        b = torch.zeros(cout, device="cuda")
        xn, wn, dzn = (t.double().permute(0, 3, 1, 2) if t.dim() == 4 and t is not wt else t
                       for t in (x, wt, dz))
        # forward
        y = torch.empty(n, h, w, cout, device="cuda", dtype=torch.bfloat16)
        K.conv_fwd(x, w_krsc(wt), b, "linear", y)
        ref = F.conv2d(x.double().permute(0, 3, 1, 2), wt.double(), padding=1).permute(0, 2, 3, 1)
        e_f = rel(y, ref)
        # dgrad (linear gate: xin > 0 gate would mask; use relu'd x with act linear)
        d = torch.empty(n, h, w, cin, device="cuda", dtype=torch.bfloat16)
        K.conv_bwd_dx(dz, w_krsc(wt), x, "linear", d)
        ref = torch.nn.grad.conv2d_input((n, cin, h, w), wt.double(),
                                         dz.double().permute(0, 3, 1, 2), padding=1)
        e_d = rel(d, ref.permute(0, 2, 3, 1))
        # wgrad
        w0 = torch.zeros(cout, 9 * cin, device="cuda")
        w1 = torch.empty_like(w0)
        K.conv_bwd_dw_sgd(dz, x, w0, w1, None, 1.0)
        g = torch.nn.grad.conv2d_weight(x.double().permute(0, 3, 1, 2), (cout, cin, 3, 3),
                                        dz.double().permute(0, 3, 1, 2), padding=1)
        e_w = rel(-w1, w_krsc(g))
        print(f"n={n} h={h} w={w} cin={cin} cout={cout}: fwd {e_f:.2e} dgrad {e_d:.2e} "
              f"wgrad {e_w:.2e}")


if __name__ == "__main__":
    main()
