"""One VGG-16 layer-1 conv forward and dgrad (64 images, 224x224, 64 -> 64
channels) for an ncu capture: python tools/conv_dgrad_probe.py"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2410_14312_b200 import kernels as K  # noqa: E402

n, h, w, cin, cout = 64, 224, 224, 64, 64
x = torch.randn(n, h, w, cin, device="cuda").relu().bfloat16()
wt = (torch.randn(cout, 9 * cin, device="cuda") * 0.02).bfloat16()
b = torch.zeros(cout, device="cuda")
y = torch.empty(n, h, w, cout, device="cuda", dtype=torch.bfloat16)
dz = torch.randn(n, h, w, cout, device="cuda").bfloat16()
d = torch.empty_like(x)
for _ in range(2):
    K.conv_fwd(x, wt, b, "relu", y)
    K.conv_bwd_dx(dz, wt, x, "relu", d)
torch.cuda.synchronize()
print("ok")
