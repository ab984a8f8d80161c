"""One conv forward and dgrad launch per VGG shape (ncu target):
python tools/conv_fwd_probe.py 224:64:64 112:64:128"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2410_14312_b200 import kernels as K  # noqa: E402

n = 64
for spec in sys.argv[1:]:
    h, cin, cout = (int(v) for v in spec.split(":"))
    x = torch.randn(n, h, h, cin, device="cuda").relu().bfloat16()
    w = (torch.randn(cout, 9 * cin, device="cuda") * 0.02).bfloat16()
    b = torch.zeros(cout, device="cuda")
    y = torch.empty(n, h, h, cout, device="cuda", dtype=torch.bfloat16)
    K.conv_fwd(x, w, b, "relu", y)
    d = torch.empty_like(x)
    K.conv_bwd_dx(y, w, x, "relu", d)
    torch.cuda.synchronize()
