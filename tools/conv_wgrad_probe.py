"""One conv wgrad launch per VGG shape given (ncu target):
python tools/conv_wgrad_probe.py 28:512:512 224:64:64"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2410_14312_b200 import kernels as K  # noqa: E402

n = 64
for spec in sys.argv[1:]:
    h, cin, cout = (int(v) for v in spec.split(":"))
    x = torch.randn(n, h, h, cin, device="cuda").relu().bfloat16()
    dz = torch.randn(n, h, h, cout, device="cuda").bfloat16()
    w0 = torch.zeros(cout, 9 * cin, device="cuda")
    w1 = torch.empty_like(w0)
    K.conv_bwd_dw_sgd(dz, x, w0, w1, None, 0.01)
    torch.cuda.synchronize()
