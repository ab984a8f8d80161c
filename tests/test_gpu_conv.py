"""Conv-stage kernels of the VGG-style pipeline (BASELINE configs[3]) against
a plain PyTorch fp32 reference of the same op on the same bf16-rounded
operands: implicit-GEMM 3x3 conv forward / dgrad / wgrad+SGD (tcgen05 with
im2col TMA operands), 2x2 max pooling and the network-input im2col.  The
reference has no convolution, so torch is the oracle here."""
import pytest
import torch
import torch.nn.functional as F

pytestmark = pytest.mark.gpu


def _k():
    from paper_2410_14312_b200 import kernels as K
    return K


def _w_krsc(w):  # torch [cout, cin, 3, 3] -> [cout, 9 * cin] tap-major
    cout, cin = w.shape[:2]
    return w.permute(0, 2, 3, 1).reshape(cout, 9 * cin)


def _nchw(x):
    return x.permute(0, 3, 1, 2)


SHAPES = [(2, 8, 8, 64, 64), (3, 14, 14, 64, 128), (2, 7, 9, 128, 256), (4, 28, 28, 64, 64),
          (1, 56, 56, 128, 128),
          # image widths 112 / 224 (the opt-in halo strips, PIPESIM_CONV_HALO=1:
          # an odd strip count, two strips per image row, two patches per tile)
          (1, 3, 112, 64, 64), (2, 5, 224, 64, 128), (1, 12, 112, 128, 64)]


@pytest.mark.parametrize("n,h,w,cin,cout", SHAPES)
@pytest.mark.parametrize("act", ["relu", "linear"])
def test_conv_fwd(n, h, w, cin, cout, act):
    K = _k()
    torch.manual_seed(0)
    x = torch.randn(n, h, w, cin, device="cuda").bfloat16()
    wt = (torch.randn(cout, cin, 3, 3, device="cuda") / (3 * cin ** 0.5)).bfloat16()
    b = torch.randn(cout, device="cuda") * 0.1
    y = torch.empty(n, h, w, cout, device="cuda", dtype=torch.bfloat16)
    K.conv_fwd(x, _w_krsc(wt).contiguous(), b, act, y)
    ref = F.conv2d(_nchw(x.float()), wt.float(), b, padding=1).permute(0, 2, 3, 1)
    if act == "relu":
        ref = ref.relu()
    err = (y.float() - ref).abs().max().item()
    assert err <= 2e-2 * ref.abs().max().item() + 1e-2, err


@pytest.mark.parametrize("n,h,w,cin,cout", SHAPES)
def test_conv_bwd_dx(n, h, w, cin, cout):
    K = _k()
    torch.manual_seed(1)
    dz = torch.randn(n, h, w, cout, device="cuda").bfloat16()
    wt = (torch.randn(cout, cin, 3, 3, device="cuda") / (3 * cin ** 0.5)).bfloat16()
    xin = torch.randn(n, h, w, cin, device="cuda").relu().bfloat16()
    d = torch.empty(n, h, w, cin, device="cuda", dtype=torch.bfloat16)
    K.conv_bwd_dx(dz, _w_krsc(wt).contiguous(), xin, "relu", d)
    ref = torch.nn.grad.conv2d_input((n, cin, h, w), wt.float(), _nchw(dz.float()), padding=1)
    ref = ref.permute(0, 2, 3, 1) * (xin.float() > 0)
    err = (d.float() - ref).abs().max().item()
    assert err <= 2e-2 * ref.abs().max().item() + 1e-2, err


@pytest.mark.parametrize("n,h,w,cin,cout", SHAPES)
def test_conv_bwd_dw_sgd(n, h, w, cin, cout):
    K = _k()
    torch.manual_seed(2)
    dz = torch.randn(n, h, w, cout, device="cuda").bfloat16()
    x = torch.randn(n, h, w, cin, device="cuda").bfloat16()
    w0 = torch.randn(cout, 9 * cin, device="cuda")
    w1 = torch.empty_like(w0)
    w16 = torch.empty(cout, 9 * cin, device="cuda", dtype=torch.bfloat16)
    lr = 0.01
    K.conv_bwd_dw_sgd(dz, x, w0, w1, w16, lr)
    g = torch.nn.grad.conv2d_weight(_nchw(x.float()), (cout, cin, 3, 3), _nchw(dz.float()),
                                    padding=1)
    ref = w0 - lr * _w_krsc(g)
    err = (w1 - ref).abs().max().item()
    assert err <= 1e-4 * g.abs().max().item() * lr * 100 + 1e-5, err
    assert torch.equal(w16, w1.bfloat16())
    # deterministic: the partial slabs are reduced in split order
    w2 = torch.empty_like(w0)
    K.conv_bwd_dw_sgd(dz, x, w0, w2, None, lr)
    assert torch.equal(w1, w2)


@pytest.mark.parametrize("n,h,w,c", [(2, 8, 8, 64), (3, 14, 6, 128), (1, 224, 224, 64)])
def test_maxpool2(n, h, w, c):
    K = _k()
    torch.manual_seed(3)
    x = torch.randn(n, h, w, c, device="cuda").relu().bfloat16()
    y = torch.empty(n, h // 2, w // 2, c, device="cuda", dtype=torch.bfloat16)
    K.maxpool2_fwd(x, y)
    ref = F.max_pool2d(_nchw(x.float()), 2).permute(0, 2, 3, 1)
    assert torch.equal(y.float(), ref)
    g = torch.randn_like(y.float()).bfloat16()
    d = torch.empty_like(x)
    K.maxpool2_bwd(g, x, y, d)
    # first maximum of each window (row-major window order) takes the gradient
    xw = x.float().reshape(n, h // 2, 2, w // 2, 2, c).permute(0, 1, 3, 5, 2, 4)
    xw = xw.reshape(n, h // 2, w // 2, c, 4)
    first = (xw == y.float().unsqueeze(-1)).float().cumsum(-1).eq(1) & (xw == y.float().unsqueeze(-1))
    want = (first.float() * g.float().unsqueeze(-1)).reshape(n, h // 2, w // 2, c, 2, 2)
    want = want.permute(0, 1, 4, 2, 5, 3).reshape(n, h, w, c)
    assert torch.equal(d.float(), want)


def test_im2col_first():
    K = _k()
    torch.manual_seed(4)
    n, h, w, c = 2, 9, 7, 3
    x = torch.randn(n, h, w, c, device="cuda").bfloat16()
    out = torch.full((n * h * w, 32), 7.0, device="cuda", dtype=torch.bfloat16)
    K.im2col_first(x, out)
    xp = F.pad(x.float(), (0, 0, 1, 1, 1, 1))
    cols = torch.stack([xp[:, r:r + h, s:s + w, :] for r in range(3) for s in range(3)], 3)
    want = torch.zeros(n * h * w, 32, device="cuda")
    want[:, :27] = cols.reshape(n * h * w, 27)
    assert torch.equal(out.float(), want)
