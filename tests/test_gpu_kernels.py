"""Layer kernels (tcgen05 GEMMs, loss, bias-SGD) vs a plain torch fp32
reference of the same op on the same bf16 inputs.

Tolerances: fp32 outputs of the bf16 GEMMs are compared at rel 2e-5 of the
output scale (only the fp32 accumulation order differs); bf16 outputs at
one bf16 ulp (2^-8 relative) of the output scale.
"""
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2410_14312_b200 import kernels as K  # noqa: E402


@pytest.fixture(autouse=True)
def _no_tf32():
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.manual_seed(0)


def _act(z, act):
    return {"linear": z, "relu": torch.relu(z), "tanh": torch.tanh(z),
            "sigmoid": torch.sigmoid(z)}[act]


def _dact_from_out(a, act):
    return {"linear": torch.ones_like(a), "relu": (a > 0).float(),
            "tanh": 1 - a * a, "sigmoid": a * (1 - a)}[act]


def _rel(got, want):
    return ((got.float() - want.float()).abs().max() / (want.float().abs().max() + 1e-30)).item()


FWD_SHAPES = [
    (128, 256, 128), (64, 784, 512), (64, 512, 256), (64, 256, 10), (5, 2, 8),
    (200, 100, 10), (256, 4096, 4096), (128, 4096, 4096), (1000, 136, 392),
    # 64-wide pair tiles (out <= 64, rows > 128), ragged rows
    (1000, 136, 64), (300, 72, 40),
    # split-K shapes (K >= 1024): ragged N, ragged last split, partial M tiles
    (1024, 4096, 4096), (512, 1024, 1536), (384, 2048, 1000), (100, 3000, 700),
    # 256 x 512 tiles with a partial last row tile / ragged rows
    (700, 1024, 2048), (1000, 512, 1024),
]


@pytest.mark.parametrize("rows,inn,out", FWD_SHAPES)
@pytest.mark.parametrize("act", ["linear", "relu", "tanh", "sigmoid"])
def test_linear_fwd(rows, inn, out, act):
    x = K.padded_bf16(rows, inn)
    x.copy_(torch.rand(rows, inn, device="cuda"))
    w = K.padded_bf16(out, inn)
    w.copy_((torch.rand(out, inn, device="cuda") * 2 - 1) / inn ** 0.5)
    b = (torch.rand(out, device="cuda") - 0.5)
    y16 = K.padded_bf16(rows, out)
    y32 = torch.zeros(rows, out, device="cuda")
    K.linear_fwd(x, w, b, act, y16=y16, y32=y32)
    torch.cuda.synchronize()
    ref = _act(x.float() @ w.float().T + b, act)
    assert _rel(y32, ref) < 2e-5
    assert _rel(y16, ref) < 2 ** -8


DX_SHAPES = [(128, 256, 128), (256, 512, 784), (256, 10, 256), (5, 8, 2),
             (1024, 4096, 4096), (300, 136, 72),
             # 256 x 512 tiles with a partial last row tile (interior fast path + edge path)
             (600, 1024, 1024), (520, 2048, 1536)]


@pytest.mark.parametrize("rows,out,inn", DX_SHAPES)
@pytest.mark.parametrize("act_prev", ["linear", "relu", "tanh"])
def test_linear_bwd_dx(rows, out, inn, act_prev):
    dz = K.padded_bf16(rows, out)
    dz.copy_(torch.randn(rows, out, device="cuda") * 1e-2)
    w = K.padded_bf16(out, inn)
    w.copy_((torch.rand(out, inn, device="cuda") * 2 - 1) / inn ** 0.5)
    xin = K.padded_bf16(rows, inn)
    xin.copy_(_act(torch.randn(rows, inn, device="cuda"), act_prev))
    d = K.padded_bf16(rows, inn)
    K.linear_bwd_dx(dz, w, xin, act_prev, d)
    torch.cuda.synchronize()
    ref = (dz.float() @ w.float()) * _dact_from_out(xin.float(), act_prev)
    assert _rel(d, ref) < 2 ** -8


DW_SHAPES = [(256, 512, 784), (256, 10, 256), (64, 128, 128), (5, 8, 2),
             (1024, 4096, 4096), (300, 136, 72), (20, 2, 8)]


@pytest.mark.parametrize("rows,out,inn", DW_SHAPES)
def test_linear_bwd_dw_sgd(rows, out, inn):
    dz = K.padded_bf16(rows, out)
    dz.copy_(torch.randn(rows, out, device="cuda") * 1e-2)
    x = K.padded_bf16(rows, inn)
    x.copy_(torch.rand(rows, inn, device="cuda"))
    w_cur = (torch.rand(out, inn, device="cuda") * 2 - 1)
    w_new = torch.empty_like(w_cur)
    w16 = K.padded_bf16(out, inn)
    lr = 0.5
    K.linear_bwd_dw_sgd(dz, x, w_cur, w_new, w16, lr)
    torch.cuda.synchronize()
    g = dz.float().T @ x.float()
    ref = w_cur - lr * g
    # the update itself (w_new - w_cur) must match to fp32-accumulation accuracy
    assert _rel(w_new - w_cur, ref - w_cur) < 5e-5
    assert _rel(w16, ref) < 2 ** -8


def _padded_i16(rows, cols):
    ld = (cols + 7) // 8 * 8
    return torch.zeros(rows, ld, dtype=torch.int16, device="cuda")[:, :cols]


@pytest.mark.parametrize("rows,out,inn", [(256, 512, 784), (1024, 4096, 4096), (300, 136, 72),
                                          (512, 1000, 520)])
def test_linear_bwd_dw_sgd_split_master(rows, out, inn):
    """Split fp32 masters (hi = bf16 operand, lo = 16-bit residual): the
    split / join round trip is exact, the update matches the fp32-master
    kernel bit for bit (same fp32 arithmetic), and hi is the new master
    rounded to bf16 (nearest; exact ties away from zero)."""
    dz = K.padded_bf16(rows, out)
    dz.copy_(torch.randn(rows, out, device="cuda") * 1e-2)
    x = K.padded_bf16(rows, inn)
    x.copy_(torch.rand(rows, inn, device="cuda"))
    w_cur = (torch.rand(out, inn, device="cuda") * 2 - 1)
    hi, lo = K.padded_bf16(out, inn), _padded_i16(out, inn)
    K.split_master(w_cur, hi, lo)
    back = torch.empty_like(w_cur)
    K.join_master(hi, lo, back)
    torch.cuda.synchronize()
    assert torch.equal(back, w_cur)
    hi2, lo2 = K.padded_bf16(out, inn), _padded_i16(out, inn)
    lr = 0.5
    K.linear_bwd_dw_sgd_split(dz, x, hi, lo, hi2, lo2, lr)
    w_new = torch.empty_like(w_cur)
    K.join_master(hi2, lo2, w_new)
    ref_new = torch.empty_like(w_cur)
    K.linear_bwd_dw_sgd(dz, x, w_cur, ref_new, None, lr)
    torch.cuda.synchronize()
    assert torch.equal(w_new, ref_new)
    assert torch.equal(hi2.float(), w_new.to(torch.bfloat16).float()) or \
        (hi2.float() - w_new.to(torch.bfloat16).float()).abs().max() <= \
        w_new.abs().max() * 2 ** -7  # ties only


def test_wgrad_in_place():
    rows, out, inn = 128, 256, 256
    dz = K.padded_bf16(rows, out)
    dz.copy_(torch.randn(rows, out, device="cuda"))
    x = K.padded_bf16(rows, inn)
    x.copy_(torch.rand(rows, inn, device="cuda"))
    w = torch.rand(out, inn, device="cuda")
    ref = w - 0.1 * (dz.float().T @ x.float())
    K.linear_bwd_dw_sgd(dz, x, w, w, None, 0.1)
    torch.cuda.synchronize()
    assert _rel(w, ref) < 2e-5


@pytest.mark.parametrize("rows,out", [(256, 512), (1024, 4096), (7, 3), (20, 2)])
def test_bias_sgd(rows, out):
    dz = K.padded_bf16(rows, out)
    dz.copy_(torch.randn(rows, out, device="cuda"))
    b = torch.rand(out, device="cuda")
    b_new = torch.empty_like(b)
    b_copy = torch.empty_like(b)
    K.bias_sgd(dz, b, b_new, b_copy, 0.05)
    torch.cuda.synchronize()
    ref = b - 0.05 * dz.float().sum(0)
    assert torch.allclose(b_new, ref, rtol=1e-5, atol=1e-5)
    assert torch.equal(b_new, b_copy)


@pytest.mark.parametrize("loss", ["softmax_cross_entropy", "mse"])
@pytest.mark.parametrize("rows,cols", [(256, 10), (1024, 4096), (3, 2)])
def test_loss(loss, rows, cols):
    y = torch.randn(rows, cols, device="cuda")
    t = torch.zeros(rows, cols, device="cuda")
    if loss == "mse":
        t = torch.randn(rows, cols, device="cuda")
    else:
        t[torch.arange(rows), torch.randint(0, cols, (rows,))] = 1.0
    dz = K.padded_bf16(rows, cols)
    rl = torch.zeros(rows, device="cuda")
    denom = rows
    K.loss_fwd_bwd(y, t, loss, "linear", denom, dz, rl)
    torch.cuda.synchronize()
    yd, td = y.double(), t.double()
    if loss == "mse":
        ref_rl = ((yd - td) ** 2).sum(1)
        ref_g = 2 * (yd - td) / denom
    else:
        lsm = torch.log_softmax(yd, 1)
        ref_rl = -(lsm * td * (td > 0.5)).sum(1)
        ref_g = (torch.softmax(yd, 1) - td) / denom
    assert torch.allclose(rl.double(), ref_rl, rtol=1e-5, atol=1e-5)
    assert _rel(dz, ref_g) < 2 ** -8


@pytest.mark.parametrize("rows,inn,out", [(128, 4096, 4096), (256, 4096, 4096), (64, 3000, 700),
                                          (200, 2048, 1000), (128, 1024, 136)])
def test_split_k_cluster_forward_deterministic(rows, inn, out):
    """Split-K forwards (one thread-block cluster per tile, DSMEM reduction in
    split order): repeated launches give identical bits, and the result
    matches the fp32 reference at the GEMM tolerance."""
    x = K.padded_bf16(rows, inn)
    x.copy_(torch.rand(rows, inn, device="cuda"))
    w = K.padded_bf16(out, inn)
    w.copy_((torch.rand(out, inn, device="cuda") * 2 - 1) / inn ** 0.5)
    b = (torch.rand(out, device="cuda") - 0.5)
    ys = []
    for _ in range(3):
        y = torch.zeros(rows, out, device="cuda")
        K.linear_fwd(x, w, b, "relu", y32=y)
        ys.append(y)
    torch.cuda.synchronize()
    assert torch.equal(ys[0], ys[1]) and torch.equal(ys[0], ys[2])
    ref = torch.relu(x.float() @ w.float().T + b)
    assert _rel(ys[0], ref) < 2e-5


@pytest.mark.parametrize("rows", [128, 256, 768, 1024])
def test_linear_fwd_split_fixup_deterministic(rows):
    """Skinny forwards split K over CTA pairs with the in-kernel fixup (the
    last split of a tile sums the partials in split order): the result is
    run-to-run bit-identical and matches fp32 torch (opt-in path:
    PIPESIM_FWD_FIX=1; with the default the cluster split runs here)."""
    inn = out = 4096
    x = K.padded_bf16(rows, inn)
    x.copy_(torch.rand(rows, inn, device="cuda"))
    w = K.padded_bf16(out, inn)
    w.copy_((torch.rand(out, inn, device="cuda") * 2 - 1) / inn ** 0.5)
    b = torch.rand(out, device="cuda") - 0.5
    ys = []
    for _ in range(3):
        y32 = torch.zeros(rows, out, device="cuda")
        K.linear_fwd(x, w, b, "relu", y32=y32)
        ys.append(y32)
    torch.cuda.synchronize()
    assert torch.equal(ys[0], ys[1]) and torch.equal(ys[0], ys[2])
    ref = torch.relu(x.float() @ w.float().T + b)
    assert _rel(ys[0], ref) < 2e-5
