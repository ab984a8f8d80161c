"""CPU checks of the conv-stage oracle (oracle/convnet_ref.py) and of the
conv network description / partition (host code, no GPU).

The reference has no convolution, so the conv oracle is pinned
here against torch autograd in float64: with a single weight version the
reference's stage_backward contract (trainer.cpp:216-267) must give exactly
the autograd gradient and input delta of the stage's forward."""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

from oracle import convnet_ref as R
from oracle import pipesim_np as O
from paper_2410_14312_b200 import convnet as CN

LAYERS = [R.Layer("conv", 3, 64, 8, 8, True, "relu"),
          R.Layer("conv", 64, 64, 4, 4, False, "relu"),
          R.Layer("conv", 64, 128, 4, 4, True, "relu"),
          R.Layer("linear", 512, 32, act="relu"),
          R.Layer("linear", 32, 10, act="linear")]


def _params(layers, seed=0):
    rng = np.random.default_rng(seed)
    return np.concatenate([np.concatenate([rng.uniform(-1, 1, L.out * L.fan_in()) /
                                           np.sqrt(L.fan_in()) * 2,
                                           rng.uniform(-0.1, 0.1, L.out)]) for L in layers])


def _autograd(layers, p, x, delta):
    pt = torch.tensor(p, requires_grad=True)
    xt = torch.tensor(x, requires_grad=True)
    n, off, cur = x.shape[0], 0, xt
    for L in layers:
        nw = L.out * L.fan_in()
        Wm, b = pt[off:off + nw].reshape(L.out, L.fan_in()), pt[off + nw:off + nw + L.out]
        off += nw + L.out
        if L.kind == "conv":
            X = cur.reshape(n, L.h, L.w, L.in_).permute(0, 3, 1, 2)
            Wt = Wm.reshape(L.out, 3, 3, L.in_).permute(0, 3, 1, 2)
            z = F.conv2d(X, Wt, b, padding=1)
            a = z.relu() if L.act == "relu" else z
            if L.pool:
                a = F.max_pool2d(a, 2)
            cur = a.permute(0, 2, 3, 1).reshape(n, -1)
        else:
            z = cur @ Wm.T + b
            cur = z.relu() if L.act == "relu" else z
    (cur * torch.tensor(delta)).sum().backward()
    return cur.detach().numpy(), pt.grad.numpy(), xt.grad.numpy()


def test_conv_stage_math_matches_autograd():
    rng = np.random.default_rng(1)
    p = _params(LAYERS)
    x = rng.random((5, 8 * 8 * 3))
    delta = rng.standard_normal((5, 10))
    cache = R.stage_forward(LAYERS, p, x)
    out, g_ref, dx_ref = _autograd(LAYERS, p, x, delta)
    np.testing.assert_allclose(cache["a"][-1], out, rtol=1e-12, atol=1e-12)
    g, dx = R.stage_backward(LAYERS, p, cache, delta)
    np.testing.assert_allclose(g, g_ref, rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(dx, dx_ref, rtol=1e-10, atol=1e-12)


def test_conv_replay_first_minibatch_is_plain_sgd():
    """Mini-batch 1 runs on version 0 in both passes (trainer.cpp:238-259's
    first-mini-batch equality): its update is one SGD step of the
    autograd gradient of the mean loss."""
    rng = np.random.default_rng(2)
    B, N, M, lr = 4, 2, 1, 0.1
    p = _params(LAYERS)
    x = rng.random((M * B, 8 * 8 * 3))
    lab = rng.integers(0, 10, M * B)
    y = np.eye(10)[lab]
    r = R.train_epoch(LAYERS, [2, 3], N, B, M, lr, x, y, p)
    cache = R.stage_forward(LAYERS, p, x)
    logits = cache["a"][-1]
    grad_out = O.loss_grad(logits, y, "softmax_cross_entropy", B)
    _, g, _ = _autograd(LAYERS, p, x, grad_out)
    np.testing.assert_allclose(r["params"], p - lr * g, rtol=1e-10, atol=1e-12)
    assert abs(r["losses"][0] - O.loss_mean(logits, y, "softmax_cross_entropy")) < 1e-12


def test_vgg16_description():
    net = CN.vgg16()
    assert len(net.layers) == 16
    assert sum(l.kind == "conv" for l in net.layers) == 13
    assert net.layers[13].in_ == 7 * 7 * 512
    # 138.36M parameters (VGG-16 with 1000 classes)
    assert net.param_count() == 138357544
    # ~15.47 G multiply-adds per 224x224 image forward
    assert abs(sum(l.flops() for l in net.layers) / 2 - 15.47e9) < 0.01e9


@pytest.mark.parametrize("W", [1, 2, 4, 8])
def test_flop_partition_is_balanced_and_contiguous(W):
    net = CN.vgg16()
    n = net.partition(W)
    assert len(n) == W and sum(n) == 16 and min(n) >= 1
    f = [l.flops() for l in net.layers]
    stages, at = [], 0
    for c in n:
        stages.append(sum(f[at:at + c]))
        at += c
    # optimal: no contiguous split has a smaller maximum (brute force on W <= 4)
    if W <= 4:
        import itertools
        best = min(max(sum(f[a:b]) for a, b in zip((0,) + cuts, cuts + (16,)))
                   for cuts in itertools.combinations(range(1, 16), W - 1))
        assert max(stages) == pytest.approx(best)


def test_layer_validation_errors():
    bad = CN.ConvNetSpec([CN.ConvLayer("conv", 3, 48, 8, 8), CN.ConvLayer("linear", 3072, 10)])
    with pytest.raises(ValueError, match="output channels % 64"):
        bad.partition(2)
    bad = CN.ConvNetSpec([CN.ConvLayer("conv", 3, 64, 8, 8), CN.ConvLayer("linear", 100, 10)])
    with pytest.raises(ValueError, match="input size"):
        bad.partition(2)
    with pytest.raises(Exception, match="cannot split"):
        CN.vgg16().partition(17)
