"""VGG-style conv pipelines on B200 (BASELINE configs[3]) against the fp64
conv oracle (oracle/convnet_ref.py: the reference's replay with conv stage
math; the reference itself has no convolution).

Bars (bf16 operands and activations, fp32 accumulate, fp32 masters):
  * pins, update_source and the device-observed version tags: bit-exact;
  * against the fp64 oracle over whole epochs: per-mini-batch loss relative
    5e-3, final weights ||W - W_ref|| / ||W_ref|| 1e-3, weight deltas
    ||dW - dW_ref|| / ||dW_ref|| 1.5e-1 (measured <= 3.4e-3 / 4.3e-4 / 9.6e-2:
    besides operand rounding, 2x2 max pooling routes a window's gradient to
    another pixel whenever bf16 rounding ties or reorders its maximum, and
    such flips compound over the 20 mini-batches of the two-epoch case);
  * one SGD step against the oracle with the device's bf16 storage rounding
    (storage="bf16", which routes pooling gradients through the rounded
    windows like the device): loss 1e-5, the Linear layers' updates 1e-4,
    every update 5e-2 (measured 4e-8 / 3e-6 / 1.9e-2: the rest is
    accumulation order flipping the rounding of near-tied windows).
"""
import numpy as np
import pytest

from oracle import convnet_ref as R
from paper_2410_14312_b200 import convnet as CN
from paper_2410_14312_b200 import pipesim as P

pytestmark = pytest.mark.gpu


def _small(image=16, cfg=(64, "M", 64, "M", 128, "M"), hidden=128, classes=10):
    return CN.vgg(cfg, image=image, classes=classes, hidden=hidden, fc_layers=2)


def _oracle_layers(net):
    return [R.Layer(l.kind, l.in_, l.out, l.h, l.w, l.pool, l.act) for l in net.layers]


def _run(net, W, N, B, M, lr, mode="timeprest", seed=3, epochs=1, storage="fp64"):
    x, lab = CN.synthetic_images(M * B, net, seed=7)
    p0 = CN.init_params(net, seed)
    s = P.Session(net, W, N, B, M, lr, mode=mode)
    s.load_params(p0)
    s.upload(x, lab, y_labels=True)
    outs = [s.run_epoch() for _ in range(epochs)]
    got = s.read_params()
    split = net.partition(W)
    y = np.eye(net.layers[-1].out)[lab]
    p_ref, refs = p0, []
    for _ in range(epochs):
        refs.append(R.train_epoch(_oracle_layers(net), split, N, B, M, lr,
                                  x.astype(np.float64), y, p_ref, mode=mode, storage=storage))
        p_ref = refs[-1]["params"]
    s.close()
    return outs, refs, got, p0


def _check(outs, refs, got, p0, W, M, mode, loss_tol=5e-3, w_tol=1e-3, dw_tol=1.5e-1):
    rels = [np.abs(r["mini_loss"] - ref["losses"]).max() / np.abs(ref["losses"]).max()
            for r, ref in zip(outs, refs)]
    want = refs[-1]["params"]
    print(f"\nMETRIC loss {max(rels):.3e} w {np.linalg.norm(got - want) / np.linalg.norm(want):.3e}"
          f" dw {np.linalg.norm(got - want) / np.linalg.norm(want - p0):.3e}")
    for r, ref in zip(outs, refs):
        pins = np.array(ref["pinned"])
        assert np.array_equal(r["pinned"], pins)
        assert np.array_equal(r["consumed"], ref["consumed"])
        assert np.array_equal(r["dev_fwd"], np.repeat(pins[:, :, None], W, axis=2))
        assert np.all(r["dev_current"] == M)
        if mode == "timeprest":
            assert np.array_equal(r["dev_bwd"], np.repeat(np.arange(M)[:, None], W, axis=1))
        rel = np.abs(r["mini_loss"] - ref["losses"]).max() / np.abs(ref["losses"]).max()
        assert rel < loss_tol, rel
    want = refs[-1]["params"]
    assert np.linalg.norm(got - want) / np.linalg.norm(want) < w_tol
    dw = np.linalg.norm(got - want) / np.linalg.norm(want - p0)
    assert dw < dw_tol, dw


@pytest.mark.parametrize("W,N", [(2, 2), (3, 4), (5, 2)])
def test_small_vgg_timeprest(W, N):
    net = _small()
    B, M, lr = 8, 2 * (W + N), 0.002
    outs, refs, got, p0 = _run(net, W, N, B, M, lr)
    _check(outs, refs, got, p0, W, M, "timeprest")


@pytest.mark.parametrize("mode", ["pipedream", "sequential"])
def test_small_vgg_other_modes(mode):
    net = _small()
    W, N, B, M, lr = 2, 2, 8, 6, 0.002
    outs, refs, got, p0 = _run(net, W, N, B, M, lr, mode=mode)
    _check(outs, refs, got, p0, W, M, mode)


def test_vgg_two_epochs_and_wider_images():
    """Two epochs (rebase), 32x32 images, a conv without pooling and a
    256-channel layer; stage 1 holds two pooled convs."""
    net = _small(image=32, cfg=(64, "M", 128, 128, "M", 256, "M"), hidden=64)
    W, N, B, M, lr = 3, 2, 4, 10, 0.0005
    outs, refs, got, p0 = _run(net, W, N, B, M, lr, epochs=2)
    _check(outs, refs, got, p0, W, M, "timeprest")


def test_vgg_explicit_stage_split():
    net = _small()
    net.stage_layers = [1, 3, 1]
    W, N, B, M, lr = 3, 2, 8, 10, 0.002
    outs, refs, got, p0 = _run(net, W, N, B, M, lr)
    _check(outs, refs, got, p0, W, M, "timeprest")


def test_vgg_eta_zero_and_repeatable():
    net = _small()
    W, N, B, M = 2, 2, 8, 8
    x, lab = CN.synthetic_images(M * B, net, seed=7)
    p0 = CN.init_params(net, 3)
    s = P.Session(net, W, N, B, M, 0.0)
    s.load_params(p0)
    s.upload(x, lab, y_labels=True)
    a = s.run_epoch()
    got = s.read_params()
    # eta = 0: weights come back exactly (fp32 masters of fp64 values)
    assert np.array_equal(got, p0.astype(np.float32).astype(np.float64))
    b = s.run_epoch()
    assert np.array_equal(a["mini_loss"], b["mini_loss"])
    assert np.all(a["mini_loss"] == a["mini_loss"][0]) or np.ptp(a["mini_loss"]) > 0
    s.close()


def test_vgg_one_step_against_bf16_storage_oracle():
    net = _small()
    W, N, B, M, lr = 2, 2, 8, 1, 0.002
    outs, refs, got, p0 = _run(net, W, N, B, M, lr, storage="bf16")
    want = refs[0]["params"]
    assert abs(outs[0]["mini_loss"][0] - refs[0]["losses"][0]) / refs[0]["losses"][0] < 1e-5
    off = 0
    for l in net.layers:
        n = l.param_count()
        dg, dr = got[off:off + n] - p0[off:off + n], want[off:off + n] - p0[off:off + n]
        err = np.linalg.norm(dg - dr) / np.linalg.norm(dr)
        assert err < (1e-4 if l.kind == "linear" else 5e-2), (l, err)
        off += n
