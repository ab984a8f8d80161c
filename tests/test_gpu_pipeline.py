"""Pipeline-step parity on B200: the GPU train_epoch (C ABI session) vs the
CPU oracle (numpy restatement, pinned to the compiled reference) on the same
seeded inputs and schedule.

Bar (stated tolerances, bf16 operands / fp32 accumulate / fp32 masters):
  * schedule, pins, update_source, per-stage consumptions and the
    device-observed version tags: bit-exact;
  * per-mini-batch loss: relative 2e-3 (1e-4 on the MNIST-shaped C1 net);
  * final weights ||W - W_ref|| / ||W_ref||: 1e-3;
  * weight deltas ||dW - dW_ref|| / ||dW_ref||: 8e-2 (bf16 operand rounding
    of gradients with cancellation).
"""
import json
import pathlib

import numpy as np
import pytest

from oracle import pipesim_np as O
from paper_2410_14312_b200 import pipesim as P

pytestmark = pytest.mark.gpu
GOLD = pathlib.Path(__file__).resolve().parent / "golden"


def _setup(widths, acts, loss, W, N, B, M, lr, seed):
    net = P.NetworkSpec(widths, acts, loss)
    data = P.make_classification_task(M * B, widths[0], widths[-1], seed=7)
    if loss == "mse":
        rng = np.random.default_rng(seed)
        data = P.Dataset(data.x, rng.uniform(-1, 1, data.y.shape))
    cfg = P.TrainConfig(net, W, N, B, M, 1, lr, seed)
    p0 = P.init_network_params(net, seed)
    return net, data, cfg, p0


def _run_both(widths, acts, loss, W, N, B, M, lr, seed, mode, epochs=1):
    net, data, cfg, p0 = _setup(widths, acts, loss, W, N, B, M, lr, seed)
    stages = P.partition_model(net, W)
    P.load_network_params(stages, p0, 0)
    onet = O.Net(widths, acts, loss)
    p_ref = p0
    logs, refs = [], []
    for e in range(1, epochs + 1):
        logs.append(P.train_epoch(stages, data, cfg, mode, e))
        refs.append(O.train_epoch(onet, W, N, B, M, lr, data.x, data.y, p_ref, mode=mode))
        p_ref = refs[-1]["params"]
    return stages, logs, refs, p0


def _check(stages, logs, refs, p0, W, mode, loss_tol=2e-3, dw_tol=8e-2, w_tol=1e-3):
    M = len(logs[0].minis)
    for log, r in zip(logs, refs):
        pins = np.array([m.pinned for m in log.minis])
        assert np.array_equal(pins, np.array(r["pinned"]))
        assert [m.consumed for m in log.minis] == r["consumed"].tolist()
        # device-observed trace: every forward read its pinned version on every stage
        assert np.array_equal(log.dev_fwd, np.repeat(pins[:, :, None], W, axis=2))
        assert np.all(log.dev_current == M)
        if mode == "timeprest":  # zero-stash: backward propagates through v = k-1
            assert np.array_equal(log.dev_bwd, np.repeat(np.arange(M)[:, None], W, axis=1))
        elif mode == "pipedream":  # stashed pin in both passes
            assert np.array_equal(log.dev_bwd, np.repeat(pins[:, :1], W, axis=1))
        losses = np.array([m.loss for m in log.minis])
        rel = np.abs(losses - r["losses"]).max() / np.abs(r["losses"]).max()
        assert rel < loss_tol, rel
    got = P.gather_network_params(stages)
    want = refs[-1]["params"]
    assert np.linalg.norm(got - want) / np.linalg.norm(want) < w_tol
    dw = np.linalg.norm((got - p0) - (want - p0)) / np.linalg.norm(want - p0)
    assert dw < dw_tol, dw


SMALL = [
    ("demo", [2, 8, 2], ["tanh", "linear"], "softmax_cross_entropy", 2, 2, 10, 6, 0.05, 42),
    ("deep4", [2, 6, 6, 6, 2], ["tanh"] * 3 + ["linear"], "softmax_cross_entropy", 4, 2, 4, 7,
     0.05, 2),
    ("mixed_mse", [30, 20, 16, 10], ["relu", "sigmoid", "linear"], "mse", 3, 4, 12, 10, 0.1, 5),
    ("relu8", [64, 48, 48, 40, 40, 32, 32, 24, 16], ["relu"] * 7 + ["linear"],
     "softmax_cross_entropy", 8, 8, 64, 6, 0.05, 3),
    ("sig_out", [16, 24, 8], ["tanh", "sigmoid"], "mse", 2, 3, 9, 5, 0.2, 9),
]


@pytest.mark.parametrize("case", SMALL, ids=[c[0] for c in SMALL])
@pytest.mark.parametrize("mode", ["timeprest", "pipedream", "sequential"])
def test_small_networks(case, mode):
    _, widths, acts, loss, W, N, B, M, lr, seed = case
    stages, logs, refs, p0 = _run_both(widths, acts, loss, W, N, B, M, lr, seed, mode, epochs=2)
    # tiny nets at large learning rates: bf16 drift compounds over 2 epochs
    _check(stages, logs, refs, p0, W, mode, loss_tol=3e-3, dw_tol=1e-1, w_tol=5e-3)


C1 = ([784, 512, 256, 10], ["relu", "relu", "linear"], "softmax_cross_entropy")


@pytest.mark.parametrize("mode,W", [("timeprest", 2), ("pipedream", 2), ("sequential", 2),
                                    ("sequential", 1)])
def test_c1_c2_mnist_shaped(mode, W):
    """configs[0]/[1]: 784-512-256-10, N=4, B=256, M=12 (= 2(W+N))."""
    stages, logs, refs, p0 = _run_both(*C1, W, 4, 256, 12, 0.05, 1, mode)
    _check(stages, logs, refs, p0, W, mode, loss_tol=1e-4)
    summ = json.loads((GOLD / "c1_summary.json").read_text())[f"{mode}.W{W}"]
    losses = np.array([m.loss for m in logs[0].minis])
    assert np.abs(losses - summ["losses"]).max() / max(summ["losses"]) < 1e-4


def test_c3_shape_reduced_width():
    """configs[2] structure (17 widths, 8 stages x 2 layers, N=8, B=1024) at
    width 256 so the fp64 oracle finishes in seconds."""
    stages, logs, refs, p0 = _run_both([256] * 17, ["relu"] * 15 + ["linear"],
                                       "softmax_cross_entropy", 8, 8, 1024, 4, 0.05, 1,
                                       "timeprest")
    _check(stages, logs, refs, p0, 8, "timeprest", loss_tol=1e-4)


def test_odd_mini_batch_count_multi_epoch():
    stages, logs, refs, p0 = _run_both([40, 56, 32, 12], ["relu", "tanh", "linear"],
                                       "softmax_cross_entropy", 3, 2, 16, 5, 0.1, 4,
                                       "timeprest", epochs=3)
    _check(stages, logs, refs, p0, 3, "timeprest")


def test_first_mini_batch_identical_across_modes():
    """proj/tests/test_trainer.cpp:238-259: with M=1 the three modes give the
    same parameters; on B200 they are bit-identical too (row-independent
    GEMM tiles, same stacked backward)."""
    widths, acts = [2, 8, 2], ["tanh", "linear"]
    finals = []
    for mode in ("timeprest", "sequential", "pipedream"):
        net, data, cfg, p0 = _setup(widths, acts, "softmax_cross_entropy", 2, 2, 8, 1, 0.1, 3)
        stages = P.partition_model(net, 2)
        P.load_network_params(stages, p0, 0)
        P.train_epoch(stages, data, cfg, mode, 1)
        finals.append(P.gather_network_params(stages))
    assert np.array_equal(finals[0], finals[1]) and np.array_equal(finals[0], finals[2])


def test_zero_learning_rate_keeps_weights():
    net, data, cfg, p0 = _setup([2, 8, 2], ["tanh", "linear"], "softmax_cross_entropy",
                                2, 2, 10, 4, 0.0, 5)
    for mode in ("timeprest", "sequential", "pipedream"):
        stages = P.partition_model(net, 2)
        P.load_network_params(stages, p0, 0)
        P.train_epoch(stages, data, cfg, mode, 1)
        # fp32 masters: the identity holds on the fp32-rounded initialisation
        np.testing.assert_array_equal(P.gather_network_params(stages),
                                      p0.astype(np.float32).astype(np.float64))


def test_deterministic_logs():
    """proj/tests/test_trainer.cpp:365-385: same seed -> identical bytes."""
    def run():
        net, data, cfg, p0 = _setup([2, 8, 2], ["tanh", "linear"], "softmax_cross_entropy",
                                    2, 2, 10, 6, 0.05, 42)
        stages = P.partition_model(net, 2)
        P.load_network_params(stages, p0, 0)
        return "".join(P.train_epoch(stages, data, cfg, "timeprest", e).to_text()
                       for e in (1, 2))
    a, b = run(), run()
    assert a == b
    assert "checksum" in a and "final checksum" in a


def test_mini_log_fields_and_retained_versions():
    """proj/tests/test_trainer.cpp:435-458 (W=4, N=2, M=7)."""
    net, data, cfg, p0 = _setup([2, 6, 6, 6, 2], ["tanh"] * 3 + ["linear"],
                                "softmax_cross_entropy", 4, 2, 4, 7, 0.05, 2)
    stages = P.partition_model(net, 4)
    P.load_network_params(stages, p0, 0)
    log = P.train_epoch(stages, data, cfg, "timeprest", 1)
    assert len(log.minis) == 7 and log.minis[0].mini == 1
    assert log.minis[2].consumed == 1 and log.minis[4].consumed == 3
    assert all(np.isfinite(m.loss) for m in log.minis)
    assert log.final_checksum == log.minis[-1].checksum
    g = P.build_nf1b_schedule(P.SimConfig(4, 2, 7))
    t = P.build_retention_timeline(P.assign_versions(g, P.SimConfig(4, 2, 7)), g)
    for s, st in enumerate(stages):
        want = {int(v) for v, a, b in t.intervals[s] if b > t.horizon}
        assert set(st.version_store) == want
        assert st.current_version == 7


def test_observer_sees_retention_timeline():
    """proj/tests/test_trainer.cpp:387-433."""
    net, data, cfg, p0 = _setup([2, 8, 2], ["tanh", "linear"], "softmax_cross_entropy",
                                2, 2, 8, 4, 0.05, 9)
    for mode in ("timeprest", "pipedream"):
        stages = P.partition_model(net, 2)
        P.load_network_params(stages, p0, 0)
        seen = []
        P.train_epoch(stages, data, cfg, mode, 1,
                      observer=lambda t, st: seen.append([set(s.version_store) for s in st]))
        r = O.train_epoch(O.Net([2, 8, 2], ["tanh", "linear"], "softmax_cross_entropy"), 2, 2,
                          8, 4, 0.05, data.x, data.y, p0, mode=mode, observe=True)
        want = [[{v for v in range(5) if r["held"][t, s, v]} for s in range(2)]
                for t in range(r["held"].shape[0])]
        assert seen == want


def test_network_loss_matches_oracle():
    widths, acts = C1[0], C1[1]
    net = P.NetworkSpec(widths, acts, C1[2])
    data = P.make_classification_task(300, 784, 10, seed=7)
    p = P.init_network_params(net, 1)
    got = P.network_loss(net, p, data)
    want = O.network_loss(O.Net(widths, acts, C1[2]), p, data.x, data.y)
    assert abs(got - want) / abs(want) < 1e-4


def test_session_resident_epochs_and_labels():
    """Resident session API (bench path): labels input == one-hot input."""
    net = P.NetworkSpec([128, 256, 64], ["relu", "linear"], "softmax_cross_entropy")
    p0 = P.init_network_params(net, 1)
    x, labels = P.make_classification_task(8 * 64, 128, 64, seed=7, as_labels=True,
                                           dtype=np.float32)
    onehot = np.zeros((len(labels), 64), np.float32)
    onehot[np.arange(len(labels)), labels] = 1
    outs = []
    for y, lab in ((labels, True), (onehot, False)):
        s = P.Session(net, 2, 4, 64, 8, 0.05, "timeprest")
        s.load_params(p0)
        s.upload(x, y, y_labels=lab)
        r1 = s.run_epoch()
        r2 = s.run_epoch()
        outs.append((r1["mini_loss"], r2["mini_loss"], s.read_params()))
        s.close()
    for a, b in zip(outs[0], outs[1]):
        np.testing.assert_array_equal(a, b)
    assert not np.array_equal(outs[0][0], outs[0][1])  # epoch 2 starts from trained weights


@pytest.mark.parametrize("widths,W", [([128, 256, 10], 2), ([784, 512, 256, 10], 2),
                                      ([784, 512, 256, 10], 1)])
def test_fused_softmax_ce_matches_loss_kernel(widths, W):
    """Class labels with <= 16 logits take the softmax-CE fused into the
    logits epilogue (and the fused two-layer forward on C1's shapes); one-hot
    targets take the separate loss kernel.  Same losses and weights."""
    acts = ["relu"] * (len(widths) - 2) + ["linear"]
    net = P.NetworkSpec(widths, acts, "softmax_cross_entropy")
    p0 = P.init_network_params(net, 1)
    x, labels = P.make_classification_task(8 * 64, widths[0], widths[-1], seed=7, as_labels=True,
                                           dtype=np.float32)
    onehot = np.zeros((len(labels), widths[-1]), np.float32)
    onehot[np.arange(len(labels)), labels] = 1
    mode = "timeprest" if W > 1 else "sequential"
    outs = []
    for y, lab in ((labels, True), (onehot, False)):
        s = P.Session(net, W, 4, 64, 8, 0.05, mode)
        s.load_params(p0)
        s.upload(x, y, y_labels=lab)
        r1 = s.run_epoch()
        r2 = s.run_epoch()
        outs.append((r1["mini_loss"], r2["mini_loss"], s.read_params()))
        s.close()
    for a, b in zip(outs[0][:2], outs[1][:2]):
        np.testing.assert_allclose(a, b, rtol=1e-5)
    d = np.linalg.norm(outs[0][2] - outs[1][2]) / np.linalg.norm(outs[1][2] - p0)
    assert d < 1e-3, d


@pytest.mark.parametrize("mode", ["timeprest", "pipedream"])
def test_forward_coalescing_is_bit_identical(mode):
    """Coalesced forwards (one GEMM over consecutive micro-batches with the same
    pinned version) must reproduce per-micro-batch launches bit for bit when
    no layer splits K (K < 512 here: GEMM rows are independent)."""
    net = P.NetworkSpec([256] * 9, ["relu"] * 7 + ["linear"], "softmax_cross_entropy")
    p0 = P.init_network_params(net, 1)
    x, lab = P.make_classification_task(6 * 512, 256, 256, seed=7, as_labels=True,
                                        dtype=np.float32)
    res = []
    for merge in (1, 0, 3):
        s = P.Session(net, 4, 8, 512, 6, 0.05, mode, fwd_merge=merge)
        s.load_params(p0)
        s.upload(x, lab, y_labels=True)
        r = s.run_epoch()
        res.append((r["mini_loss"], r["dev_fwd"], s.read_params()))
        s.close()
    for other in res[1:]:
        for a, b in zip(res[0], other):
            np.testing.assert_array_equal(a, b)


def test_forward_coalescing_with_split_k():
    """At widths where skinny forwards split K (a 128-row forward of a
    1024-wide layer runs as clusters of K chunks, a 512-row one does not),
    coalescing only reorders fp32 sums: losses and weights agree to fp32
    rounding, and version traces stay exact."""
    net = P.NetworkSpec([1024] * 5, ["relu"] * 3 + ["linear"], "softmax_cross_entropy")
    p0 = P.init_network_params(net, 1)
    x, lab = P.make_classification_task(6 * 512, 1024, 1024, seed=7, as_labels=True,
                                        dtype=np.float32)
    res = []
    for merge in (1, 0):
        s = P.Session(net, 2, 4, 512, 6, 0.05, "timeprest", fwd_merge=merge)
        s.load_params(p0)
        s.upload(x, lab, y_labels=True)
        r = s.run_epoch()
        res.append((r["mini_loss"], r["dev_fwd"], s.read_params()))
        s.close()
    np.testing.assert_allclose(res[0][0], res[1][0], rtol=1e-4)
    np.testing.assert_array_equal(res[0][1], res[1][1])
    d = np.linalg.norm(res[0][2] - res[1][2]) / np.linalg.norm(res[1][2])
    assert d < 1e-4


@pytest.mark.parametrize("precision", ["bf16", "fp32"])
def test_streamed_host_epoch_matches_resident(precision):
    """pb_session_train_epoch from page-locked host buffers streams the upload
    inside the epoch (per-mini-batch H2D + conversion on its own stream,
    stage 1 and the loss wait per mini-batch); results are bit-identical to
    upload + resident epoch, over several epochs and a buffer change."""
    import torch
    net = P.NetworkSpec([96, 128, 64, 10], ["relu", "tanh", "linear"], "softmax_cross_entropy")
    W, N, B, M = 3, 4, 64, 7
    x, lab = P.make_classification_task(M * B, 96, 10, seed=7, as_labels=True, dtype=np.float32)
    x2 = (x[::-1] * 0.5).copy()
    res = []
    for streamed in (False, True):
        s = P.Session(net, W, N, B, M, 0.05, "timeprest", precision=precision)
        s.load_params(P.init_network_params(net, 1))
        xs = [torch.from_numpy(a).pin_memory() for a in (x, x2)]
        yh = torch.from_numpy(lab).pin_memory()
        outs = []
        for e, xh in enumerate((xs[0], xs[0], xs[1])):
            if streamed:
                r = s.train_epoch_host(xh.data_ptr(), "f32", yh.data_ptr(), "labels")
            else:
                s.upload(xh.numpy(), yh.numpy(), y_labels=True)
                r = s.run_epoch()
            outs.append((r["mini_loss"].copy(), r["dev_fwd"].copy()))
        outs.append(s.read_params())
        s.close()
        res.append(outs)
    for a, b in zip(res[0][:-1], res[1][:-1]):
        np.testing.assert_array_equal(a[0], b[0])
        np.testing.assert_array_equal(a[1], b[1])
    np.testing.assert_array_equal(res[0][-1], res[1][-1])


def test_split_master_round_trip_is_exact():
    """Split fp32 masters (bf16 hi in the version pool + 16-bit residual):
    load_params -> read_params returns the fp32 rounding of the input bit for
    bit, including values on bf16 rounding ties and of both signs."""
    net = P.NetworkSpec([256, 512, 256], ["relu", "linear"], "softmax_cross_entropy")
    p0 = P.init_network_params(net, 3)
    ties = np.array([1.0 + 2.0 ** -8, -(1.0 + 3 * 2.0 ** -8), 2.0 ** -130, -3.0e38, 1e-45])
    p0[:len(ties)] = ties
    s = P.Session(net, 2, 4, 256, 2, 0.05, "timeprest")
    s.load_params(p0)
    got = s.read_params()
    s.close()
    np.testing.assert_array_equal(got, p0.astype(np.float32).astype(np.float64))


def test_split_masters_match_fp32_masters():
    """The same epochs with split masters (default for pair-kernel layers) and
    with fp32 masters (PIPESIM_SPLIT_MASTER=0 in a subprocess).  The update is
    the same fp32 arithmetic; the bf16 GEMM operand differs only on exact
    rounding ties (half away from zero instead of half to even, ~1 weight in
    65536), which bf16 training amplifies like any operand perturbation
    (measured: dW 1.4e-4 after one mini-batch, 8e-3 after four).  The bar is
    the one the bf16 path meets against the fp64 oracle."""
    import subprocess
    import sys
    code = r'''
import sys, numpy as np
sys.path.insert(0, ".")
from paper_2410_14312_b200 import pipesim as P
net = P.NetworkSpec([512] * 4, ["relu", "relu", "linear"], "softmax_cross_entropy")
p0 = P.init_network_params(net, 1)
x, lab = P.make_classification_task(4 * 512, 512, 512, seed=7, as_labels=True, dtype=np.float32)
s = P.Session(net, 2, 4, 512, 4, 0.05, "timeprest")
s.load_params(p0); s.upload(x, lab, y_labels=True)
r1 = s.run_epoch(); r2 = s.run_epoch()
np.save(sys.argv[1], np.concatenate([r1["mini_loss"], r2["mini_loss"], s.read_params()]))
'''
    import os
    import tempfile
    outs = []
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with tempfile.TemporaryDirectory() as td:
        for flag in ("1", "0"):
            f = os.path.join(td, f"r{flag}.npy")
            env = dict(os.environ, PIPESIM_SPLIT_MASTER=flag)
            subprocess.run([sys.executable, "-c", code, f], check=True, env=env, cwd=root)
            outs.append(np.load(f))
    a, b = outs
    p0 = np.concatenate([np.zeros(8), P.init_network_params(
        P.NetworkSpec([512] * 4, ["relu", "relu", "linear"], "softmax_cross_entropy"), 1)])
    assert np.abs(a[:8] - b[:8]).max() / np.abs(b[:8]).max() < 1e-4
    assert np.linalg.norm(a[8:] - b[8:]) / np.linalg.norm(b[8:]) < 1e-4
    dw = np.linalg.norm((a - p0)[8:] - (b - p0)[8:]) / np.linalg.norm((b - p0)[8:])
    assert dw < 8e-2, dw
