"""Device parity at the configurations the round-1 suite did not run:

* C5: the whole (W, N) sweep grid, W in {2, 4, 8} x N in 2..16 at the
  strict-measurement length M = 2(W + N) (ledger.cpp:121-142), on a
  reduced-width 8-layer network.  For every cell the device-observed version
  tags (forward pins, backward consumptions, current version), the trace
  document in the reference's schema (export.cpp:78-139, v_closed_form and
  v_measured included -- they diverge at (8,2) and (8,3)), the pins and
  consumed versions must equal the ledger bit for bit, and the losses the
  fp64 oracle's within the bf16 tolerance.  N = 1 is the reference's domain
  error (config.hpp:48-51).
* C3 structure (17 widths, W=8 stages x 2 layers, N=8, B=1024) at width 256
  with M = 32 = 2(W+N), so the steady-state regime the paper is about runs.
* Python run_training: resume from per-stage checkpoints is bit-identical to
  an uninterrupted run (proj/tests/test_checkpoint.cpp:136-158).
"""
import json

import numpy as np
import pytest

from oracle import pipesim_np as O
from oracle import ref as R
from paper_2410_14312_b200 import pipesim as P

pytestmark = pytest.mark.gpu

C5_WIDTHS = [24, 32, 32, 24, 24, 32, 24, 24, 12]
C5_ACTS = ["relu", "tanh", "relu", "relu", "tanh", "relu", "relu", "linear"]
C5_CELLS = [(W, N) for W in (2, 4, 8) for N in range(2, 17)]


@pytest.mark.parametrize("W,N", C5_CELLS, ids=[f"W{w}N{n}" for w, n in C5_CELLS])
def test_c5_grid_device_traces(W, N):
    M = 2 * (W + N)
    B = 2 * N
    net = P.NetworkSpec(C5_WIDTHS, C5_ACTS, "softmax_cross_entropy")
    p0 = P.init_network_params(net, 1)
    x, y = O.make_classification_task(M * B, C5_WIDTHS[0], C5_WIDTHS[-1], seed=7)
    s = P.Session(net, W, N, B, M, 0.05, "timeprest")
    try:
        s.load_params(p0)
        s.upload(x, y)
        r = s.run_epoch()
        doc = s.trace_document()
    finally:
        s.close()
    ref = O.train_epoch(O.Net(C5_WIDTHS, C5_ACTS, "softmax_cross_entropy"), W, N, B, M, 0.05,
                        x, y, p0)
    pins = np.array(ref["pinned"])
    assert np.array_equal(r["pinned"], pins)
    assert np.array_equal(r["consumed"], ref["consumed"])
    assert np.array_equal(r["dev_fwd"], np.repeat(pins[:, :, None], W, axis=2))
    assert np.array_equal(r["dev_bwd"], np.repeat(np.arange(M)[:, None], W, axis=1))
    assert np.all(r["dev_current"] == M)
    want = P.schedule_document_json(
        P.SimConfig(workers=W, micro_batches=N, mini_batches=M, samples_per_mini_batch=B))
    assert doc == want
    d = json.loads(doc)
    # the v laws: measured = floor((W-1)/(N+1)) + 1; closed form floor((W+N-2)/N)
    closed = P.closed_form_v(W, N)
    assert closed == (W + N - 2) // N
    assert (W - 1) // (N + 1) + 1 == O.measure_version_difference(
        O.assign_versions(O.build_schedule(W, N, M), W, N, M)["update_source"], W, N, M)
    if R.available():
        theirs = json.loads(R.schedule_document(W, N, M, 0))
        for k in ("samples_per_mini_batch",):
            d.get("config", {}).pop(k, None)
            theirs.get("config", {}).pop(k, None)
        assert d == theirs
    losses = r["mini_loss"]
    rel = np.abs(losses - ref["losses"]).max() / np.abs(ref["losses"]).max()
    assert rel < 3e-3, rel


@pytest.mark.parametrize("W", [2, 4, 8])
def test_c5_single_micro_batch_is_domain_error(W):
    net = P.NetworkSpec(C5_WIDTHS, C5_ACTS, "softmax_cross_entropy")
    with pytest.raises(P.DomainError) as ei:
        P.Session(net, W, 1, 4, 4, 0.05, "timeprest")
    assert ei.value.field == "micro_batches"


def test_c3_structure_steady_state():
    """configs[2] structure at width 256, M = 32: the v-steady regime at W=8,
    N=8 (pins 3G,3H,4A-4F:1 ...), traces exact, losses / weights vs fp64."""
    widths, acts = [256] * 17, ["relu"] * 15 + ["linear"]
    W, N, B, M = 8, 8, 1024, 32
    net = P.NetworkSpec(widths, acts, "softmax_cross_entropy")
    p0 = P.init_network_params(net, 1)
    data = P.make_classification_task(M * B, 256, 256, seed=7)
    cfg = P.TrainConfig(net, W, N, B, M, 1, 0.05, 1)
    stages = P.partition_model(net, W)
    P.load_network_params(stages, p0, 0)
    log = P.train_epoch(stages, data, cfg, "timeprest", 1)
    ref = O.train_epoch(O.Net(widths, acts, "softmax_cross_entropy"), W, N, B, M, 0.05,
                        data.x, data.y, p0)
    pins = np.array([m.pinned for m in log.minis])
    assert np.array_equal(pins, np.array(ref["pinned"]))
    assert [m.consumed for m in log.minis] == ref["consumed"].tolist()
    assert np.array_equal(log.dev_fwd, np.repeat(pins[:, :, None], W, axis=2))
    assert np.array_equal(log.dev_bwd, np.repeat(np.arange(M)[:, None], W, axis=1))
    # steady state reached: update_source gap k - consumed = measured v = 1
    cons = ref["consumed"]
    assert all(k + 1 - cons[k] == 1 for k in range(M // 2, M))
    losses = np.array([m.loss for m in log.minis])
    assert np.abs(losses - ref["losses"]).max() / np.abs(ref["losses"]).max() < 1e-4
    got = P.gather_network_params(stages)
    want = ref["params"]
    assert np.linalg.norm(got - want) / np.linalg.norm(want) < 1e-3
    dw = np.linalg.norm(got - want) / np.linalg.norm(want - p0)
    assert dw < 8e-2, dw


@pytest.mark.parametrize("mode", ["timeprest", "pipedream", "sequential"])
def test_python_run_training_resume_is_bit_identical(mode, tmp_path):
    """run_training (trainer.cpp:704-758) for 3 epochs vs 2 epochs + resume:
    identical last-epoch log, final checksum and checkpoint bytes."""
    net = P.NetworkSpec([20, 16, 12, 4], ["relu", "tanh", "linear"], "softmax_cross_entropy")
    W = 1 if mode == "sequential" else 3
    data = P.make_classification_task(6 * 8, 20, 4, seed=7)
    cfg = P.TrainConfig(net, W, 2, 8, 6, 3, 0.1, 9)
    full = P.run_training(cfg, mode, data, str(tmp_path / "a"))
    part = P.run_training(P.TrainConfig(net, W, 2, 8, 6, 2, 0.1, 9), mode, data,
                          str(tmp_path / "b"))
    res = P.run_training(cfg, mode, data, str(tmp_path / "b"), resume=True)
    assert (full.first_epoch, part.first_epoch, res.first_epoch) == (1, 1, 3)
    assert len(res.logs) == 1
    assert res.logs[0].to_text() == full.logs[-1].to_text()
    assert res.final_checksum == full.final_checksum
    for s in range(1, W + 1):
        f = P.checkpoint_filename(s, 3)
        assert (tmp_path / "a" / f).read_bytes() == (tmp_path / "b" / f).read_bytes()
    # a missing sibling stage file refuses the resume (trainer.cpp:717-742)
    if W > 1:
        (tmp_path / "b" / P.checkpoint_filename(2, 3)).unlink()
        with pytest.raises(P.IntegrityError) as ei:
            P.run_training(cfg, mode, data, str(tmp_path / "b"), resume=True)
        assert (ei.value.stage_id, ei.value.epoch) == (2, 3)
