"""Per-stage checkpoints (host side, no GPU): the native writer produces the
reference's file format byte for byte (proj/src/checkpoint.cpp:39-67), each
build restores the other's files, and the integrity failures of
proj/tests/test_checkpoint.cpp:82-134 raise IntegrityError naming the stage
and epoch."""
import numpy as np
import pytest

from oracle import ref as R
from paper_2410_14312_b200 import pipesim as P

NET = P.NetworkSpec([12, 9, 7, 3], ["relu", "tanh", "linear"], "softmax_cross_entropy")


def _stages(version=5):
    stages = P.partition_model(NET, 2)
    rng = np.random.default_rng(3)
    p = rng.normal(size=NET.param_count()) * 10.0 ** rng.integers(-5, 3, NET.param_count())
    p[:3] = [0.0, 1e-300, -0.1]
    P.load_network_params(stages, p.astype(np.float32).astype(np.float64), version)
    return stages


def _layers(st):
    return [(l.in_, l.out, P.ACTIVATIONS.index(l.act)) for l in st.layers]


def test_checkpoint_file_matches_reference_bytes(tmp_path):
    if not R.available():
        pytest.skip("oracle/_ref not built")
    for st in _stages():
        ours = tmp_path / f"ours-{st.stage_id}.ckpt"
        theirs = tmp_path / f"ref-{st.stage_id}.ckpt"
        P.checkpoint_stage(st, NET.loss, 4, str(ours))
        R.checkpoint_stage(st.stage_id, st.first_layer, _layers(st), st.current_version,
                           st.current_params(), 1, 4, theirs)
        assert ours.read_bytes() == theirs.read_bytes()


def test_cross_restore_is_exact(tmp_path):
    if not R.available():
        pytest.skip("oracle/_ref not built")
    for st in _stages(version=7):
        a = tmp_path / "a.ckpt"
        R.checkpoint_stage(st.stage_id, st.first_layer, _layers(st), 7, st.current_params(), 1,
                           2, a)
        r = P.restore_stage(str(a), st.stage_id, 2)
        assert r.epoch == 2 and r.loss == NET.loss and r.stage.current_version == 7
        assert r.stage.first_layer == st.first_layer
        assert [(l.in_, l.out, l.act) for l in r.stage.layers] == \
            [(l.in_, l.out, l.act) for l in st.layers]
        np.testing.assert_array_equal(r.stage.current_params(), st.current_params())
        b = tmp_path / "b.ckpt"
        P.checkpoint_stage(st, NET.loss, 2, str(b))
        vals, v, e = R.restore_stage(b, st.stage_id, 2)
        np.testing.assert_array_equal(vals, st.current_params())
        assert (v, e) == (7, 2)


def test_large_stage_round_trip(tmp_path):
    """> 2^18 values: the text is formatted on host threads; the file and its
    digest still round-trip exactly."""
    net = P.NetworkSpec([700, 600, 10], ["relu", "linear"], "mse")
    st = P.partition_model(net, 2)[0]
    p = np.random.default_rng(0).normal(size=st.param_count()).astype(np.float32)
    st.version_store = {1: p.astype(np.float64)}
    st.current_version = 1
    f = tmp_path / "big.ckpt"
    P.checkpoint_stage(st, "mse", 1, str(f))
    r = P.restore_stage(str(f), 1, 1)
    np.testing.assert_array_equal(r.stage.current_params(), st.current_params())
    if R.available():
        vals, _, _ = R.restore_stage(f, 1, 1, cap=st.param_count())
        np.testing.assert_array_equal(vals, st.current_params())


def test_integrity_failures(tmp_path):
    """test_checkpoint.cpp:82-134: truncated, tampered, wrong stage / epoch,
    missing file."""
    st = _stages()[0]
    f = tmp_path / "s.ckpt"
    P.checkpoint_stage(st, NET.loss, 3, str(f))
    text = f.read_bytes()
    cases = {
        "truncated": text[:len(text) * 2 // 3],
        "tampered": text[:-3] + bytes([text[-3] ^ 1]) + text[-2:],
    }
    assert cases["tampered"] != text
    for name, body in cases.items():
        g = tmp_path / f"{name}.ckpt"
        g.write_bytes(body)
        with pytest.raises(P.IntegrityError) as ei:
            P.restore_stage(str(g), 1, 3)
        assert (ei.value.stage_id, ei.value.epoch) == (1, 3), name
    with pytest.raises(P.IntegrityError):
        P.restore_stage(str(f), 2, 3)
    with pytest.raises(P.IntegrityError):
        P.restore_stage(str(f), 1, 4)
    with pytest.raises(P.IntegrityError) as ei:
        P.restore_stage(str(tmp_path / "missing.ckpt"), 2, 9)
    assert (ei.value.stage_id, ei.value.epoch) == (2, 9)
    with pytest.raises(P.IoError):
        P.checkpoint_stage(st, NET.loss, 3, str(tmp_path / "no" / "such" / "dir.ckpt"))
