"""Product plan layer (native host C++ behind the C ABI) vs the reference:
schedule grids, validator, version ledger, retention, v-table and the
domain contract must be bit-exact.  CPU only."""
import json
import pathlib

import numpy as np
import pytest

from oracle import pipesim_np as O
from oracle import ref
from paper_2410_14312_b200 import pipesim as P

GOLD = pathlib.Path(__file__).resolve().parent / "golden"
MODES = {0: "timeprest", 1: "pipedream"}


def _cfg(w, n, m):
    return P.SimConfig(workers=w, micro_batches=n, mini_batches=m)


def _grid(w, n, m, mode):
    c = _cfg(w, n, m)
    return P.build_nf1b_schedule(c) if mode == "timeprest" else P.build_1f1b_schedule(c)


def test_plan_goldens_product():
    for c in json.loads((GOLD / "plan_goldens.json").read_text()):
        w, n, m, mode = c["W"], c["N"], c["M"], MODES[c["mode"]]
        g = _grid(w, n, m, mode)
        assert g.cells.tolist() == c["grid"], (w, n, m, mode)
        led = P.assign_versions(g, _cfg(w, n, m))
        for key in ("commits", "pins", "consumptions", "update_source", "full_commit_slot"):
            assert np.asarray(getattr(led, key)).tolist() == c[key], (key, w, n, m, mode)
        t = P.build_retention_timeline(led, g)
        assert t.intervals.tolist() == c["retention"] and t.peak_concurrent == c["peak"]
        assert P.closed_form_v(w, n) == c["v_closed"]
        if c["v_measured"] is not None:
            assert P.measure_version_difference(led, strict=False) == c["v_measured"]


@pytest.mark.parametrize("name", ["4-2-7", "4-4-4", "3-2-6", "5-2-6", "5-3-6"])
def test_timeline_goldens_product(name):
    w, n, m = map(int, name.split("-"))
    g = _grid(w, n, m, "timeprest")
    assert O.render_ascii(g.cells) == (GOLD / f"timeline-{name}.txt").read_text()


def test_appendix_a_traces():
    """the C1-shaped grid and pins."""
    g = _grid(2, 4, 4, "timeprest")
    assert g.horizon() == 22
    led = P.assign_versions(g, _cfg(2, 4, 4))
    pins = [int(p[3]) for p in led.pins]
    assert pins[:8] == [0, 0, 0, 0, 0, 0, 1, 1]
    assert led.update_source.tolist() == [0, 1, 2, 3]
    g = _grid(4, 2, 6, "timeprest")
    assert P.assign_versions(g, _cfg(4, 2, 6)).update_source.tolist() == [0, 0, 1, 2, 3, 4]


def test_v_table_sweep():
    """C5: closed-form and measured v over W in {2,4,8} x N in 2..16."""
    for w in (2, 4, 8):
        for n in range(2, 17):
            m = 2 * (w + n)
            led = P.assign_versions(_grid(w, n, m, "timeprest"), _cfg(w, n, m))
            assert P.measure_version_difference(led) == (w - 1) // (n + 1) + 1
            assert P.closed_form_v(w, n) == (w + n - 2) // n
            assert P.overlap_condition(w, n) == (w > n + 1)
    with pytest.raises(P.DomainError) as e:
        P.closed_form_v(8, 1)
    assert e.value.field == "micro_batches"


@pytest.mark.parametrize("bad,field", [((1, 2, 3), "workers"), ((2, 1, 3), "micro_batches"),
                                       ((2, 2, 0), "mini_batches")])
def test_domain_errors(bad, field):
    with pytest.raises(P.DomainError) as e:
        P.build_nf1b_schedule(_cfg(*bad))
    assert e.value.field == field
    assert field.split("_")[0] in str(e.value)


def test_insufficient_horizon_and_structural():
    g = _grid(4, 2, 5, "timeprest")
    led = P.assign_versions(g, _cfg(4, 2, 5))
    with pytest.raises(P.InsufficientHorizonError):
        P.measure_version_difference(led, strict=True)
    with pytest.raises(P.StructuralError):
        P.assign_versions(g, _cfg(4, 2, 6))  # grid does not match config
    bad = g.copy()
    bad.clear(2, 3)
    with pytest.raises(P.StructuralError):
        P.assign_versions(bad, _cfg(4, 2, 5))


def _mutations(g):
    """Hand-mutated grids in the spirit of proj/tests/test_schedule.cpp:138-195."""
    out = []
    W, H = g.workers(), g.horizon()
    for s in range(1, W + 1):
        for t in range(1, H + 1, 3):
            c = g.copy()
            c.clear(s, t)
            out.append(c)
    for s in range(1, W + 1):
        for t in range(1, H, 4):
            c = g.copy()
            a, b = c.at(s, t), c.at(s, t + 1)
            c.put(s, t, b)
            c.put(s, t + 1, a)
            out.append(c)
    c = g.copy()
    c.put(1, H + 1, P.Task(P.FORWARD, 1, 1))  # duplicate forward
    out.append(c)
    return out


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("w,n,m,mode", [(3, 2, 4, "timeprest"), (4, 3, 3, "timeprest"),
                                        (3, 2, 4, "pipedream")])
def test_validator_matches_reference(w, n, m, mode):
    cfg = _cfg(w, n, m)
    g = _grid(w, n, m, mode)
    assert P.validate_schedule(g, cfg).valid()
    for c in _mutations(g):
        mine = [(P.VIOLATION_KINDS.index(v.kind), v.message)
                for v in P.validate_schedule(c, cfg).violations]
        theirs = ref.validate(w, n, m, 0 if mode == "timeprest" else 1, c.cells)
        assert mine == theirs


def test_sequences_and_staleness():
    g = _grid(8, 2, 20, "timeprest")
    led = P.assign_versions(g, _cfg(8, 2, 20))
    d = P.decompose_sequences(led, 20)
    assert sorted(x for s in d.sequences for x in s) == list(range(1, 21))
    assert d.version_difference_measured == 3
    assert all(v == 0 for v in P.staleness_report(led))  # zero-stash nF1B
    g = _grid(4, 2, 8, "pipedream")
    led = P.assign_versions(g, _cfg(4, 2, 8))
    st = P.staleness_report(led)
    assert max(st) > 0  # 1F1B consumes stashed versions


def test_partition_init_synthetic_match_reference():
    spec = P.NetworkSpec([784, 512, 256, 10], ["relu", "relu", "linear"],
                         "softmax_cross_entropy")
    st = P.partition_model(spec, 2)
    assert [s.first_layer for s in st] == [0, 1] and [len(s.layers) for s in st] == [1, 2]
    spec16 = P.NetworkSpec([4096] * 17, ["relu"] * 15 + ["linear"], "softmax_cross_entropy")
    assert [len(s.layers) for s in P.partition_model(spec16, 8)] == [2] * 8
    np.testing.assert_array_equal(P.init_network_params(spec, 1),
                                  O.init_network_params([784, 512, 256, 10], 1))
    d = P.make_synthetic_task(64, 5)
    x, y = O.make_synthetic_task(64, 5)
    np.testing.assert_array_equal(d.x, x)
    np.testing.assert_array_equal(d.y, y)
    data = P.make_classification_task(100, 13, 7, seed=7)
    x, y = O.make_classification_task(100, 13, 7, seed=7)
    np.testing.assert_array_equal(data.x, x)
    np.testing.assert_array_equal(data.y, y)
    with pytest.raises(P.DomainError):
        P.partition_model(P.NetworkSpec([3, 2], ["linear"]), 2)


def test_digest_matches_to_chars_restatement():
    rng = np.random.default_rng(0)
    vals = np.concatenate([rng.normal(size=200) * 10.0 ** rng.integers(-8, 8, 200),
                           [0.0, 1.0, 0.1, 1e-4, 1e16, -2.5, 5e-324, 1e22]])
    assert P.digest_values(vals) == O.params_digest(vals)
    for v in vals:
        assert P.format_double(float(v)) == O.format_double(float(v))


def test_parallel_digest_matches_serial_restatement():
    """Above 2^18 values the digest formats chunks on host threads and folds
    them in order; the text and hash are those of the serial reference loop
    (trainer.cpp:599-607), across chunk and ring boundaries."""
    rng = np.random.default_rng(1)
    n = (1 << 15) * 37 + 12345
    vals = (rng.normal(size=n) * 10.0 ** rng.integers(-6, 6, n)).astype(np.float32)
    vals = vals.astype(np.float64)
    assert P.digest_values(vals) == O.params_digest(vals)
