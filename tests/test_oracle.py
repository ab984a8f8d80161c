"""Pins the CPU oracle (oracle/pipesim_np.py, a numpy restatement of the
reference) against the reference's golden files and against the compiled
reference itself (oracle/_ref, when built).  CPU only."""
import json
import pathlib

import numpy as np
import pytest

from oracle import pipesim_np as O
from oracle import ref

GOLD = pathlib.Path(__file__).resolve().parent / "golden"
REF_GOLD = pathlib.Path("/root/reference/proj/tests/golden")
TIMELINES = ["4-2-7", "4-4-4", "3-2-6", "5-2-6", "5-3-6"]


@pytest.mark.parametrize("name", TIMELINES)
def test_timeline_goldens(name):
    w, n, m = map(int, name.split("-"))
    text = O.render_ascii(O.build_schedule(w, n, m))
    assert text == (GOLD / f"timeline-{name}.txt").read_text()
    if REF_GOLD.exists():  # the reference's own golden file, byte for byte
        assert text == (REF_GOLD / f"timeline-{name}.txt").read_text()


def _plan_cases():
    return json.loads((GOLD / "plan_goldens.json").read_text())


def test_plan_goldens_restatement():
    modes = {0: "timeprest", 1: "pipedream"}
    for c in _plan_cases():
        w, n, m, mode = c["W"], c["N"], c["M"], modes[c["mode"]]
        g = O.build_schedule(w, n, m, mode)
        assert g.tolist() == c["grid"], (w, n, m, mode)
        led = O.assign_versions(g, w, n, m, mode)
        for key in ("commits", "pins", "consumptions", "update_source", "full_commit_slot"):
            assert np.asarray(led[key]).tolist() == c[key], (key, w, n, m, mode)
        iv, peak = O.retention_timeline(g, led, w, m, mode)
        assert iv.tolist() == c["retention"] and peak.tolist() == c["peak"]
        assert O.closed_form_v(w, n) == c["v_closed"]
        if c["v_measured"] is not None:
            assert O.measure_version_difference(led["update_source"], w, n, m,
                                                strict=False) == c["v_measured"]


def test_version_difference_table():
    """SURVEY Appendix A / proj/tests/test_ledger.cpp:115-128: measured v is
    floor((W-1)/(N+1))+1 and diverges from the closed form at (8,2), (8,3)."""
    for w in (2, 4, 8):
        for n in range(2, 17):
            m = 2 * (w + n)
            g = O.build_schedule(w, n, m)
            led = O.assign_versions(g, w, n, m)
            v = O.measure_version_difference(led["update_source"], w, n, m)
            assert v == (w - 1) // (n + 1) + 1
    assert O.closed_form_v(8, 2) == 4 and O.closed_form_v(8, 3) == 3


TRAIN = {
    "demo": ([2, 8, 2], [2, 0], 1, 2, 2, 10, 6, 0.05, 42),
    "deep4": ([2, 6, 6, 6, 2], [2, 2, 2, 0], 1, 4, 2, 4, 7, 0.05, 2),
    "scalar": ([1, 1, 1], [0, 0], 0, 2, 2, 2, 2, 0.2, 11),
    "mixed": ([30, 20, 16, 10], [1, 3, 0], 0, 3, 4, 12, 10, 0.1, 5),
    "relu8": ([64, 48, 48, 40, 40, 32, 32, 24, 16], [1] * 7 + [0], 1, 8, 8, 64, 6, 0.05, 3),
}


@pytest.mark.parametrize("name", sorted(TRAIN))
@pytest.mark.parametrize("mode", ["timeprest", "pipedream", "sequential"])
def test_train_goldens_restatement(name, mode):
    """Two epochs of the restated replay vs the fp64 reference (1e-12)."""
    widths, acts, loss, W, N, B, M, lr, seed = TRAIN[name]
    g = np.load(GOLD / "train_goldens.npz")
    key = f"{name}.{mode}"
    net = O.Net(widths, acts, loss)
    x, y = O.make_classification_task(M * B, widths[0], widths[-1], seed=7)
    p = O.init_network_params(widths, seed)
    losses = []
    for _ in range(2):
        r = O.train_epoch(net, W, N, B, M, lr, x, y, p, mode=mode, observe=True)
        p = r["params"]
        losses.append(r["losses"])
        assert np.array_equal(np.array(r["pinned"]), g[key + ".pinned"][-1])
        assert np.array_equal(r["consumed"], g[key + ".consumed"][-1])
    np.testing.assert_allclose(p, g[key + ".params"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(np.array(losses), g[key + ".losses"], rtol=1e-12, atol=1e-13)
    if mode != "sequential":  # version store == retention at every slot (last epoch)
        assert np.array_equal(r["held"], g[key + ".held"])
    # the reference's own log text carries the same losses
    log = bytes(g[key + ".log"]).decode()
    logged = [float(line.split(" loss ")[1].split()[0]) for line in log.splitlines()
              if " loss " in line]
    np.testing.assert_allclose(logged, np.array(losses).reshape(-1), rtol=1e-12)
    # ... and its final checksum is the digest of the final parameters, in the
    # reference's FNV-1a variant (offset basis 1469598103934665603, text.cpp:39-51)
    final = log.splitlines()[-1]
    assert final.startswith("epoch 2 final checksum ")
    want = final.split()[-1]
    assert O.params_digest(g[key + ".params"]) == want
    from paper_2410_14312_b200 import pipesim as P
    assert P.digest_values(g[key + ".params"]) == want


def test_c1_summary_restatement():
    summ = json.loads((GOLD / "c1_summary.json").read_text())
    widths, acts = [784, 512, 256, 10], ["relu", "relu", "linear"]
    net = O.Net(widths, acts, "softmax_cross_entropy")
    x, y = O.make_classification_task(12 * 256, 784, 10, seed=7)
    p0 = O.init_network_params(widths, 1)
    for key, s in summ.items():
        mode, w = key.split(".")
        r = O.train_epoch(net, int(w[1:]), 4, 256, 12, 0.05, x, y, p0, mode=mode)
        np.testing.assert_allclose(r["losses"], s["losses"], rtol=1e-12)
        d = r["params"] - p0
        assert abs(np.linalg.norm(d) - s["delta_norm"]) < 1e-12 * s["delta_norm"] + 1e-15
        assert np.array(r["pinned"]).reshape(-1).tolist() == \
            np.array(s["pinned"]).reshape(-1).tolist()


def test_rng_and_synthetic_task():
    for seed in (0, 1, 7, 12345678901234):
        g = O.MT19937_64(seed)
        a = g.draw(1000)
        assert a.dtype == np.uint64
    if ref.available():
        np.testing.assert_array_equal(O.init_network_params([5, 7, 3], 9),
                                      ref.init_params([5, 7, 3], [2, 0], 0, 9))
        x, y = O.make_synthetic_task(40, 3)
        rx, ry = ref.synthetic(40, 3)
        np.testing.assert_array_equal(x, rx)
        np.testing.assert_array_equal(y, ry)


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
def test_restatement_vs_compiled_reference_sweep():
    for mode, mid in (("timeprest", 0), ("pipedream", 1)):
        for w in range(2, 9):
            for n in (2, 3, 5, 8):
                m = 2 * (w + n)
                g = O.build_schedule(w, n, m, mode)
                assert np.array_equal(g, ref.schedule(w, n, m, mid))
                led = O.assign_versions(g, w, n, m, mode)
                rl = ref.ledger(w, n, m, mid)
                for k in rl:
                    assert np.array_equal(np.asarray(led[k]).reshape(rl[k].shape), rl[k])


def test_format_double_examples():
    cases = {1.0: "1", 0.1: "0.1", 1e-05: "1e-05", 0.0001: "1e-04", 0.001: "0.001",
             123456789012345680000.0: "123456789012345680000", 1e22: "1e+22",
             -2.5: "-2.5", 0.0: "0", 1.5e-300: "1.5e-300", 2.0 ** -1074: "5e-324",
             100.0: "100", 1e16: "1e+16", 12345.678: "12345.678"}
    for v, s in cases.items():
        assert O.format_double(v) == s, (v, O.format_double(v), s)
