"""The reference-facing C++ API: a program written against the reference's
headers (tests/cpp/dropin_test.cpp) builds and links against the B200
library.  CPU: compile + host plan checks.  GPU: the training checks."""
import os
import pathlib
import shutil
import subprocess

import numpy as np
import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]
SRC = ROOT / "tests" / "cpp" / "dropin_test.cpp"
BIN = ROOT / "tests" / "cpp" / "dropin_test"
LIB = ROOT / "paper_2410_14312_b200" / "lib"


def _build():
    if BIN.exists() and BIN.stat().st_mtime >= SRC.stat().st_mtime and \
            BIN.stat().st_mtime >= (LIB / "libpipesim_b200.so").stat().st_mtime:
        return
    cxx = shutil.which("g++") or "g++"
    subprocess.run([cxx, "-std=c++20", "-O1", f"-I{ROOT / 'include'}", str(SRC),
                    f"-L{LIB}", "-lpipesim_b200", f"-Wl,-rpath,{LIB}", "-o", str(BIN)],
                   check=True)


def test_dropin_compiles_and_plan_checks_pass():
    _build()
    r = subprocess.run([str(BIN), "--plan-only"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert "all checks passed" in r.stdout


@pytest.mark.gpu
def test_dropin_training_on_gpu():
    _build()
    r = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "all checks passed" in r.stdout


# ---------------------------------------------------------------- numeric parity
PSRC = ROOT / "tests" / "cpp" / "dropin_parity.cpp"
PBIN = ROOT / "tests" / "cpp" / "dropin_parity"


def _build_parity():
    if PBIN.exists() and PBIN.stat().st_mtime >= PSRC.stat().st_mtime and \
            PBIN.stat().st_mtime >= (LIB / "libpipesim_b200.so").stat().st_mtime:
        return
    cxx = shutil.which("g++") or "g++"
    subprocess.run([cxx, "-std=c++20", "-O1", f"-I{ROOT / 'include'}", str(PSRC),
                    f"-L{LIB}", "-lpipesim_b200", f"-Wl,-rpath,{LIB}", "-o", str(PBIN)],
                   check=True)


def _fmt(v):
    from oracle import pipesim_np as O
    return " ".join(O.format_double(float(a)) for a in np.asarray(v).reshape(-1))


def _run_parity(cmd, tmp, widths, acts, loss, W, N, B, M, epochs, lr, seed, mode, x, y, p):
    _build_parity()
    ACT = ["linear", "relu", "tanh", "sigmoid"]
    inp, out = tmp / "in.txt", tmp / "out.txt"
    inp.write_text("\n".join([
        "widths " + " ".join(map(str, widths)),
        "acts " + " ".join(str(ACT.index(a)) for a in acts),
        f"loss {0 if loss == 'mse' else 1}",
        f"cfg {W} {N} {B} {M} {epochs} {lr!r} {seed} {mode}",
        f"x {x.shape[0]} {x.shape[1]} {_fmt(x)}",
        f"y {y.shape[0]} {y.shape[1]} {_fmt(y)}",
        f"params {_fmt(p)}"]) + "\n")
    r = subprocess.run([str(PBIN), cmd, str(inp), str(out)], capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    res = {}
    for line in out.read_text().splitlines():
        key, _, rest = line.partition(" ")
        if key.endswith(".log") or key.endswith(".checksum"):
            res.setdefault(key, []).append(rest)
        else:
            res[key] = np.array([float(t) for t in rest.split()]) if rest else np.zeros(0)
    return res


CPP_CASES = [
    ("c1_timeprest", [784, 512, 256, 10], ["relu", "relu", "linear"], "softmax_cross_entropy",
     2, 4, 256, 12, 0.05, 1, "timeprest", 1e-4, 1e-3, 8e-2),
    ("c1_pipedream", [784, 512, 256, 10], ["relu", "relu", "linear"], "softmax_cross_entropy",
     2, 4, 256, 12, 0.05, 1, "pipedream", 1e-4, 1e-3, 8e-2),
    # tiny nets at lr 0.1 over 2 epochs: the bars of test_gpu_pipeline's small nets
    ("deep4_mse", [30, 20, 16, 12, 10], ["relu", "sigmoid", "tanh", "linear"], "mse",
     4, 2, 12, 7, 0.1, 5, "timeprest", 3e-3, 5e-3, 1e-1),
    ("seq_w1", [64, 96, 10], ["tanh", "linear"], "softmax_cross_entropy",
     1, 1, 32, 5, 0.1, 3, "sequential", 3e-3, 5e-3, 1e-1),
]


@pytest.mark.gpu
@pytest.mark.parametrize("case", CPP_CASES, ids=[c[0] for c in CPP_CASES])
def test_cpp_train_epoch_matches_oracle(case, tmp_path):
    """The C++ drop-in pipesim::train_epoch (two epochs) against the fp64
    oracle on the same seeded inputs and schedule: losses, pins and consumed
    versions (exact), final weights, retained version_store keys and the
    to_text layout (proj/src/trainer.cpp:628-640) with its final checksum =
    params_digest of the returned stages."""
    from oracle import pipesim_np as O
    from paper_2410_14312_b200 import pipesim as P
    _, widths, acts, loss, W, N, B, M, lr, seed, mode, loss_tol, w_tol, dw_tol = case
    x, y = O.make_classification_task(M * B, widths[0], widths[-1], seed=7)
    p0 = O.init_network_params(widths, seed)
    res = _run_parity("train", tmp_path, widths, acts, loss, W, N, B, M, 2, lr, seed, mode, x, y,
                      p0)
    net = O.Net(widths, acts, loss)
    p = p0
    for e in (1, 2):
        ref = O.train_epoch(net, W, N, B, M, lr, x, y, p, mode=mode)
        p = ref["params"]
        np.testing.assert_array_equal(res[f"e{e}.pinned"],
                                      np.array(ref["pinned"]).reshape(-1))
        np.testing.assert_array_equal(res[f"e{e}.consumed"], ref["consumed"])
        rel = np.abs(res[f"e{e}.losses"] - ref["losses"]).max() / np.abs(ref["losses"]).max()
        assert rel < loss_tol, (e, rel)
        log = res[f"e{e}.log"]
        assert len(log) == M + 1
        for k, line in enumerate(log[:-1]):
            head = (f"epoch {e} mini {k + 1} loss "
                    f"{O.format_double(res[f'e{e}.losses'][k])} pinned")
            assert line.startswith(head) and " consumed " in line and " checksum " in line
    got = res["final.params"]
    assert np.linalg.norm(got - p) / np.linalg.norm(p) < w_tol
    dw = np.linalg.norm((got - p0) - (p - p0)) / np.linalg.norm(p - p0)
    assert dw < dw_tol, dw
    assert res["e2.log"][-1] == f"epoch 2 final checksum {P.digest_values(got)}"
    # version_store keys = the versions the retention rule keeps past the horizon
    if mode != "sequential":
        g = P._build(P.SimConfig(W, N, M, samples_per_mini_batch=B), mode)
        t = P.build_retention_timeline(P.assign_versions(g, P.SimConfig(W, N, M)), g)
        for s in range(W):
            want = sorted({int(v) for v, a, b in t.intervals[s] if b > t.horizon})
            keys = res[f"final.stage{s + 1}.versions"].astype(int).tolist()
            assert keys == want + [-1, M]


@pytest.mark.gpu
def test_cpp_network_gradient_fp32_verify(tmp_path):
    """pipesim::network_gradient / network_loss (trainer.hpp:169-173) in the
    fp32 FFMA verify precision against the fp64 oracle: relative 1e-4 on the
    gradient (recovered as W0 - W1 of an lr=1 step: absolute error ~ulp(W)),
    1e-5 on the loss."""
    from oracle import pipesim_np as O
    widths, acts, loss = [40, 32, 24, 10], ["tanh", "relu", "linear"], "softmax_cross_entropy"
    x, y = O.make_classification_task(48, 40, 10, seed=7)
    p0 = O.init_network_params(widths, 4)
    res = _run_parity("gradient", tmp_path, widths, acts, loss, 1, 1, 48, 1, 1, 1.0, 4,
                      "sequential", x, y, p0)
    net = O.Net(widths, acts, loss)
    g_ref = O.network_gradient(net, p0, x, y)
    rel = np.linalg.norm(res["gradient"] - g_ref) / np.linalg.norm(g_ref)
    assert rel < 1e-4, rel
    l_ref = O.network_loss(net, p0, x, y)
    assert abs(res["loss"][0] - l_ref) / abs(l_ref) < 1e-5


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["timeprest", "pipedream", "sequential"])
def test_cpp_resume_is_bit_identical(mode, tmp_path):
    """proj/tests/test_checkpoint.cpp:136-158: run_training for 3 epochs
    equals 2 epochs + resume from the per-stage checkpoints -- same last
    epoch log (losses, pins, checksums), final checksum and checkpoint files,
    byte for byte."""
    from oracle import pipesim_np as O
    widths, acts = [20, 16, 12, 4], ["relu", "tanh", "linear"]
    W = 1 if mode == "sequential" else 3
    x, y = O.make_classification_task(6 * 8, 20, 4, seed=7)
    res = _run_parity("resume", tmp_path, widths, acts, "softmax_cross_entropy", W, 2, 8, 6,
                      3, 0.1, 9, mode, x, y, O.init_network_params(widths, 9))
    assert res["first_epoch"].astype(int).tolist() == [1, 1, 3]
    assert res["full.checksum"] == res["resumed.checksum"]
    assert res["full.last.log"] == res["resumed.last.log"]
    np.testing.assert_array_equal(res["full.last.losses"], res["resumed.last.losses"])
    assert all(v == 1 for v in res["ckpt_equal"][1::2])
