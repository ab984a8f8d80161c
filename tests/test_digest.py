"""The reference's params_digest (trainer.cpp:599-607: shortest round-trip
decimals of every parameter, '\\n'-separated, folded with FNV-1a 64,
text.cpp:24-52) computed on the device: the formatter (shortest.cuh) is
pinned to std::to_chars on the host, and the device digest (digest_dev.cu:
parallel formatting + nibble-map / affine decomposition of the FNV fold) must
equal the serial host digest bit for bit."""
import ctypes as C
import pathlib
import subprocess

import numpy as np
import pytest

from paper_2410_14312_b200 import _native as N
from paper_2410_14312_b200 import pipesim as P

ROOT = pathlib.Path(__file__).resolve().parents[1]
CSRC = ROOT / "paper_2410_14312_b200" / "csrc"


def test_host_shortest_matches_to_chars(tmp_path):
    exe = tmp_path / "shortest_check"
    subprocess.run(["g++", "-O2", "-std=c++20", f"-I{CSRC}", str(ROOT / "tests/cpp/shortest_check.cpp"),
                    "-o", str(exe)], check=True)
    r = subprocess.run([str(exe), "1500000"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:]
    assert "0 mismatches" in r.stdout


def test_python_format_double_integers():
    # large / integral values print their exact digits, like std::to_chars
    assert P.format_double(float(np.float32(2.9871056e18))) == "2987105636463935488"
    assert P.format_double(10.0) == "10"
    assert P.format_double(1e22) == "1e+22"
    assert P.format_double(-1.6827471309251281e+20) == "-168274713092512808960"
    assert P.format_double(1e23) == "1e+23"
    assert P.format_double(-0.0) == "-0"
    assert P.format_double(1e-05) == "1e-05"


def _host_digest(v32):
    v = np.ascontiguousarray(v32, np.float32).astype(np.float64)
    out = C.create_string_buffer(17)
    N.check(N.lib().pb_params_digest(v.ctypes.data_as(C.POINTER(C.c_double)), len(v), out))
    return out.value.decode()


def _device_digest(v32):
    v = np.ascontiguousarray(v32, np.float32)
    out = C.create_string_buffer(17)
    ms = C.c_float()
    N.check(N.lib().pb_device_digest_f32(v.ctypes.data_as(C.POINTER(C.c_float)), len(v), out,
                                         C.byref(ms)))
    return out.value.decode(), ms.value


def _samples(n, seed):
    g = np.random.default_rng(seed)
    bits = g.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32).view(np.float32)
    bits = bits[np.isfinite(bits)]
    w = g.uniform(-0.05, 0.05, n).astype(np.float32)
    edges = np.ldexp(np.float32(1), np.arange(-149, 128)).astype(np.float32)
    v = np.concatenate([bits, w, edges, -edges, np.arange(1000, dtype=np.float32),
                        np.float32([0.0, -0.0, 0.1, 1e-7, 3.4028235e38])])
    return g.permutation(v)


@pytest.mark.gpu
def test_device_format_matches_to_chars():
    v = _samples(100_000, 3)
    out = C.create_string_buffer(32 * len(v))
    N.check(N.lib().pb_device_format_f32(v.ctypes.data_as(C.POINTER(C.c_float)), len(v), out))
    raw = out.raw
    for i, x in enumerate(v):
        got = raw[32 * i:32 * i + 32].split(b"\0", 1)[0].decode()
        assert got == P.format_double(float(x)), (float(x), got)


@pytest.mark.gpu
@pytest.mark.parametrize("n", [0, 1, 4095, 4097, 1_000_003])
def test_device_digest_matches_serial_fold(n):
    v = _samples(n, n)[:n]
    assert _device_digest(v)[0] == _host_digest(v)


@pytest.mark.gpu
def test_device_digest_multi_segment():
    # > one 4M-value segment: the FNV state carries across segments
    g = np.random.default_rng(11)
    v = g.normal(0, 0.02, 9_000_000).astype(np.float32)
    dev, ms = _device_digest(v)
    assert dev == _host_digest(v)


# ---------------------------------------------------------------- in-epoch
def _versions_at_digest(W, N, B, M, mode):
    """[k-1][s-1]: the version stage s holds when mini k's digest is taken
    (stage-1 commit of k; stage s > 1: its latest commit in an earlier slot,
    trainer.cpp:492-501), then the final row (all M)."""
    if mode == "sequential":
        rows = [[k] * W for k in range(1, M + 1)]
    else:
        cfg = P.SimConfig(workers=W, micro_batches=N, mini_batches=M, samples_per_mini_batch=B)
        g = P.build_nf1b_schedule(cfg) if mode == "timeprest" else P.build_1f1b_schedule(cfg)
        rows = []
        for k in range(1, M + 1):
            t1 = g.backward_slot(k, 1)
            row = [k]
            for s in range(2, W + 1):
                row.append(max([u for u in range(1, M + 1) if g.backward_slot(u, s) < t1],
                               default=0))
            rows.append(row)
    return rows + [[M] * W]


def _session(widths, acts, W, N, B, M, mode, **kw):
    net = P.NetworkSpec(widths, acts, "softmax_cross_entropy")
    s = P.Session(net, W, N, B, M, 0.05, mode, **kw)
    s.load_params(P.init_network_params(net, 1))
    x, lab = P.make_classification_task(M * B, widths[0], widths[-1], seed=7, as_labels=True,
                                        dtype=np.float32)
    s.upload(x, lab, y_labels=True)
    return s


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["timeprest", "pipedream", "sequential"])
@pytest.mark.parametrize("graph", [True, False])
def test_in_epoch_digests_match_snapshots(mode, graph):
    """Every per-mini-batch digest taken inside the epoch equals the serial
    host digest of the same fp32 masters (the per-commit snapshots)."""
    W, N, B, M = 4, 2, 64, 12
    s = _session([96, 128, 128, 96, 64, 10], ["relu", "relu", "tanh", "relu", "linear"],
                 W, N, B, M, mode, snapshots=True, digests=True, use_graph=graph)
    for epoch in range(2):  # the second epoch replays the graph
        s.run_epoch()
        dig = s.digests()
        for k, row in enumerate(_versions_at_digest(W, N, B, M, mode)):
            vals = np.concatenate([s.snapshot(st + 1, v) for st, v in enumerate(row)])
            assert dig[k] == _host_digest(vals), (epoch, k + 1, row)
        assert s.params_digest(M) == dig[M]
    s.close()


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["timeprest", "pipedream"])
def test_in_epoch_digests_split_masters(mode):
    """Split fp32 masters (bf16 hi in the version pool + 16-bit residual): the
    digest joins them on the fly; the last mini-batch's and the final digest
    equal the host digest of the read-back masters."""
    W, N, B, M = 4, 2, 256, 12
    widths = [256, 256, 384, 256, 512, 256]
    s = _session(widths, ["relu", "tanh", "relu", "relu", "linear"], W, N, B, M, mode,
                 digests=True)
    net = P.NetworkSpec(widths, ["linear"] * 5, "softmax_cross_entropy")
    p0 = P.init_network_params(net, 1).astype(np.float32)
    assert s.params_digest(0) == _host_digest(p0)
    s.run_epoch()
    dig = s.digests()
    rows = _versions_at_digest(W, N, B, M, mode)
    vals = np.concatenate([s.read_version(st + 1, v) for st, v in enumerate(rows[M - 1])])
    assert dig[M - 1] == _host_digest(vals)
    assert dig[M] == _host_digest(s.read_params())
    s.close()
