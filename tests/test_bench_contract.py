"""bench.py contract pieces that run without a GPU: the CPU reference arm's
sizing (every core, capped by memory), its JSON line (driver keys present,
value = aggregate of the concurrent runs), and the roofline byte count of the
wgrad+SGD launch (split masters: 8 B per parameter + operands)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_reference_runs_use_cores_within_memory():
    n = bench.ref_parallel_runs()
    assert 1 <= n <= (os.cpu_count() or 1)


def test_reference_arm_line(monkeypatch, capsys):
    # stand-in for the compiled reference step (the real one takes ~1 min)
    class _Fut:
        def result(self):
            return ("reference", 2.0)

    class _Pool:
        def __init__(self, *a, **k):
            pass

        def submit(self, fn, *a):
            return _Fut()

        def shutdown(self):
            pass

    import concurrent.futures as cf
    monkeypatch.setattr(cf, "ProcessPoolExecutor", _Pool)
    monkeypatch.setattr(bench, "ref_parallel_runs", lambda: 3)
    monkeypatch.setattr(os, "cpu_count", lambda: 8)
    monkeypatch.setattr(bench, "_ref_digest_seconds", lambda: 0.5)
    monkeypatch.delenv("RANK", raising=False)

    class A:
        gpus, steps, warmup = 1, 5, 3

    assert bench.run_reference_arm(A) == 0
    line = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "cpu_baseline", "e2e"):
        assert key in line, key
    samples = bench.REF_SAMPLE["M"] * bench.REF_SAMPLE["B"]
    assert line["impl"] == "reference"
    assert abs(line["value"] - 3 * samples / 2.0) < 1e-12  # aggregate of 3 runs
    assert line["cpu_baseline"]["cores"] == 3
    assert line["steps"] == 1 and line["warmup"] == 0  # what each process actually ran
    assert abs(line["cpu_baseline"]["digest_share"] - 0.25) < 1e-12
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]


def test_reference_arm_other_ranks_exit(monkeypatch):
    monkeypatch.setenv("RANK", "1")

    class A:
        gpus, steps, warmup = 2, 1, 1

    assert bench.run_reference_arm(A) == 0


def test_sgd_bytes_per_launch():
    n = bench.WIDTH
    assert bench.SGD_BYTES == n * n * 8 + 2 * 1024 * n * 2
