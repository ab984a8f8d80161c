"""The fused two-layer dgrad (csrc/dgrad_chain.cuh) against the CPU oracle:
stages whose top layer is narrow (out <= 64) over an input of 64..256
columns, so the session emits one dgrad_chain launch for the top two
dgrads.  Covers K1 = 3 / 10 / 64, n1 = 64 / 128 / 192 / 256 (1-4 k-blocks of
the second GEMM), ragged row tiles (B = 100, 300), tanh / sigmoid / relu
gates, the delta to an upstream stage (W=2) and to a layer of the same stage
(W=1), MSE and softmax-CE.  Same bars as test_gpu_pipeline."""
import pathlib
import sys

import pytest

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent))
from test_gpu_pipeline import _check, _run_both  # noqa: E402

pytestmark = pytest.mark.gpu

CASES = [
    # name, widths, acts, loss, W, N, B, M, lr, seed
    ("seq_k64_n128", [96, 192, 128, 64], ["relu", "tanh", "linear"], "mse", 1, 2, 100, 4, 0.05, 4),
    ("w2_k3_n64_ragged", [300, 256, 64, 3], ["tanh", "sigmoid", "linear"],
     "softmax_cross_entropy", 2, 3, 300, 5, 0.05, 6),
    ("w2_k10_n192", [200, 320, 192, 10], ["relu", "relu", "linear"], "softmax_cross_entropy",
     2, 2, 128, 6, 0.05, 8),
    ("c2_seq_n256", [784, 512, 256, 10], ["relu", "relu", "linear"], "softmax_cross_entropy",
     1, 4, 256, 4, 0.05, 1),
]


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
@pytest.mark.parametrize("mode", ["timeprest", "sequential"])
def test_dgrad_chain_matches_oracle(case, mode):
    name, widths, acts, loss, W, N, B, M, lr, seed = case
    if W == 1 and mode != "sequential":
        pytest.skip("W=1 runs the sequential mode only (config.hpp:45-47)")
    stages, logs, refs, p0 = _run_both(widths, acts, loss, W, N, B, M, lr, seed, mode)
    _check(stages, logs, refs, p0, W, mode, loss_tol=3e-3, dw_tol=1e-1, w_tol=5e-3)


def test_dgrad_chain_is_emitted():
    """C1's stage 2 backward runs one fused launch instead of two dgrads:
    kernels per epoch drop by one per mini-batch against the same session
    with PIPESIM_DGRAD_CHAIN=0 (a subprocess: the switch is read once)."""
    import subprocess
    import sys
    code = ("from paper_2410_14312_b200 import pipesim as P\n"
            "net = P.NetworkSpec([784, 512, 256, 10], ['relu', 'relu', 'linear'], "
            "'softmax_cross_entropy')\n"
            "s = P.Session(net, 2, 4, 256, 6, 0.05, 'timeprest')\n"
            "print(s.kernels_per_epoch)\n")
    n = []
    for v in ("1", "0"):
        env = dict(__import__("os").environ, PIPESIM_DGRAD_CHAIN=v)
        out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True,
                             text=True, check=True).stdout.split()
        n.append(int(out[-1]))
    assert n[1] - n[0] == 6, n
