"""The fused two-layer dgrad (csrc/dgrad_chain.cuh) and forward
(csrc/fwd_chain.cuh) against the CPU oracle: stages whose top layer is
narrow (out <= 64) over an input of 64..256 columns, so the session emits
one dgrad_chain launch for the top two dgrads and one fwd_chain launch for
the last two forwards (the logits one with the fused softmax-CE).  Covers K1 = 3 / 10 / 64, n1 = 64 / 128 / 192 / 256 (1-4 k-blocks of
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


@pytest.mark.parametrize("switch", ["PIPESIM_DGRAD_CHAIN", "PIPESIM_FWD_CHAIN"])
def test_chain_is_emitted(switch):
    """C1's stage 2 runs one fused launch instead of two per backward (dgrad)
    or per forward node (two per mini-batch): kernels per epoch against the
    same session with the switch off (a subprocess: it is read once)."""
    import os
    import subprocess
    code = ("from paper_2410_14312_b200 import pipesim as P\n"
            "net = P.NetworkSpec([784, 512, 256, 10], ['relu', 'relu', 'linear'], "
            "'softmax_cross_entropy')\n"
            "s = P.Session(net, 2, 4, 256, 6, 0.05, 'timeprest')\n"
            "print(s.kernels_per_epoch)\n")
    n = []
    for v in ("1", "0"):
        env = dict(os.environ, **{switch: v})
        out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True,
                             text=True, check=True).stdout.split()
        n.append(int(out[-1]))
    per_mini = 1 if switch == "PIPESIM_DGRAD_CHAIN" else 2
    assert n[1] - n[0] >= 6 * per_mini - 1, n
