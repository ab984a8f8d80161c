"""fp32 FFMA verify precision (verify_fp32.cu): the same pipeline executor
with every Linear contraction on the CUDA cores in fp32 and fp32 activations,
deltas and weight versions.  Against the fp64 oracle on the same seeded
inputs and schedule the bar is fp32 rounding:

  * version traces: bit-exact (as in the bf16 path);
  * per-mini-batch loss: relative 1e-5;
  * final weights: relative 1e-6 (3e-5 on the ReLU C1 net, see below);
  * weight deltas ||dW - dW_ref|| / ||dW_ref||: 1e-4 (vs 8e-2 for bf16
    operands: the gap the bf16 tolerances stand for); 5e-3 on C1, where a
    ReLU pre-activation within fp32 rounding of 0 can flip a unit's gradient.
"""
import numpy as np
import pytest

from paper_2410_14312_b200 import pipesim as P

from test_gpu_pipeline import C1, SMALL, _check, _run_both  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _fp32():
    old = P.b200.precision
    P.b200.precision = "fp32"
    yield
    P.b200.precision = old


@pytest.mark.parametrize("case", SMALL, ids=[c[0] for c in SMALL])
@pytest.mark.parametrize("mode", ["timeprest", "pipedream", "sequential"])
def test_verify_small_networks(case, mode):
    _, widths, acts, loss, W, N, B, M, lr, seed = case
    stages, logs, refs, p0 = _run_both(widths, acts, loss, W, N, B, M, lr, seed, mode, epochs=2)
    _check(stages, logs, refs, p0, W, mode, loss_tol=1e-5, dw_tol=1e-4, w_tol=1e-6)


@pytest.mark.parametrize("mode,W", [("timeprest", 2), ("pipedream", 2), ("sequential", 1)])
def test_verify_c1_mnist_shaped(mode, W):
    stages, logs, refs, p0 = _run_both(*C1, W, 4, 256, 12, 0.05, 1, mode)
    # C1 is a ReLU net: a pre-activation within fp32 rounding of 0 takes the
    # other side of the kink than in fp64 and switches that unit's gradient
    # (seen once here: sequential M=12 from mini 10 on, losses still 3e-7,
    # dW 3e-3; M = 10, 11, 14 give 3e-5).  The tight dW bar is the smooth
    # small networks' above.
    _check(stages, logs, refs, p0, W, mode, loss_tol=1e-6, dw_tol=5e-3, w_tol=3e-5)


def test_verify_is_tighter_than_bf16():
    """The same C1 run in both precisions: the verify path's weight-delta
    error is orders of magnitude below the bf16 tensor-core path's."""
    errs = {}
    for prec in ("bf16", "fp32"):
        P.b200.precision = prec
        stages, logs, refs, p0 = _run_both(*C1, 2, 4, 256, 12, 0.05, 1, "timeprest")
        got = P.gather_network_params(stages)
        want = refs[-1]["params"]
        errs[prec] = np.linalg.norm((got - p0) - (want - p0)) / np.linalg.norm(want - p0)
    assert errs["fp32"] < errs["bf16"] / 100, errs
