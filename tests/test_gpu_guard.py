"""Buffer-overrun guard: every session buffer is followed by a 4 KB canary
(PIPESIM_GUARD=1, read when the session is created) that the epoch must leave
intact -- kernels writing past a buffer inside the session's single arena
allocation are invisible to compute-sanitizer.  This found the conv
networks' Linear activation rows sized without their 8-aligned padding (the
loss kernel's padded dZ rows overran the slot)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

SCRIPT = r"""
import sys
sys.path.insert(0, {root!r})
import numpy as np
from paper_2410_14312_b200 import convnet as CN
from paper_2410_14312_b200 import pipesim as P
cases = []
for split in ([1, 2, 2], [1, 1, 1, 2], [2, 3]):
    net = CN.vgg((64, "M", 64, 128, "M"), image=16, classes=10, hidden=64, fc_layers=2)
    net.stage_layers = split
    cases.append((net, len(split), CN.synthetic_images(8 * 64, net, seed=7), CN.init_params(net, 1)))
for widths, acts, W in (([784, 512, 256, 10], ["relu", "relu", "linear"], 2),
                        ([30, 20, 16, 10], ["relu", "sigmoid", "linear"], 3),
                        ([96, 128, 128, 96, 64, 10], ["relu", "relu", "tanh", "relu", "linear"], 4)):
    net = P.NetworkSpec(widths, acts, "softmax_cross_entropy")
    cases.append((net, W, P.make_classification_task(8 * 64, widths[0], widths[-1], seed=7,
                  as_labels=True, dtype=np.float32), P.init_network_params(net, 1)))
for net, W, (x, lab), p0 in cases:
    for mode in ("timeprest", "pipedream", "sequential"):
        s = P.Session(net, W, 4, 64, 8, 0.002, mode=mode)
        s.load_params(p0)
        s.upload(x, lab, y_labels=True)
        s.run_epoch()
        s.run_epoch()
        s.close()
print("guards intact")
"""


def test_no_kernel_writes_past_a_session_buffer():
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PIPESIM_GUARD="1")
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=root)], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "guards intact" in r.stdout, r.stderr[-3000:]
