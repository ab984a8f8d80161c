"""Run-to-run determinism of a conv pipeline epoch (lr > 0): which stage's
parameters differ between two eager runs."""
import os
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_2410_14312_b200 import convnet as CN
from paper_2410_14312_b200 import pipesim as P


CFG = tuple(int(v) if v != "M" else v for v in os.environ.get("CFG", "64,M,64,128,M").split(","))
FCL = int(os.environ.get("FCL", "2"))


def run(split, N=4, B=64, M=8, graph=False):
    net = CN.vgg(CFG, image=16, classes=10, hidden=64, fc_layers=FCL)
    net.stage_layers = split
    x, lab = CN.synthetic_images(M * B, net, seed=7)
    s = P.Session(net, len(split), N, B, M, 0.002, use_graph=graph)
    s.load_params(CN.init_params(net, 1))
    s.upload(x, lab, y_labels=True)
    r = s.run_epoch()
    out = (r["mini_loss"].copy(), s.read_params())
    s.close()
    return out, [l.param_count() for l in net.layers]


split = [int(v) for v in sys.argv[1].split(",")] if len(sys.argv) > 1 else [1, 1, 1, 2]
bad = 0
for rep in range(3):
    (a, sizes), _ = run(split)[0:2], None
    b = run(split)[0]
    off, diffs = 0, []
    for n in sizes:
        diffs.append(float(np.abs(a[1][off:off + n] - b[1][off:off + n]).max()))
        off += n
    print(os.environ.get("TAG", ""), split, "per-layer max param diff", ["%.1e" % d for d in diffs])
