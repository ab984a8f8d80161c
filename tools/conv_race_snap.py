"""First committed version that differs between two eager runs (snapshots)."""
import os
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_2410_14312_b200 import convnet as CN
from paper_2410_14312_b200 import pipesim as P

split = [int(v) for v in sys.argv[1].split(",")]
snaps = os.environ.get("SNAPS", "1") == "1"


def run():
    net = CN.vgg((64, "M", 64, 128, "M"), image=16, classes=10, hidden=64, fc_layers=2)
    net.stage_layers = split
    x, lab = CN.synthetic_images(8 * 64, net, seed=7)
    s = P.Session(net, len(split), 4, 64, 8, 0.002, use_graph=False, snapshots=snaps)
    s.load_params(CN.init_params(net, 1))
    s.upload(x, lab, y_labels=True)
    r = s.run_epoch()
    out = {}
    if snaps:
        for st in range(1, len(split) + 1):
            for v in range(1, 9):
                out[(st, v)] = s.snapshot(st, v)
    out["final"] = s.read_params()
    out["dev"] = (r["dev_fwd"].copy(), r["dev_bwd"].copy())
    s.close()
    return out


a, b = run(), run()
print(split, "snapshots" if snaps else "", "final diff", np.abs(a["final"] - b["final"]).max(),
      "traces equal", all(np.array_equal(p, q) for p, q in zip(a["dev"], b["dev"])))
if snaps:
    for st in range(1, len(split) + 1):
        print("  stage", st, ["%.0e" % np.abs(a[(st, v)] - b[(st, v)]).max() for v in range(1, 9)])
    # where the last stage first differs
    st = len(split)
    for v in range(1, 9):
        d = np.abs(a[(st, v)] - b[(st, v)])
        if d.max() > 0:
            idx = np.nonzero(d)[0]
            print("  last stage first differs at version", v, "elements", idx[:20], "count", len(idx),
                  "size", d.size)
            break
