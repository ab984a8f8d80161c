"""Split fp32 masters vs fp32 masters after one and four mini-batches: relative
difference of the weight deltas (timing-independent check of the split
update).   python tools/split_check.py"""
import os
import subprocess
import sys
import numpy as np

code = r'''
import sys, numpy as np
sys.path.insert(0, ".")
from paper_2410_14312_b200 import pipesim as P
M = int(sys.argv[2])
net = P.NetworkSpec([512] * 4, ["relu", "relu", "linear"], "softmax_cross_entropy")
p0 = P.init_network_params(net, 1)
x, lab = P.make_classification_task(M * 512, 512, 512, seed=7, as_labels=True, dtype=np.float32)
s = P.Session(net, 2, 4, 512, M, 0.05, "timeprest")
s.load_params(p0); s.upload(x, lab, y_labels=True)
r = s.run_epoch()
np.save(sys.argv[1], np.concatenate([r["mini_loss"], s.read_params() - p0.astype(np.float32)]))
'''
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for M in (1, 4):
    outs = []
    for flag in ("1", "0"):
        f = f"/tmp/split_{flag}_{M}.npy"
        subprocess.run([sys.executable, "-c", code, f, str(M)], check=True, cwd=root,
                       env=dict(os.environ, PIPESIM_SPLIT_MASTER=flag))
        outs.append(np.load(f))
    a, b = outs
    d = a[M:] - b[M:]
    print(f"M={M}: loss diff {np.abs(a[:M] - b[:M]).max():.3e}, dW rel {np.linalg.norm(d) / np.linalg.norm(b[M:]):.3e}, "
          f"max |d| {np.abs(d).max():.3e}, n differing {int((d != 0).sum())} of {d.size}")
