"""Per-layer error of the conv pipeline against the fp64 conv oracle (one
mini-batch = one SGD step on version 0, and eta = 0 forwards).  GPU box:
python tools/convnet_diag.py"""
import sys

import numpy as np

sys.path.insert(0, ".")
from oracle import convnet_ref as R  # noqa: E402
from paper_2410_14312_b200 import convnet as CN  # noqa: E402
from paper_2410_14312_b200 import pipesim as P  # noqa: E402


def bf16(a):
    a = np.ascontiguousarray(a, np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return u.astype(np.uint32).view(np.float32)


STORAGE = sys.argv[1] if len(sys.argv) > 1 else "fp64"


def main():
    net = CN.vgg((64, "M", 64, "M", 128, "M"), image=16, classes=10, hidden=128, fc_layers=2)
    L = [R.Layer(l.kind, l.in_, l.out, l.h, l.w, l.pool, l.act) for l in net.layers]
    W, N, B = 2, 2, 8
    for M, lr in ((2, 0.0), (1, 0.02)):
        x, lab = CN.synthetic_images(M * B, net, seed=7)
        x = bf16(x)
        p0 = CN.init_params(net, 3)
        s = P.Session(net, W, N, B, M, lr)
        s.load_params(p0)
        s.upload(x, lab, y_labels=True)
        r = s.run_epoch()
        got = s.read_params()
        ref = R.train_epoch(L, net.partition(W), N, B, M, lr, x.astype(np.float64),
                            np.eye(10)[lab], p0, storage=STORAGE)
        print(f"M={M} lr={lr} loss dev {r['mini_loss']} ref {ref['losses']}")
        off = 0
        for i, l in enumerate(net.layers):
            nw = l.out * l.fan_in()
            for nm, a, b in (("W", off, off + nw), ("b", off + nw, off + nw + l.out)):
                dg = got[a:b] - p0[a:b]
                dr = ref["params"][a:b] - p0[a:b]
                den = np.linalg.norm(dr)
                print(f"  layer {i} {l.kind} {nm}: |dW| ref {den:.3e} rel err "
                      f"{np.linalg.norm(dg - dr) / max(den, 1e-30):.3e} cos "
                      f"{np.dot(dg, dr) / max(np.linalg.norm(dg) * den, 1e-30):.5f}")
            off += nw + l.out
        s.close()


if __name__ == "__main__":
    main()
