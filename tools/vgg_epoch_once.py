"""One VGG-16 epoch (ncu launch-list target): python tools/vgg_epoch_once.py W N B M"""
import sys

sys.path.insert(0, ".")
from paper_2410_14312_b200 import convnet as CN  # noqa: E402
from paper_2410_14312_b200 import pipesim as P  # noqa: E402

W, N, B, M = (int(v) for v in sys.argv[1:5])
net = CN.vgg16()
s = P.Session(net, W, N, B, M, 1e-4)
s.load_params(CN.init_params(net, 1))
x, lab = CN.synthetic_images(M * B, net, seed=7)
s.upload(x, lab, y_labels=True)
r = s.run_epoch()
print("epoch ms", r["device_ms"], "loss", r["mini_loss"][:2])
