"""VGG-16 pipeline throughput on one B200 (BASELINE configs[3]): 224x224x3
synthetic ImageNet-shaped images, 1000 classes, nF1B at W stages sharing the
GPU, CUDA graph, data resident (plus one epoch from page-locked host
buffers).  Reports images/s, the step's conv+FC TFLOP/s against the sustained
bf16 peak, the partition and the per-stage bubble.

  python tools/vgg_bench.py [--W 4 8] [--N 4] [--B 64] [--M 32] [--out FILE]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_14312_b200 import convnet as CN  # noqa: E402
from paper_2410_14312_b200 import pipesim as P  # noqa: E402


def peaks():
    try:
        with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                               "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return d.get("bf16_tflops_sustained", 1384.0)
    except OSError:
        return 1384.0


def run(W, N, B, M, reps, image=224, lr=1e-4, profile=False, mode="timeprest"):
    net = CN.vgg16(image=image)
    s = P.Session(net, W, N, B, M, lr, mode=mode)
    s.load_params(CN.init_params(net, 1))
    x, lab = CN.synthetic_images(M * B, net, seed=7)
    s.upload(x, lab, y_labels=True)
    first = s.run_epoch()
    for _ in range(2):
        s.run_epoch()
    ms = [s.run_epoch()["device_ms"] for _ in range(reps)]
    last = s.run_epoch()
    out = {"W": W, "N": N, "B": B, "M": M, "mode": mode, "image": image,
           "partition": net.partition(W), "epoch_ms": float(np.median(ms)),
           "epoch_ms_all": [float(v) for v in ms], "kernels_per_epoch": s.kernels_per_epoch,
           "device_gb": s.device_bytes / 1e9,
           "loss_first": [float(v) for v in first["mini_loss"][:3]],
           "loss_last": [float(v) for v in last["mini_loss"][-3:]],
           "finite": bool(np.all(np.isfinite(last["mini_loss"])))}
    samples = M * B
    out["images_per_s"] = samples / (out["epoch_ms"] / 1000.0)
    out["tflops"] = net.flops_per_sample() * samples / (out["epoch_ms"] / 1000.0) / 1e12
    out["frac_of_sustained"] = out["tflops"] / peaks()
    out["gflop_per_image"] = net.flops_per_sample() / 1e9
    if profile:
        pr = s.profile_epoch()["profile"]
        out["bubble"] = pr["bubble"]
        out["busy_ms"] = pr["busy_ms"]
        out["profile_makespan_ms"] = pr["makespan_ms"]
    s.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--W", type=int, nargs="+", default=[4, 8])
    ap.add_argument("--N", type=int, default=4)
    ap.add_argument("--B", type=int, default=64)
    ap.add_argument("--M", type=int, default=32)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--image", type=int, default=224)
    ap.add_argument("--profile", action="store_true")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    rows = []
    for W in args.W:
        r = run(W, args.N, args.B, args.M, args.reps, args.image, profile=args.profile)
        print(json.dumps(r), flush=True)
        rows.append(r)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
