"""Throughput of the BASELINE configs other than the bench workload, on one
B200 (same executor, CUDA graph, data resident):

  C1  784-512-256-10 (ReLU, ReLU, linear; softmax-CE), W=2, N=4, B=256,
      nF1B, M=12 (= 2(W+N)) and M=32;
  C2  the same network at W=1 (sequential, the reference's only W=1 mode) and
      W=2 (timeprest);
  C3  16 x 4096 at W = 1, 2, 4, 8 stages on the one GPU (N=8, B=1024, M=32).

C1/C2 are launch-bound (0.6 GFLOP per mini-batch): the table gives us per
mini-batch next to the launch floor (kernel launches x ~2 us graph-node
cost), GEMM TFLOP/s and the fraction of the sustained bf16 peak.

  python tools/configs.py [--out FILE]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_14312_b200 import pipesim as P  # noqa: E402

SUSTAINED = 1384.0


def flops_per_sample(widths):
    p = [widths[i] * widths[i + 1] for i in range(len(widths) - 1)]
    return 2 * sum(p) + 2 * sum(p) + 2 * sum(p[1:])


def run(widths, acts, W, N, B, M, mode, reps=5):
    net = P.NetworkSpec(widths, acts, "softmax_cross_entropy")
    s = P.Session(net, W, N, B, M, 0.05, mode)
    s.load_params(P.init_network_params(net, 1))
    x, lab = P.make_classification_task(M * B, widths[0], widths[-1], seed=7, as_labels=True,
                                        dtype=np.float32)
    s.upload(x, lab, y_labels=True)
    for _ in range(3):
        s.run_epoch()
    ms = float(np.median([s.run_epoch()["device_ms"] for _ in range(reps)]))
    launches = s.kernels_per_epoch
    s.close()
    samples = M * B
    tf = flops_per_sample(widths) * samples / (ms / 1000.0) / 1e12
    return {"W": W, "N": N, "B": B, "M": M, "mode": mode, "epoch_ms": ms,
            "samples_per_s": samples / (ms / 1000.0), "us_per_mini": 1000.0 * ms / M,
            "launches_per_epoch": launches, "launch_floor_us_per_mini": 2.0 * launches / M,
            "gemm_tflops": tf, "frac_of_sustained": tf / SUSTAINED}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    c1 = ([784, 512, 256, 10], ["relu", "relu", "linear"])
    rows = []
    for name, W, mode, M in (("C1", 2, "timeprest", 12), ("C1", 2, "timeprest", 32),
                             ("C2", 1, "sequential", 12), ("C2", 2, "timeprest", 12),
                             ("C1-1F1B", 2, "pipedream", 12)):
        r = run(*c1, W, 4, 256, M, mode)
        r["config"] = name
        rows.append(r)
        print(json.dumps(r), file=sys.stderr, flush=True)
    c3 = ([4096] * 17, ["relu"] * 15 + ["linear"])
    for W in (1, 2, 4, 8):
        mode = "sequential" if W == 1 else "timeprest"
        r = run(*c3, W, 8, 1024, 32, mode, reps=3)
        r["config"] = f"C3 W={W}"
        rows.append(r)
        print(json.dumps(r), file=sys.stderr, flush=True)
    if args.out:
        json.dump(rows, open(args.out, "w"), indent=1)
    print("| config | W | mode | M | samples/s | us / mini-batch | launch floor us / mini | "
          "GEMM TFLOP/s | % sustained |")
    print("|---|---|---|---|---|---|---|---|---|")
    for r in rows:
        print(f"| {r['config']} | {r['W']} | {r['mode']} | {r['M']} | {r['samples_per_s']:.0f} | "
              f"{r['us_per_mini']:.1f} | {r['launch_floor_us_per_mini']:.1f} | "
              f"{r['gemm_tflops']:.1f} | {100 * r['frac_of_sustained']:.1f} |")


if __name__ == "__main__":
    main()
