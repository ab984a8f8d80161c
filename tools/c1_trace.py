"""In-graph kernel timeline of C1 (784-512-256-10, W=2, N=4, B=256, M=32,
TiMePReSt): torch.profiler (CUPTI) records every kernel of one graph-launched
epoch with its stream and device timestamps; prints the kernels of three
steady-state mini-batches and per-kernel-name mean durations.
GPU box: python tools/c1_trace.py [--mode timeprest|pipedream] [--out trace.json]"""
import argparse
import collections
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_14312_b200 import pipesim as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", default="timeprest")
    ap.add_argument("--out", default=None)
    ap.add_argument("--M", type=int, default=32)
    args = ap.parse_args()
    widths, acts = [784, 512, 256, 10], ["relu", "relu", "linear"]
    net = P.NetworkSpec(widths, acts, "softmax_cross_entropy")
    W, N, B, M = 2, 4, 256, args.M
    s = P.Session(net, W, N, B, M, 0.05, args.mode)
    s.load_params(P.init_network_params(net, 1))
    x, lab = P.make_classification_task(M * B, 784, 10, seed=7, as_labels=True, dtype=np.float32)
    s.upload(x, lab, y_labels=True)
    for _ in range(3):
        s.run_epoch()
    ms = [s.run_epoch()["device_ms"] for _ in range(5)]
    print("graph epoch us/mini", 1000 * np.median(ms) / M)
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        s.run_epoch()
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    rows = []
    for e in evs:
        rows.append({"name": e.name, "t0": e.time_range.start, "t1": e.time_range.end,
                     "stream": getattr(e, "device_resource_id", -1)})
    rows.sort(key=lambda r: r["t0"])
    if not rows:
        print("no kernel events")
        return
    t_first, t_last = rows[0]["t0"], rows[-1]["t1"]
    print("kernels", len(rows), "span us", t_last - t_first, "per mini", (t_last - t_first) / M)
    by = collections.defaultdict(list)
    for r in rows:
        by[r["name"][:60]].append(r["t1"] - r["t0"])
    for k, v in sorted(by.items(), key=lambda kv: -sum(kv[1])):
        print(f"{len(v):5d} {np.mean(v):7.2f} us {sum(v):8.1f} {k}")
    # three steady-state mini-batches (middle of the epoch)
    mid = t_first + (t_last - t_first) * 0.5
    span = 3 * (t_last - t_first) / M
    print("--- window", span, "us")
    for r in rows:
        if mid <= r["t0"] <= mid + span:
            print(f"{r['t0'] - mid:8.2f} {r['t1'] - r['t0']:6.2f} s{r['stream']:<4} {r['name'][:70]}")
    if args.out:
        with open(args.out, "w") as f:
            json.dump(rows, f)


if __name__ == "__main__":
    main()
