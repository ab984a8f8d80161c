"""BASELINE configs[4]: micro-batches N = 1..16 x workers W in
{2, 4, 8}.  Per cell:

  * version difference: the closed form floor((W+N-2)/N) and the value
    measured on the schedule's ledger (plan layer, strict mode), and N = 1
    must raise the reference's domain error (config.hpp:48-51);
  * slot-model idle fraction of the nF1B grid (metrics.cpp:71-72);
  * on the GPU: samples/s of one epoch of the 16 x 4096 MLP with the C3 micro
    size (B = 128 N rows, M = 2(W+N) mini-batches, all W stages on this GPU,
    CUDA graph) and the pipeline bubble from a profiled epoch,
    1 - sum(stage busy) / (W * makespan) (on one GPU the W stages share the
    SMs, so this is stage-stream occupancy, not idle hardware).

  python tools/sweep.py [--workers 2,4,8] [--micro 1-16] [--no-gpu] [--out FILE]
Writes JSON (one record per cell) and prints a markdown table.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_14312_b200 import pipesim as P  # noqa: E402


def plan_cell(W, N):
    rec = {"W": W, "N": N}
    M = 2 * (W + N)
    cfg = P.SimConfig(workers=W, micro_batches=N, mini_batches=M, samples_per_mini_batch=128 * N)
    try:
        P.validate(cfg)
    except P.DomainError as e:
        rec["domain_error"] = str(e)
        return rec
    grid = P.build_nf1b_schedule(cfg)
    ledger = P.assign_versions(grid, cfg)
    rec["M"] = M
    rec["closed_form_v"] = P.closed_form_v(W, N)
    rec["measured_v"] = P.measure_version_difference(ledger, strict=True)
    rec["horizon"] = grid.horizon()
    idle = int(np.sum(grid.cells[:, :, 0] == 0))
    rec["slot_idle_fraction"] = idle / (W * grid.horizon())
    return rec


def gpu_cell(rec, width=4096, layers=16):
    W, N, M = rec["W"], rec["N"], rec["M"]
    B = 128 * N
    net = P.NetworkSpec([width] * (layers + 1), ["relu"] * (layers - 1) + ["linear"],
                        "softmax_cross_entropy")
    s = P.Session(net, W, N, B, M, 0.05, "timeprest")
    s.load_params(P.init_network_params(net, 1))
    x, lab = P.make_classification_task(M * B, width, width, seed=7, as_labels=True,
                                        dtype=np.float32)
    s.upload(x, lab, y_labels=True)
    s.run_epoch()
    ms = min(s.run_epoch()["device_ms"] for _ in range(2))
    prof = s.profile_epoch()["profile"]
    s.close()
    rec["samples_per_s"] = M * B / (ms / 1000.0)
    rec["epoch_ms"] = ms
    rec["bubble"] = prof["bubble"]
    rec["profiled_epoch_ms"] = prof["makespan_ms"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workers", default="2,4,8")
    ap.add_argument("--micro", default="1-16")
    ap.add_argument("--no-gpu", action="store_true")
    ap.add_argument("--width", type=int, default=4096)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    Ws = [int(v) for v in args.workers.split(",")]
    lo, hi = (int(v) for v in args.micro.split("-"))
    rows = []
    t0 = time.time()
    for W in Ws:
        for N in range(lo, hi + 1):
            rec = plan_cell(W, N)
            if "domain_error" not in rec:
                assert rec["measured_v"] == (W - 1) // (N + 1) + 1  # test_ledger.cpp:115-128
                if not args.no_gpu:
                    gpu_cell(rec, args.width)
            rows.append(rec)
            print(json.dumps(rec), file=sys.stderr, flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump({"cells": rows, "seconds": time.time() - t0,
                       "network": f"{args.width} x 16 layers", "B": "128*N", "M": "2(W+N)"},
                      f, indent=1)
    print("| W | N | closed v | measured v | slot idle | samples/s | epoch ms | bubble |")
    print("|---|---|---|---|---|---|---|---|")
    for r in rows:
        if "domain_error" in r:
            print(f"| {r['W']} | {r['N']} | domain error | | | | | |")
            continue
        g = (f"{r['samples_per_s']:.0f} | {r['epoch_ms']:.2f} | {r['bubble']:.3f}"
             if "samples_per_s" in r else "- | - | -")
        print(f"| {r['W']} | {r['N']} | {r['closed_form_v']} | {r['measured_v']} | "
              f"{r['slot_idle_fraction']:.4f} | {g} |")


if __name__ == "__main__":
    main()
