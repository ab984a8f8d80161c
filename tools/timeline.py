"""Node timeline of one profiled epoch of the benchmark step (profile_epoch:
CUDA events around every node on its stream, no graph): concurrency over
time, per-stage busy fraction, fill / steady / drain split, and a Chrome
trace (chrome://tracing / Perfetto) of the nodes.

  python tools/timeline.py [--out-json FILE] [--trace FILE]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_14312_b200 import pipesim as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out-json", default=None)
    ap.add_argument("--trace", default=None)
    ap.add_argument("--W", type=int, default=8)
    ap.add_argument("--M", type=int, default=32)
    args = ap.parse_args()
    W, N, B, M = args.W, 8, 1024, args.M
    net = P.NetworkSpec([4096] * 17, ["relu"] * 15 + ["linear"], "softmax_cross_entropy")
    s = P.Session(net, W, N, B, M, 0.05, "timeprest")
    s.load_params(P.init_network_params(net, 1))
    x, lab = P.make_classification_task(M * B, 4096, 4096, seed=7, as_labels=True,
                                        dtype=np.float32)
    s.upload(x, lab, y_labels=True)
    s.run_epoch()
    graph_ms = s.run_epoch()["device_ms"]
    s.profile_epoch()
    prof = s.profile_epoch()["profile"]
    s.close()
    nodes = prof["nodes"]
    T = prof["makespan_ms"]
    grid = np.linspace(0, T, 2001)
    conc = np.zeros(len(grid))
    for n in nodes:
        conc += (grid >= n["start_ms"]) & (grid < n["end_ms"])
    first_bwd_end = min(n["end_ms"] for n in nodes if not n["fwd"])
    last_fwd_start = max(n["start_ms"] for n in nodes if n["fwd"])
    summary = {
        "graph_epoch_ms": graph_ms, "profiled_epoch_ms": T, "bubble": prof["bubble"],
        "mean_active_nodes": float(conc.mean()),
        "fraction_time_with_0_active": float((conc == 0).mean()),
        "fraction_time_with_1_active": float((conc == 1).mean()),
        "fraction_time_with_ge3_active": float((conc >= 3).mean()),
        "fill_ms (until the first backward ends)": first_bwd_end,
        "drain_ms (after the last forward starts)": T - last_fwd_start,
        "stage_busy_fraction": [b / T for b in prof["busy_ms"]],
    }
    print(json.dumps(summary, indent=1))
    if args.out_json:
        json.dump({"summary": summary, "nodes": nodes}, open(args.out_json, "w"))
    if args.trace:
        ev = []
        for n in nodes:
            name = (f"fwd k{n['mini']} micro {n['micro'][0] + 1}-{n['micro'][1] + 1}" if n["fwd"]
                    else f"bwd k{n['mini']}")
            ev.append({"name": name, "ph": "X", "pid": 0, "tid": n["stage"] * 2 + (0 if n["fwd"] else 1),
                       "ts": 1000 * n["start_ms"], "dur": 1000 * (n["end_ms"] - n["start_ms"])})
        json.dump({"traceEvents": ev}, open(args.trace, "w"))


if __name__ == "__main__":
    main()
