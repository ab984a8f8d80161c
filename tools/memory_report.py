"""TiMePReSt (nF1B) vs PipeDream (1F1B) per-stage memory.

The paper's one quantitative memory claim: TiMePReSt uses
about 50% / 40% less GPU memory than PipeDream in stage 0 / stage 1 (VGG-16,
two GPUs), because it drops horizontal weight stashing.  The reference models
this with the slot model (proj/src/metrics.cpp:73-101): per stage,
peak retained weight versions x stage params + peak stashed samples x width.

For each config and mode this prints, per stage:
  * the slot model: peak retained versions (build_retention_timeline's
    peak_concurrent, ledger.cpp:224-264) and peak stashed samples
    (metrics.cpp:80-94), both from the product's plan layer;
  * the B200 session's own allocation (pb_plan_memory, host only): weight
    bytes (bf16 version pool + fp32 masters) and activation bytes;
  * with --measure (GPU): the cudaMemGetInfo drop when the session is created.

  python tools/memory_report.py [--measure] [--md profiles/memory_r2.md]
"""
from __future__ import annotations

import argparse
import json
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

from paper_2410_14312_b200 import pipesim as P  # noqa: E402

CONFIGS = {
    # name: widths, acts, W, N, B, M
    "C1 784-512-256-10 W=2": ([784, 512, 256, 10], ["relu", "relu", "linear"], 2, 4, 256, 32),
    "C3 16x4096 W=2": ([4096] * 17, ["relu"] * 15 + ["linear"], 2, 8, 1024, 32),
    "C3 16x4096 W=8": ([4096] * 17, ["relu"] * 15 + ["linear"], 8, 8, 1024, 32),
}
MODES = ("timeprest", "pipedream")


def slot_model(W, N, B, M, mode):
    """peak retained versions and peak stashed samples per stage
    (metrics.cpp:73-94, restated over the product's plan layer)."""
    cfg = P.SimConfig(workers=W, micro_batches=N, mini_batches=M, samples_per_mini_batch=B)
    grid = P.build_nf1b_schedule(cfg) if mode == "timeprest" else P.build_1f1b_schedule(cfg)
    ledger = P.assign_versions(grid, cfg)
    tl = P.build_retention_timeline(ledger, grid)
    nf1b = mode == "timeprest"
    units = N if nf1b else 1
    unit_samples = B // units
    stash = []
    for s in range(1, W + 1):
        iv = []
        for k in range(1, M + 1):
            b = grid.backward_slot(k, s)
            for j in range(1, units + 1):
                f = grid.forward_slot(k, j if nf1b else 0, s)
                iv.append((f, b))
        peak = 0
        for t in range(1, grid.horizon() + 1):
            peak = max(peak, sum(unit_samples for f, b in iv if f <= t <= b))
        stash.append(peak)
    return list(tl.peak_concurrent), stash


def stage_params(widths, W):
    net = P.NetworkSpec(widths, ["linear"] * (len(widths) - 1), "softmax_cross_entropy")
    return [st.param_count() for st in P.partition_model(net, W)]


def measure_bytes(widths, acts, W, N, B, M, mode):
    import torch
    net = P.NetworkSpec(widths, acts, "softmax_cross_entropy")
    torch.cuda.synchronize()
    free0, _ = torch.cuda.mem_get_info()
    s = P.Session(net, W, N, B, M, 0.05, mode=mode, use_graph=False)
    torch.cuda.synchronize()
    free1, _ = torch.cuda.mem_get_info()
    dev = s.device_bytes
    del s
    return free0 - free1, dev


def report(measure=False):
    rows = []
    for name, (widths, acts, W, N, B, M) in CONFIGS.items():
        net = P.NetworkSpec(widths, acts, "softmax_cross_entropy")
        sp = stage_params(widths, W)
        for mode in MODES:
            peak_v, stash = slot_model(W, N, B, M, mode)
            mem = P.plan_memory(net, W, N, B, M, mode=mode)
            r = {"config": name, "mode": mode, "W": W, "N": N, "B": B, "M": M,
                 "stage_params": sp, "slot_peak_versions": peak_v,
                 "slot_peak_stashed_samples": stash,
                 "pool_versions": mem["pool"].tolist(), "act_slots": mem["act_slots"].tolist(),
                 "weight_bytes": mem["weight_bytes"].tolist(),
                 "act_bytes": mem["act_bytes"].tolist()}
            if measure:
                r["measured_session_bytes"], r["arena_bytes"] = measure_bytes(
                    widths, acts, W, N, B, M, mode)
            rows.append(r)
    return rows


def to_markdown(rows):
    mb = 1 / 2**20
    out = ["# TiMePReSt vs PipeDream: per-stage memory (SURVEY §8(f)#3)", "",
           "Slot model = the reference's metrics.cpp:73-101 quantities (peak retained weight "
           "versions, peak stashed samples), computed by the product's plan layer. "
           "Session = the bytes the B200 session allocates for that stage "
           "(`pb_plan_memory`: weights = bf16 version pool + fp32 masters; activations = "
           "activation slots + scratch deltas + logits). "
           "Paper claim (PAPER.md:486, VGG-16 on 2 GPUs): TiMePReSt uses ~50% / ~40% less "
           "memory than PipeDream in stage 0 / stage 1.", ""]
    by = {}
    for r in rows:
        by.setdefault(r["config"], {})[r["mode"]] = r
    for name, d in by.items():
        t, p = d["timeprest"], d["pipedream"]
        out += [f"## {name} (N={t['N']}, B={t['B']}, M={t['M']})", "",
                "| stage | mode | slot: peak versions | slot: peak stashed samples | "
                "session: versions held | weights MiB | activations MiB | total MiB |",
                "|---|---|---|---|---|---|---|---|"]
        for s in range(t["W"]):
            for r in (t, p):
                tot = r["weight_bytes"][s] + r["act_bytes"][s]
                out.append(f"| {s} | {r['mode']} | {r['slot_peak_versions'][s]} | "
                           f"{r['slot_peak_stashed_samples'][s]} | {r['pool_versions'][s]} | "
                           f"{r['weight_bytes'][s] * mb:.1f} | {r['act_bytes'][s] * mb:.1f} | "
                           f"{tot * mb:.1f} |")
        out += ["", "| stage | TiMePReSt / PipeDream total | weights | activations | "
                "slot-model footprint (versions x params + samples x width) |",
                "|---|---|---|---|---|"]
        for s in range(t["W"]):
            tt = t["weight_bytes"][s] + t["act_bytes"][s]
            pt = p["weight_bytes"][s] + p["act_bytes"][s]
            width = 4096 if "4096" in name else 512
            fs = [r["slot_peak_versions"][s] * r["stage_params"][s] +
                  r["slot_peak_stashed_samples"][s] * width for r in (t, p)]
            out.append(f"| {s} | {tt / pt:.2f} ({100 * (1 - tt / pt):.0f}% less) | "
                       f"{t['weight_bytes'][s] / p['weight_bytes'][s]:.2f} | "
                       f"{t['act_bytes'][s] / max(1, p['act_bytes'][s]):.2f} | "
                       f"{fs[0] / fs[1]:.2f} |")
        if "measured_session_bytes" in t:
            out += ["", f"Measured on the GPU (cudaMemGetInfo drop at session creation, all "
                    f"stages on one device): TiMePReSt {t['measured_session_bytes'] * mb:.0f} MiB, "
                    f"PipeDream {p['measured_session_bytes'] * mb:.0f} MiB "
                    f"(arena {t['arena_bytes'] * mb:.0f} / {p['arena_bytes'] * mb:.0f} MiB)."]
        out.append("")
    return "\n".join(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--measure", action="store_true")
    ap.add_argument("--md", default="")
    ap.add_argument("--json", default="")
    a = ap.parse_args()
    rows = report(a.measure)
    md = to_markdown(rows)
    print(md)
    if a.md:
        pathlib.Path(a.md).write_text(md)
    if a.json:
        pathlib.Path(a.json).write_text(json.dumps(rows, indent=1))


if __name__ == "__main__":
    main()
