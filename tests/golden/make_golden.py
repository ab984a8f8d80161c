#!/usr/bin/env python3
"""Regenerates the committed golden fixtures from the REFERENCE ITSELF.

Run in the build container (needs /root/reference and oracle/_ref built by
`make -C oracle`):   python tests/golden/make_golden.py

Outputs (all small, committed):
  timeline-*.txt       ASCII timelines of the reference's own golden configs
                       (proj/tests/golden/timeline-*.txt), rendered by the
                       compiled reference (byte-identical to those files)
  plan_goldens.json    grids, ledgers, retention and v for a W x N x M sweep
  train_goldens.npz    per-mini losses / pins / consumed / final params of
                       small networks in all three modes (fp64 reference)
  c1_summary.json      784-512-256-10 (C1) reference losses and parameter
                       summaries (the full vectors are recomputed by the
                       numpy restatement on the GPU box)
"""
import json
import pathlib
import sys

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))
from oracle import pipesim_np as O  # noqa: E402
from oracle import ref  # noqa: E402

TIMELINES = ["4-2-7", "4-4-4", "3-2-6", "5-2-6", "5-3-6"]

PLAN_CASES = [(w, n, m, mode) for mode in (0, 1) for w in (2, 3, 4, 5, 8) for n in (2, 3, 4, 8)
              for m in (1, 3, 2 * (w + n))]

# (name, widths, acts, loss, W, N, B, M, lr, seed)
TRAIN_CASES = [
    ("demo", [2, 8, 2], [2, 0], 1, 2, 2, 10, 6, 0.05, 42),
    ("deep4", [2, 6, 6, 6, 2], [2, 2, 2, 0], 1, 4, 2, 4, 7, 0.05, 2),
    ("scalar", [1, 1, 1], [0, 0], 0, 2, 2, 2, 2, 0.2, 11),
    ("mixed", [30, 20, 16, 10], [1, 3, 0], 0, 3, 4, 12, 10, 0.1, 5),
    ("relu8", [64, 48, 48, 40, 40, 32, 32, 24, 16], [1] * 7 + [0], 1, 8, 8, 64, 6, 0.05, 3),
]


def main():
    if not ref.available():
        sys.exit("build oracle/_ref first: make -C oracle")
    for f in TIMELINES:
        w, n, m = map(int, f.split("-"))
        (HERE / f"timeline-{f}.txt").write_text(ref.render_ascii(w, n, m))

    plan = []
    for w, n, m, mode in PLAN_CASES:
        g = ref.schedule(w, n, m, mode)
        led = ref.ledger(w, n, m, mode)
        iv, peak = ref.retention(w, n, m, mode)
        try:
            v = ref.measure_v(w, n, m, mode, strict=False) if mode == 0 and m >= 2 else None
        except ref.RefError:
            v = None
        plan.append(dict(W=w, N=n, M=m, mode=mode, grid=g.tolist(),
                         **{k: np.asarray(a).tolist() for k, a in led.items()},
                         retention=iv.tolist(), peak=peak.tolist(), v_measured=v,
                         v_closed=ref.closed_form_v(w, n)))
    (HERE / "plan_goldens.json").write_text(json.dumps(plan, separators=(",", ":")))

    arrays = {}
    for name, widths, acts, loss, W, N, B, M, lr, seed in TRAIN_CASES:
        x, y = O.make_classification_task(M * B, widths[0], widths[-1], seed=7)
        p0 = ref.init_params(widths, acts, loss, seed)
        for mode in ("timeprest", "pipedream", "sequential"):
            r = ref.train(widths, acts, loss, W, N, B, M, lr, seed, mode, x, y, p0,
                          epochs=2, observe=(mode != "sequential"))
            key = f"{name}.{mode}"
            arrays[key + ".params"] = r["params"]
            arrays[key + ".losses"] = r["losses"]
            arrays[key + ".pinned"] = r["pinned"]
            arrays[key + ".consumed"] = r["consumed"]
            if r["held"] is not None:
                arrays[key + ".held"] = r["held"].astype(np.int8)
            arrays[key + ".log"] = np.frombuffer(r["log"].encode(), np.uint8)
    np.savez_compressed(HERE / "train_goldens.npz", **arrays)

    widths, acts = [784, 512, 256, 10], [1, 1, 0]
    W, N, B, M = 2, 4, 256, 12
    x, y = O.make_classification_task(M * B, 784, 10, seed=7)
    p0 = ref.init_params(widths, acts, 1, 1)
    summ = {}
    for mode, w in (("timeprest", 2), ("pipedream", 2), ("sequential", 2), ("sequential", 1)):
        r = ref.train(widths, acts, 1, w, N, B, M, 0.05, 1, mode, x, y, p0)
        d = r["params"] - p0
        summ[f"{mode}.W{w}"] = dict(losses=r["losses"][0].tolist(),
                                    pinned=r["pinned"][0].tolist(),
                                    consumed=r["consumed"][0].tolist(),
                                    delta_norm=float(np.linalg.norm(d)),
                                    delta_sum=float(d.sum()),
                                    params_norm=float(np.linalg.norm(r["params"])),
                                    log=r["log"])
    (HERE / "c1_summary.json").write_text(json.dumps(summ, indent=1))
    print("goldens written to", HERE)


if __name__ == "__main__":
    main()
