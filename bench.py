#!/usr/bin/env python3
"""Benchmark of the B200 TiMePReSt pipeline step.

Workload (BASELINE.json configs[2], the largest that fits one GPU):
  deep MLP 16 x Linear(4096->4096) (widths 17 x 4096; ReLU x15, linear;
  softmax-CE over 4096 classes), mini-batch B=1024, N=8 micro-batches,
  W=8 pipeline stages, M=32 mini-batches per step.  One "step" is one
  train_epoch: the full nF1B schedule over M mini-batches (fill, steady
  state, drain), i.e. M*B = 32768 samples.
At --gpus 1 all 8 stages run on the one GPU (per-stage streams).

Prints ONE JSON line (rank 0).  `value` = samples/s with the epoch's data
resident in HBM; `e2e` = the same metric through the C ABI
(pb_session_train_epoch) from pinned host buffers, H2D inside the timed
region, loss read back every step.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WIDTH, LAYERS = 4096, 16
CFG = dict(widths=[WIDTH] * (LAYERS + 1), acts=["relu"] * (LAYERS - 1) + ["linear"],
           loss="softmax_cross_entropy", W=8, N=8, B=1024, M=32, lr=0.05, seed=1)
METRIC = "training samples/sec at 1/2/4/8 B200 pipeline stages; GEMM % of tensor peak"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return dict(hbm=p["hbm_gbs"], bf16=p["bf16_tflops"],
                    bf16_sus=p.get("bf16_tflops_sustained", p["bf16_tflops"]),
                    src="measured")
    except Exception:
        return dict(hbm=6650.0, bf16=1590.0, bf16_sus=1400.0, src="fallback")


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device=0):
        self.device = device
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx = max(mx, float(r[1]))
                for n, v in zip(names, r[4:8]):
                    if v.lower() == "active":
                        reasons.add(n)
            except Exception:
                pass
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        load = [v for v in sm if v > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(load), "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def gemm_flops_per_sample(widths):
    """F = 2ΣP (fwd) + 2ΣP (wgrad) + 2Σ_{l>=1} P (dgrad)."""
    P = [widths[i] * widths[i + 1] for i in range(len(widths) - 1)]
    return 2 * sum(P) + 2 * sum(P) + 2 * sum(P[1:])


REF_SAMPLE = dict(W=8, N=2, B=2, M=1)  # the reference's minimum step for this network


def _ref_one_step(_=None):
    """One reference train_epoch on the bounded sample; returns seconds
    (runs in a worker process: the compiled reference is single-threaded)."""
    sys.path.insert(0, ROOT)
    from oracle import ref
    from oracle import pipesim_np as O
    widths, acts = CFG["widths"], [1] * (LAYERS - 1) + [0]
    S = REF_SAMPLE
    x, y = O.make_classification_task(S["M"] * S["B"], WIDTH, WIDTH, seed=7)
    if ref.available():
        p = ref.init_params(widths, acts, 1, 1)
        r = ref.train(widths, acts, 1, S["W"], S["N"], S["B"], S["M"], 0.05, 1, "timeprest",
                      x, y, p)
        return ("reference", r["seconds"])
    # oracle port (numpy) when the compiled reference is not on this box
    net = O.Net(widths, ["relu"] * (LAYERS - 1) + ["linear"], "softmax_cross_entropy")
    p = np.random.default_rng(1).uniform(-1, 1, O.param_count(widths)) / 64.0
    t = time.perf_counter()
    O.train_epoch(net, S["W"], S["N"], S["B"], S["M"], 0.05, x, y, p)
    return ("port", time.perf_counter() - t)


def start_cpu_reference(runs):
    """Starts `runs` independent reference steps, one per host core, in the
    background (they overlap the GPU measurement).  Returns a finisher."""
    import concurrent.futures as cf
    import multiprocessing as mp
    runs = max(1, min(runs, os.cpu_count() or 1))
    ex = cf.ProcessPoolExecutor(max_workers=runs, mp_context=mp.get_context("spawn"))
    futs = [ex.submit(_ref_one_step) for _ in range(runs)]

    def finish():
        res = [f.result() for f in futs]
        ex.shutdown()
        kind = res[0][0]
        secs = statistics.median(r[1] for r in res)
        S = REF_SAMPLE
        samples = S["M"] * S["B"]
        return dict(value=samples / secs, unit="samples/s", cores=1, kind=kind,
                    sample=(f"16x4096 MLP, W=8 nF1B, N={S['N']}, B={S['B']}, M={S['M']} "
                            f"({samples} samples) per run; median of {runs} independent "
                            f"single-threaded runs ({runs} host cores in parallel), "
                            f"{secs:.1f} s each"))
    return finish


def cpu_reference(steps, warmup):
    return start_cpu_reference(steps)()


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cb = cpu_reference(args.steps, args.warmup)
    secs = (REF_SAMPLE["M"] * REF_SAMPLE["B"]) / cb["value"]
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": "samples/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000.0 * secs, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "deep MLP 16x4096, W=8 nF1B (bounded CPU sample)",
                       "model": "mlp-16x4096", "parallelism": "cpu-1thread"},
            "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": "samples/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mini-batches", type=int, default=CFG["M"])
    ap.add_argument("--stages", type=int, default=CFG["W"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2410_14312_b200 import pipesim as P
    from paper_2410_14312_b200 import _native as Nn

    cpu_finish = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu_finish = start_cpu_reference(1)  # overlaps the GPU measurement

    W, Nm, B, M = args.stages, CFG["N"], CFG["B"], args.mini_batches
    net = P.NetworkSpec(CFG["widths"], CFG["acts"], CFG["loss"])
    # N GPUs: the W=8 stages are split into N contiguous ranges, one process
    # per GPU, activations / deltas cross GPUs point to point over NVLink.
    # PIPESIM_REPLICAS=1 instead runs N independent full pipelines.
    split = world > 1 and not os.environ.get("PIPESIM_REPLICAS")
    if split:
        ids = [P.nccl_unique_ids(world)] if rank == 0 else [None]
        dist.broadcast_object_list(ids, src=0)
        sess = P.Session(net, W, Nm, B, M, CFG["lr"], "timeprest", device=local,
                         use_graph=not args.no_graph, rank=rank, world=world, nccl_ids=ids[0])
    else:
        sess = P.Session(net, W, Nm, B, M, CFG["lr"], "timeprest", device=local,
                         use_graph=not args.no_graph)
    p0 = P.init_network_params(net, CFG["seed"])
    sess.load_params(p0)
    rows = M * B
    # pinned host inputs: x (f32) and class labels (int32), same generator as the oracle
    x_np, labels_np = P.make_classification_task(rows, WIDTH, WIDTH, seed=7, as_labels=True,
                                                 dtype=np.float32)
    x_h = torch.from_numpy(x_np).pin_memory()
    y_h = torch.from_numpy(labels_np).pin_memory()
    h2d = x_h.numel() * 4 + y_h.numel() * 4
    sess.upload(x_h.numpy(), y_h.numpy(), y_labels=True)

    L = Nn.lib()
    from paper_2410_14312_b200._session_abi import pb_epoch_out
    loss_buf = np.zeros(M)
    out = pb_epoch_out(loss_buf.ctypes.data_as(C.POINTER(C.c_double)), None, None, None, None,
                       None, 0.0)

    def resident_step():
        Nn.check(L.pb_session_run_epoch(sess._h, C.byref(out)))

    def e2e_step():
        Nn.check(L.pb_session_train_epoch(sess._h, x_h.data_ptr(), 1, y_h.data_ptr(), 2,
                                          C.byref(out)))

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        resident_step()
    barrier()
    with ClockSampler(local) as clocks:
        t0 = time.perf_counter()
        dev_ms = []
        for _ in range(args.steps):
            resident_step()
            dev_ms.append(out.device_ms)
        barrier()
        wall = time.perf_counter() - t0
    ms_step = float(np.mean(dev_ms))
    if world > 1:
        t = torch.tensor([ms_step], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step = float(t.item())
    jobs = 1 if split else world  # a split pipeline processes the step's rows once
    value = jobs * rows / (ms_step / 1000.0)

    # ---- e2e through the C ABI: H2D of the step's inputs + D2H of the losses
    for _ in range(2):
        e2e_step()
    barrier()
    e2e_ms = []
    for _ in range(args.steps):
        t = time.perf_counter()
        e2e_step()
        e2e_ms.append(1000.0 * (time.perf_counter() - t))
    barrier()
    e2e_step_ms = float(np.mean(e2e_ms))
    if world > 1:
        t = torch.tensor([e2e_step_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_step_ms = float(t.item())
    e2e_value = jobs * rows / (e2e_step_ms / 1000.0)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    peaks = _peaks()
    fps = gemm_flops_per_sample(CFG["widths"])
    step_tflops = fps * rows / (ms_step / 1000.0) / 1e12

    roof = kernel_roofline(peaks)
    roof["step_gemm_tflops"] = step_tflops
    roof["step_frac_of_sustained"] = step_tflops / peaks["bf16_sus"]

    cb = None
    if cpu_finish is not None:
        try:
            cb = cpu_finish()
        except Exception as e:  # noqa: BLE001
            cb = {"value": None, "error": str(e)}

    line = {
        "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "weak" if (world > 1 and not split) else "strong",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": "deep MLP 16x4096 (BASELINE configs[2]) nF1B pipeline step",
                   "model": "mlp-16x4096-relu-ce4096", "global_batch": B, "seq_len": None,
                   "micro_batches": Nm, "stages": W, "mini_batches_per_step": M,
                   "samples_per_step": rows,
                   "parallelism": f"pp{W}-on-{world}gpu" + ("-replicas" if world > 1 and not split else ""),
                   "l2": "working set (bf16 weights 537 MB + fp32 masters 1.07 GB) > L2, no flush",
                   "precision": "bf16 operands, fp32 accumulate, fp32 master weights"},
        "roofline": roof,
        "cpu_baseline": cb,
        "e2e": {"value": e2e_value, "unit": "samples/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": M * 4 * B + M * 8, "ms_per_step": e2e_step_ms},
        "gpu_launches": sess.kernels_per_epoch,
        "clocks": clocks.summary(),
        "wall_s": wall,
    }
    print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


def kernel_roofline(peaks):
    """Dominant kernel: the tcgen05 GEMM at the workload's dgrad shape
    (M=1024 rows, N=K=4096; 34.4 GFLOP per launch), timed alone with CUDA
    events on its launch stream over 50 launches.  The three GEMM shapes of
    the step are all reported."""
    import torch
    from paper_2410_14312_b200 import kernels as K
    torch.manual_seed(0)
    res = {}
    shapes = {"fwd_128x4096x4096": (128, 4096, 4096, "fwd"),
              "dgrad_1024x4096x4096": (1024, 4096, 4096, "dgrad"),
              "wgrad_4096x4096x1024": (4096, 4096, 1024, "wgrad")}
    for name, (m, n, k, kind) in shapes.items():
        if kind == "fwd":
            x = K.padded_bf16(m, k); x.normal_()
            w = K.padded_bf16(n, k); w.normal_()
            b = torch.zeros(n, device="cuda")
            y = K.padded_bf16(m, n)
            fn = lambda: K.linear_fwd(x, w, b, "relu", y16=y)  # noqa: E731
        elif kind == "dgrad":
            dz = K.padded_bf16(m, k); dz.normal_()
            w = K.padded_bf16(k, n); w.normal_()
            xin = K.padded_bf16(m, n); xin.normal_()
            d = K.padded_bf16(m, n)
            fn = lambda: K.linear_bwd_dx(dz, w, xin, "relu", d)  # noqa: E731
        else:
            dz = K.padded_bf16(k, m); dz.normal_()
            xx = K.padded_bf16(k, n); xx.normal_()
            w32 = torch.zeros(m, n, device="cuda")
            w16 = K.padded_bf16(m, n)
            fn = lambda: K.linear_bwd_dw_sgd(dz, xx, w32, w32, w16, 0.0)  # noqa: E731
        for _ in range(5):
            fn()
        st = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(st)
        reps = 50
        for _ in range(reps):
            fn()
        e1.record(st)
        e1.synchronize()
        us = e0.elapsed_time(e1) * 1000.0 / reps
        flops = 2.0 * m * n * k
        res[name] = {"us": us, "tflops": flops / us / 1e6}
    dom = res["dgrad_1024x4096x4096"]
    traffic = None
    try:  # DRAM bytes per launch of the same kernel from the committed ncu capture
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            traffic = json.load(f)["dgrad_1024x4096x4096"]["bytes"]
    except Exception:
        pass
    return {"bound": "tensor", "kernel": "gemm_bf16_tcgen05_pair (dgrad shape)",
            "achieved": dom["tflops"], "peak": peaks["bf16"], "unit": "TFLOP/s",
            "frac": dom["tflops"] / peaks["bf16"], "peak_source": peaks["src"] + " burst bf16",
            "traffic": traffic, "traffic_unit": "bytes/launch (dram read+write, ncu)",
            "flops_per_launch": 2.0 * 1024 * 4096 * 4096, "per_shape": res}


if __name__ == "__main__":
    sys.exit(main())
