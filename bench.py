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
(pb_session_train_epoch) from pinned host buffers (x in bf16, class labels
int32): the H2D copies run inside the timed epoch, streamed per mini-batch
beside the compute, and the losses are read back every step.

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
        self.rows = []  # (host time, fields)
        self.proc = None
        self.window = None  # (t0, t1) host times of the timed region

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.perf_counter(), [x.strip() for x in line.split(",")]))

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
        rows = self.rows
        if self.window:  # samples taken during the timed region (sampling starts before)
            t0, t1 = self.window
            inside = [r for t, r in rows if t0 <= t <= t1 + 0.1]
            rows = inside or [r for _, r in rows[-2:]]
        else:
            rows = [r for _, r in rows]
        for r in rows:
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


def ref_parallel_runs():
    """How many single-threaded reference runs the host can hold at once:
    every core, capped by memory (one run of the 16x4096 f64 network holds
    ~15 GB max RSS: parameters, versions, gradients)."""
    cores = os.cpu_count() or 1
    try:
        import psutil
        mem = max(1, int(psutil.virtual_memory().available // (16 << 30)))
    except Exception:  # noqa: BLE001
        mem = 4
    return max(1, min(cores, mem))


def start_cpu_reference(runs):
    """Starts `runs` independent single-threaded reference steps, one per host
    core, in the background (they may overlap the GPU measurement).  The
    finisher reports the aggregate samples/s of the concurrent runs (the
    reference is single-threaded, so independent replicas are how it uses
    several cores) and `cores` = runs."""
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
        return dict(value=runs * samples / secs, unit="samples/s", cores=runs, kind=kind,
                    sec_per_run=secs,
                    sample=(f"16x4096 MLP, W=8 nF1B, N={S['N']}, B={S['B']}, M={S['M']} "
                            f"({samples} samples) per run; {runs} concurrent independent "
                            f"single-threaded runs on {runs} host cores (median "
                            f"{secs:.1f} s each), value = aggregate samples/s"))
    return finish


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    runs = ref_parallel_runs()
    cb = start_cpu_reference(runs)()
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": "samples/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000.0 * cb.pop("sec_per_run"), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "deep MLP 16x4096, W=8 nF1B (bounded CPU sample)",
                       "model": "mlp-16x4096", "parallelism": f"cpu-{runs}x1thread"},
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

    # the executor runs an 8-stage pipeline on one GPU without split-K
    # forwards (throughput over latency, session.cu); the standalone per-shape
    # timings below use the same kernels
    os.environ.setdefault("PIPESIM_SPLITK", "0")
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # PIPESIM_ONE_GPU=1: every rank on cuda:0 (exercises the multi-process
    # stage split on a one-GPU box; not a multi-GPU throughput number)
    one_gpu = os.environ.get("PIPESIM_ONE_GPU") == "1"
    if one_gpu:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if one_gpu:
            dist.init_process_group("gloo")
        else:
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
    # transport between the GPUs: CUDA IPC peer memory (default; the path the
    # multi-process GPU tests run) or NCCL send/recv (PIPESIM_TRANSPORT=nccl)
    transport = os.environ.get("PIPESIM_TRANSPORT", "ipc")
    if split and transport == "nccl":
        ids = [P.nccl_unique_ids(world)] if rank == 0 else [None]
        dist.broadcast_object_list(ids, src=0)
        sess = P.Session(net, W, Nm, B, M, CFG["lr"], "timeprest", device=local,
                         use_graph=not args.no_graph, rank=rank, world=world, nccl_ids=ids[0])
    elif split:
        sess = P.Session(net, W, Nm, B, M, CFG["lr"], "timeprest", device=local,
                         rank=rank, world=world, transport="ipc")
        blobs = [None] * world
        dist.all_gather_object(blobs, sess.ipc_export())
        sess.ipc_connect(blobs)
    else:
        # uninstrumented: the per-launch kernel timing runs in separate
        # sessions afterwards (in_step_kernels), so its event nodes do not
        # perturb the timed step
        sess = P.Session(net, W, Nm, B, M, CFG["lr"], "timeprest", device=local,
                         use_graph=not args.no_graph)
    p0 = P.init_network_params(net, CFG["seed"])
    sess.load_params(p0)
    kernels_per_step = sess.kernels_per_epoch
    rows = M * B
    # pinned host inputs: x (f32) and class labels (int32), same generator as the oracle
    x_np, labels_np = P.make_classification_task(rows, WIDTH, WIDTH, seed=7, as_labels=True,
                                                 dtype=np.float32)
    # e2e input: x rounded to bf16 on the host once (the bf16 path's operand
    # type: identical numerics, no device conversion, half the H2D bytes) and
    # int32 class labels, both page-locked
    x_h = torch.from_numpy(x_np).to(torch.bfloat16).pin_memory()
    y_h = torch.from_numpy(labels_np).pin_memory()
    h2d = x_h.numel() * 2 + y_h.numel() * 4
    sess.upload(x_np, labels_np, y_labels=True)

    L = Nn.lib()
    from paper_2410_14312_b200._session_abi import pb_epoch_out
    loss_buf = np.zeros(M)
    out = pb_epoch_out(loss_buf.ctypes.data_as(C.POINTER(C.c_double)), None, None, None, None,
                       None, 0.0)

    def resident_step():
        Nn.check(L.pb_session_run_epoch(sess._h, C.byref(out)))

    def e2e_step():
        Nn.check(L.pb_session_train_epoch(sess._h, x_h.data_ptr(), 3, y_h.data_ptr(), 2,
                                          C.byref(out)))

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    with ClockSampler(local) as clocks:  # sampling starts before the warm-up
        for _ in range(args.warmup):
            resident_step()
        barrier()
        t0 = time.perf_counter()
        dev_ms = []
        for _ in range(args.steps):
            resident_step()
            dev_ms.append(out.device_ms)
        barrier()
        wall = time.perf_counter() - t0
        clocks.window = (t0, t0 + wall)
    ms_step = float(np.mean(dev_ms))
    if world > 1:
        t = torch.tensor([ms_step], device="cpu" if one_gpu else "cuda")
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
        t = torch.tensor([e2e_step_ms], device="cpu" if one_gpu else "cuda")
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

    roof = kernel_roofline(peaks, in_step_kernels(P, net, W, Nm, B, M, local, sess)
                           if not split else {})
    roof["step_gemm_tflops"] = step_tflops
    roof["step_frac_of_sustained"] = step_tflops / peaks["bf16_sus"]
    if split:
        roof["note"] = ("in-step per-launch timing runs only in the single-process (N=1) "
                        "configuration; with the stages split over processes the line gives "
                        "the alone table and the step-level GEMM rate")

    cb = None
    if cpu_finish is not None:
        try:
            cb = cpu_finish()
            cb.pop("sec_per_run", None)
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
                   "parallelism": f"pp{W}-on-{world}gpu" + ("-replicas" if world > 1 and not split else
                                                            (f"-{transport}" if split else "")),
                   "l2": "working set (bf16 weights 537 MB + fp32 masters 1.07 GB) > L2, no flush",
                   "precision": "bf16 operands, fp32 accumulate, fp32 master weights"},
        "roofline": roof,
        "cpu_baseline": cb,
        "e2e": {"value": e2e_value, "unit": "samples/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": M * 4 * B + M * 8, "ms_per_step": e2e_step_ms},
        "gpu_launches": kernels_per_step,
        "other_configs": other_configs(P) if world == 1 else None,
        "clocks": clocks.summary(),
        "wall_s": wall,
    }
    print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


DOMINANT = "fwd"  # largest share of the step (ncu launch list, profiles/)


def other_configs(P):
    """BASELINE configs[0]/[1] on this GPU (784-512-256-10, N=4, B=256,
    M=12): W=2 nF1B and W=1 sequential, device-timed epochs with resident
    data.  Launch-bound (0.6 GFLOP per mini-batch); reported beside the
    headline, not as it."""
    out = {}
    widths, acts = [784, 512, 256, 10], ["relu", "relu", "linear"]
    net = P.NetworkSpec(widths, acts, "softmax_cross_entropy")
    for key, W, mode in (("C1_mnist_mlp_W2_nf1b", 2, "timeprest"),
                         ("C2_mnist_mlp_W1_sequential", 1, "sequential")):
        B, M = 256, 12
        s = P.Session(net, W, 4, B, M, CFG["lr"], mode)
        s.load_params(P.init_network_params(net, CFG["seed"]))
        x, lab = P.make_classification_task(M * B, 784, 10, seed=7, as_labels=True,
                                            dtype=np.float32)
        s.upload(x, lab, y_labels=True)
        for _ in range(3):
            s.run_epoch()
        ms = float(np.median([s.run_epoch()["device_ms"] for _ in range(5)]))
        s.close()
        out[key] = {"samples_per_s": M * B / (ms / 1000.0), "us_per_mini_batch": 1000.0 * ms / M}
    return out


def in_step_kernels(P, net, W, Nm, B, M, device, main_sess):
    """In-step launch statistics of the three GEMM kinds: one instrumented
    session each (CUDA events around every launch of that kind, recorded
    inside the graph on the launch stream), same workload as the timed step,
    two epochs, the second kept."""
    out = {}
    main_sess.close()  # free HBM for the instrumented sessions
    for kind in (DOMINANT, "dgrad", "wgrad"):
        s = P.Session(net, W, Nm, B, M, CFG["lr"], "timeprest", device=device,
                      timed_kernel=kind)
        s.load_params(P.init_network_params(net, CFG["seed"]))
        x, lab = P.make_classification_task(M * B, WIDTH, WIDTH, seed=7, as_labels=True,
                                            dtype=np.float32)
        s.upload(x, lab, y_labels=True)
        s.run_epoch()
        s.run_epoch()
        ms, fl = s.kernel_timeline()
        out[kind] = (ms, fl)
        s.close()
    return out


def _stats(ms, fl, hbm_bytes=None):
    d = {"launches_per_step": int(len(ms)), "mean_us": float(1000.0 * ms.mean()),
         "tflops": float(fl.sum() / (ms.sum() / 1000.0) / 1e12)}
    if hbm_bytes is not None:
        d["hbm_gbs"] = float(hbm_bytes * len(ms) / (ms.sum() / 1000.0) / 1e9)
    return d


# HBM bytes of one wgrad+SGD launch (4096 x 4096 layer, one mini-batch):
# split masters read hi + lo and write hi + lo (8 B / parameter) + dZ and X
SGD_BYTES = WIDTH * WIDTH * 8 + 2 * 1024 * WIDTH * 2


def kernel_roofline(peaks, runs):
    """Roofline of the dominant kernel, the forward GEMM (bias+ReLU fused):
    algorithmic flops of every forward launch of the timed step (2*rows*N*K)
    / its device duration, from CUDA events around each launch inside the
    graph on its stage stream (kernels overlap other stages' kernels, so this
    is the in-step rate), against the sustained bf16 peak.  Also: the same
    in-step statistics for dgrad and wgrad+SGD (the SGD epilogue moves
    10 B/param + operands: HBM GB/s reported), and each GEMM shape timed alone
    (graph-captured, weights rotated through 6 copies > L2 so they stream
    from HBM as in the pipeline)."""
    import torch
    from paper_2410_14312_b200 import kernels as K
    torch.manual_seed(0)
    n = WIDTH
    alone = {}
    ws = [K.padded_bf16(n, n).normal_() for _ in range(6)]
    for m in (128, 256, 1024):
        x = K.padded_bf16(m, n).normal_()
        b = torch.zeros(n, device="cuda")
        y = K.padded_bf16(m, n)
        us = K.graph_time_us([lambda w=w: K.linear_fwd(x, w, b, "relu", y16=y) for w in ws])
        alone[f"fwd_{m}x{n}x{n}"] = {"us": us, "tflops": 2.0 * m * n * n / us / 1e6}
    dz = K.padded_bf16(1024, n).normal_()
    xin = K.padded_bf16(1024, n).normal_()
    d = K.padded_bf16(1024, n)
    us = K.graph_time_us([lambda w=w: K.linear_bwd_dx(dz, w, xin, "relu", d) for w in ws])
    alone[f"dgrad_1024x{n}x{n}"] = {"us": us, "tflops": 2.0 * 1024 * n * n / us / 1e6}
    del ws
    xx = K.padded_bf16(1024, n).normal_()
    # the session's split fp32 masters: read hi/lo of the current version,
    # write hi/lo of the new one (8 B per parameter), two alternating sets
    his = [K.padded_bf16(n, n) for _ in range(2)]
    los = [torch.zeros(n, n, dtype=torch.int16, device="cuda") for _ in range(2)]
    us = K.graph_time_us([lambda i=i: K.linear_bwd_dw_sgd_split(dz, xx, his[i], los[i], his[i],
                                                                 los[i], 0.0)
                          for i in range(2)])
    alone[f"wgrad_sgd_{n}x{n}x1024"] = {"us": us, "tflops": 2.0 * 1024 * n * n / us / 1e6,
                                        "hbm_gbs": SGD_BYTES / us / 1e3}
    traffic = None
    try:  # DRAM bytes per launch of the same kernel from the committed ncu capture
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            traffic = json.load(f)["fwd_1024x4096x4096"]["bytes"]
    except Exception:
        pass
    in_step = {}
    for kind, (ms, fl) in runs.items():
        in_step[kind] = _stats(ms, fl, SGD_BYTES if kind == "wgrad" else None)
    achieved = in_step.get("fwd", {}).get("tflops")
    return {"bound": "tensor", "kernel": "forward GEMM gemm_bf16_tcgen05_pair/_tcgen05 "
            "(bias+ReLU epilogue), in-step", "achieved": achieved, "peak": peaks["bf16_sus"],
            "unit": "TFLOP/s", "frac": achieved / peaks["bf16_sus"] if achieved else None,
            "peak_source": peaks["src"] + " sustained bf16 (kernel timed inside the step)",
            "traffic": traffic, "traffic_unit": "bytes/launch at 1024x4096x4096 (dram read+write, ncu; algorithmic 50.3 MB)",
            "flops_per_launch": "2*rows*4096*4096 (rows = coalesced micro-batches, 128..1024)",
            "in_step": in_step, "alone": alone}


if __name__ == "__main__":
    sys.exit(main())
