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


# Bounded samples of the benchmark workload for the CPU reference (the same
# 16x4096 network and W=8, N=8 nF1B schedule, one mini-batch).  Every
# reference mini-batch pays fixed costs independent of B: params_digest over
# all 268M parameters (trainer.cpp:492-501, ~45 s on one core) and the 2 GB
# version copy, so B is chosen large enough to amortise them; the digest
# share is measured and reported beside the value.
REF_SAMPLE = dict(W=8, N=8, B=64, M=1)   # reference arm (--impl reference): ~8 min per run
CPU_SAMPLE = dict(W=8, N=8, B=8, M=1)    # cpu_baseline of our line: ~100 s on one core


def _ref_one_step(S=None):
    """One reference train_epoch on a bounded sample; returns (kind, seconds)
    (runs in a worker process: the compiled reference is single-threaded)."""
    sys.path.insert(0, ROOT)
    from oracle import ref
    from oracle import pipesim_np as O
    S = S or REF_SAMPLE
    widths, acts = CFG["widths"], [1] * (LAYERS - 1) + [0]
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


def _ref_digest_seconds():
    """Seconds of the reference's params_digest over the whole 16x4096
    network, timed on 1/16 of the parameters and scaled (the digest is
    linear in the parameter count)."""
    sys.path.insert(0, ROOT)
    from oracle import ref
    if not ref.available():
        return None
    from oracle import pipesim_np as O
    n = O.param_count(CFG["widths"])
    v = np.random.default_rng(1).uniform(-1, 1, n // 16) / 64.0
    secs, _ = ref.digest_seconds(v)
    return secs * n / len(v)


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


def start_cpu_reference(runs, S=None):
    """Starts `runs` independent single-threaded reference steps, one per host
    core, in the background (they may overlap the GPU measurement), plus one
    digest timing.  The finisher reports the aggregate samples/s of the
    concurrent runs (the reference is single-threaded, so independent
    replicas are how it uses several cores) and `cores` = runs."""
    import concurrent.futures as cf
    import multiprocessing as mp
    S = S or REF_SAMPLE
    runs = max(1, min(runs, os.cpu_count() or 1))
    ex = cf.ProcessPoolExecutor(max_workers=runs, mp_context=mp.get_context("spawn"))
    futs = [ex.submit(_ref_one_step, S) for _ in range(runs)]

    def finish():
        res = [f.result() for f in futs]
        try:
            dig = _ref_digest_seconds()
        except Exception:  # noqa: BLE001
            dig = None
        ex.shutdown()
        kind = res[0][0]
        secs = statistics.median(r[1] for r in res)
        samples = S["M"] * S["B"]
        out = dict(value=runs * samples / secs, unit="samples/s", cores=runs, kind=kind,
                   sec_per_run=secs,
                   sample=(f"16x4096 MLP, W={S['W']} nF1B, N={S['N']}, B={S['B']}, M={S['M']} "
                           f"({samples} samples) per run; {runs} concurrent independent "
                           f"single-threaded runs on {runs} host cores (median "
                           f"{secs:.1f} s each), value = aggregate samples/s"))
        if dig is not None:
            # per mini-batch: params_digest of all stages (trainer.cpp:492-501)
            out["digest_s_per_mini_batch"] = dig
            out["digest_share"] = min(1.0, S["M"] * dig / secs)
            out["samples_per_s_excl_digest"] = runs * samples / max(1e-9, secs - S["M"] * dig)
        return out
    return finish


def run_reference_arm(args):
    """The reference's own CPU implementation (oracle/_ref: the unmodified
    reference sources, or the numpy port where they were not built) on the
    host's cores.  Each process runs exactly one bounded step (REF_SAMPLE);
    `steps` / `warmup` report what actually ran."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    runs = ref_parallel_runs()
    cb = start_cpu_reference(runs)()
    S = REF_SAMPLE
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": "samples/s",
            "n_gpus": args.gpus, "steps": 1, "warmup": 0,
            "steps_requested": args.steps, "warmup_requested": args.warmup,
            "ms_per_step": 1000.0 * cb.pop("sec_per_run"), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "deep MLP 16x4096 (BASELINE configs[2]), W=8 N=8 nF1B, "
                                   f"bounded CPU sample: B={S['B']}, M={S['M']} per run",
                       "model": "mlp-16x4096-relu-ce4096", "global_batch": S["B"],
                       "micro_batches": S["N"], "stages": S["W"],
                       "mini_batches_per_step": S["M"],
                       "parallelism": f"cpu-{runs}x1thread"},
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
    ap.add_argument("--no-dropin", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)

    # split-K forwards follow the session's own policy (on only when a process
    # holds <= 2 stages, i.e. one stage per GPU: latency over throughput); the
    # standalone per-shape timings below must use the step's configuration,
    # so a process holding more stages turns split-K off for them as well
    world_env = int(os.environ.get("WORLD_SIZE", "1"))
    if args.stages / max(1, world_env) > 2 and not os.environ.get("PIPESIM_REPLICAS"):
        os.environ.setdefault("PIPESIM_SPLITK", "0")
    elif os.environ.get("PIPESIM_REPLICAS"):
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
        cpu_finish = start_cpu_reference(1, CPU_SAMPLE)  # overlaps the GPU measurement

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
    # e2e input: f32 rows and int32 class labels in page-locked host memory;
    # the epoch copies them (per mini-batch, on a copy stream) and converts x
    # to the bf16 operand on the device inside the timed region
    x_h = torch.from_numpy(x_np).pin_memory()
    y_h = torch.from_numpy(labels_np).pin_memory()
    h2d = x_h.numel() * 4 + y_h.numel() * 4
    sess.upload(x_np, labels_np, y_labels=True)

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

    # ---- N > 1: pipeline-boundary traffic (the program's own transfer list)
    # and per-stage busy time / bubble from one node-timed epoch
    pipeline = None
    if split:
        xfers = P.plan_transfers(net, W, Nm, B, M, "timeprest", rank=rank, world=world)
        sent = {}
        for kind, d, peer, nbytes in xfers:
            if kind == "send":
                key = f"{min(rank, peer)}-{max(rank, peer)}:{'act' if d == 0 else 'delta'}"
                sent[key] = sent.get(key, 0) + nbytes
        prof = sess.profile_epoch()["profile"]
        mine = {"rank": rank, "sent": sent, "makespan_ms": prof["makespan_ms"],
                "busy_ms": [b for b in prof["busy_ms"] if b >= 0]}
        allp = [None] * world
        dist.all_gather_object(allp, mine)
        if rank == 0:
            bytes_per_boundary = {}
            for m in allp:
                for k, v in m["sent"].items():
                    bytes_per_boundary[k] = bytes_per_boundary.get(k, 0) + v
            busy = [b for m in allp for b in m["busy_ms"]]
            mk = max(m["makespan_ms"] for m in allp)
            pipeline = {
                "boundary_bytes_per_step": bytes_per_boundary,
                "boundary_GBps_at_step_rate": {k: v / (ms_step / 1000.0) / 1e9
                                               for k, v in bytes_per_boundary.items()},
                "transport": transport + ("" if transport == "ipc" else " (unverified on hardware)"),
                "stage_busy_ms": busy, "profile_makespan_ms": mk,
                "bubble": 1.0 - sum(busy) / (len(busy) * mk) if mk > 0 else None,
                "note": ("busy / bubble from one epoch timed per node without the graph "
                         "(Session.profile_epoch); bytes from the program's transfer list"),
            }

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    peaks = _peaks()
    fps = gemm_flops_per_sample(CFG["widths"])
    step_tflops = fps * rows / (ms_step / 1000.0) / 1e12

    roof = kernel_roofline(peaks, in_step_kernels(P, net, W, Nm, B, M, local, sess)
                           if not split else {}, ms_step)
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
        "pipeline": pipeline,
        "other_configs": other_configs(P) if world == 1 else None,
        "e2e_dropin": dropin_e2e() if world == 1 and not args.no_dropin else None,
        "clocks": clocks.summary(),
        "wall_s": wall,
    }
    print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


DOMINANT = "fwd"  # instrumented first (largest share of the step in the ncu launch list)


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
    if os.environ.get("PIPESIM_BENCH_VGG", "1") != "0":
        out.update(vgg_config(P))
    return out


def vgg_config(P):
    """BASELINE configs[3]: VGG-16 on 224x224x3 synthetic images (1000
    classes), 8 nF1B stages on this GPU (flop-balanced), B=64, N=4, M=16,
    bf16 conv stages (implicit-GEMM tcgen05), data resident; images/s and
    the conv + FC GEMM rate against the sustained bf16 peak."""
    from paper_2410_14312_b200 import convnet as CN
    net = CN.vgg16()
    W, N, B, M = 8, 4, 64, 16
    s = P.Session(net, W, N, B, M, 1e-4, "timeprest")
    s.load_params(CN.init_params(net, CFG["seed"]))
    x, lab = CN.synthetic_images(M * B, net, seed=7)
    s.upload(x, lab, y_labels=True)
    for _ in range(2):
        s.run_epoch()
    ms = float(np.median([s.run_epoch()["device_ms"] for _ in range(3)]))
    s.close()
    rate = M * B / (ms / 1000.0)
    tflops = net.flops_per_sample() * rate / 1e12
    return {"C4_vgg16_224_W8_nf1b": {"images_per_s": rate, "ms_per_epoch": ms, "images_per_epoch": M * B,
                                      "partition": net.partition(W), "gemm_tflops": tflops,
                                      "frac_of_sustained": tflops / _peaks()["bf16_sus"]}}


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
FWD_BYTES = lambda m: m * WIDTH * 2 + WIDTH * WIDTH * 2 + m * WIDTH * 2  # noqa: E731


def alone_us(kind, m):
    """Device time of ONE launch of a GEMM kind at m rows, timed alone
    (graph-captured, weights rotated through 6 copies > L2 so they stream
    from HBM as in the pipeline)."""
    import torch
    from paper_2410_14312_b200 import kernels as K
    torch.manual_seed(0)
    n = WIDTH
    if kind == "fwd":
        ws = [K.padded_bf16(n, n).normal_() for _ in range(6)]
        x = K.padded_bf16(m, n).normal_()
        b = torch.zeros(n, device="cuda")
        y = K.padded_bf16(m, n)
        return K.graph_time_us([lambda w=w: K.linear_fwd(x, w, b, "relu", y16=y) for w in ws])
    if kind == "dgrad":
        ws = [K.padded_bf16(n, n).normal_() for _ in range(6)]
        dz = K.padded_bf16(m, n).normal_()
        xin = K.padded_bf16(m, n).normal_()
        d = K.padded_bf16(m, n)
        return K.graph_time_us([lambda w=w: K.linear_bwd_dx(dz, w, xin, "relu", d) for w in ws])
    # wgrad + SGD with the session's split fp32 masters: read hi/lo of the
    # current version, write hi/lo of the new one, two alternating sets
    dz = K.padded_bf16(m, n).normal_()
    xx = K.padded_bf16(m, n).normal_()
    his = [K.padded_bf16(n, n) for _ in range(2)]
    los = [torch.zeros(n, n, dtype=torch.int16, device="cuda") for _ in range(2)]
    return K.graph_time_us([lambda i=i: K.linear_bwd_dw_sgd_split(dz, xx, his[i], los[i], his[i],
                                                                   los[i], 0.0)
                            for i in range(2)])


def kernel_roofline(peaks, runs, ms_step):
    """Roofline of the step's dominant kernel.

    Every GEMM launch of one timed step is known with its shape (the
    instrumented sessions of in_step_kernels record each launch's algorithmic
    flops 2*rows*N*K).  Each distinct shape is timed ALONE; a kind's time per
    step is the sum over its launches of the alone time of their shape.  The
    dominant kernel is the kind with the largest such time; `achieved` = its
    algorithmic flops per step / that time (= flops per launch / mean launch
    duration), against the BURST bf16 peak (each launch timed alone).
    `share_of_step` = that alone time / ms_per_step (the cross-check: it must
    be <= 1).  The in-step per-launch durations are reported too, but they
    are concurrency-inflated (2-3 GEMMs of different stages share the SMs),
    so they are not a kernel rate."""
    import collections
    kinds = {}
    for kind, (ms, fl) in runs.items():
        rows = np.rint(fl / (2.0 * WIDTH * WIDTH)).astype(int)
        hist = collections.Counter(rows.tolist())
        shapes = {}
        t_ms = 0.0
        for m, cnt in sorted(hist.items()):
            us = alone_us(kind, m)
            shapes[f"{m}x{WIDTH}x{WIDTH}"] = {"launches": cnt, "us": us,
                                              "tflops": 2.0 * m * WIDTH * WIDTH / us / 1e6}
            if kind == "wgrad":
                shapes[f"{m}x{WIDTH}x{WIDTH}"]["hbm_gbs"] = SGD_BYTES / us / 1e3
            t_ms += cnt * us / 1000.0
        kinds[kind] = {"launches_per_step": int(len(ms)), "flops_per_step": float(fl.sum()),
                       "alone_ms_per_step": t_ms,
                       "tflops": float(fl.sum() / (t_ms / 1000.0) / 1e12) if t_ms else None,
                       "share_of_step": t_ms / ms_step, "shapes": shapes,
                       "in_step_concurrency_inflated": _stats(
                           ms, fl, SGD_BYTES if kind == "wgrad" else None)}
    traffic = None
    try:  # DRAM bytes per launch of the same kernel from the committed ncu capture
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            traffic = json.load(f)
    except Exception:
        pass
    if not kinds:
        return {"bound": "tensor", "achieved": None, "peak": peaks["bf16"], "unit": "TFLOP/s",
                "frac": None, "traffic": None}
    dom = max(kinds, key=lambda k: kinds[k]["alone_ms_per_step"])
    d = kinds[dom]
    names = {"fwd": "forward GEMM (bias+ReLU epilogue)", "dgrad": "dgrad GEMM (act' gate)",
             "wgrad": "wgrad GEMM + fused SGD epilogue (split fp32 masters)"}
    tr = None
    if traffic:
        key = {"fwd": "fwd_1024x4096x4096", "dgrad": "dgrad_1024x4096x4096",
               "wgrad": "wgrad_sgd_4096x4096x1024"}[dom]
        tr = traffic.get(key, {}).get("bytes")
    return {"bound": "tensor", "kernel": names[dom], "dominant": dom,
            "achieved": d["tflops"], "peak": peaks["bf16"], "unit": "TFLOP/s",
            "frac": d["tflops"] / peaks["bf16"] if d["tflops"] else None,
            "peak_source": peaks["src"] + " burst bf16 (each launch timed alone)",
            "traffic": tr,
            "traffic_unit": "dram read+write bytes per launch at the 1024-row shape (ncu)",
            "flops_per_launch": "2*rows*4096*4096 (rows per launch in `kinds[..].shapes`)",
            "share_of_step": d["share_of_step"], "kinds": kinds}


def dropin_e2e(configs=("c1", "c3")):
    """The reference-facing C++ pipesim::train_epoch timed end to end by
    tools/bin/dropin_bench (fp64 stages and dataset in host memory, digests,
    version_store refill), with its per-phase breakdown."""
    exe = os.path.join(ROOT, "tools", "bin", "dropin_bench")
    out = {}
    if not os.path.exists(exe):
        return {"error": "tools/bin/dropin_bench not built"}
    for c in configs:
        try:
            r = subprocess.run([exe, c, "3"], capture_output=True, text=True, timeout=600)
            out[c] = json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else \
                {"error": r.stderr[-500:]}
        except Exception as e:  # noqa: BLE001
            out[c] = {"error": str(e)}
    return out


if __name__ == "__main__":
    sys.exit(main())
