"""GEMM yardstick: our tcgen05 kernels vs cuBLAS (torch.mm, bf16) on the
layer shapes of the 16x4096 benchmark.  Prints one line per shape.

  python tools/gemm_yardstick.py [--reps 50]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_14312_b200 import kernels as K  # noqa: E402


def timeit(fn, reps):
    """Device time per call: `reps` calls captured in one CUDA graph (the
    per-call host cost of the ctypes path would otherwise dominate small
    kernels), replayed after warm-up, timed with CUDA events."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    g.replay()
    e1.record(st)
    e1.synchronize()
    return e0.elapsed_time(e1) * 1000.0 / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--n", type=int, default=4096)
    args = ap.parse_args()
    n = args.n
    out = []
    for m in (128, 256, 512, 1024):
        x = K.padded_bf16(m, n); x.normal_()
        w = K.padded_bf16(n, n); w.normal_()
        b = torch.zeros(n, device="cuda")
        y = K.padded_bf16(m, n)
        ours = timeit(lambda: K.linear_fwd(x, w, b, "relu", y16=y), args.reps)
        cub = timeit(lambda: torch.mm(x, w.t()), args.reps)
        out.append(("fwd", m, n, n, ours, cub))
    dz = K.padded_bf16(1024, n); dz.normal_()
    w = K.padded_bf16(n, n); w.normal_()
    xin = K.padded_bf16(1024, n); xin.normal_()
    d = K.padded_bf16(1024, n)
    ours = timeit(lambda: K.linear_bwd_dx(dz, w, xin, "relu", d), args.reps)
    cub = timeit(lambda: torch.mm(dz, w), args.reps)
    out.append(("dgrad", 1024, n, n, ours, cub))
    xx = K.padded_bf16(1024, n); xx.normal_()
    w32 = torch.zeros(n, n, device="cuda")
    w16 = K.padded_bf16(n, n)
    ours = timeit(lambda: K.linear_bwd_dw_sgd(dz, xx, w32, w32, w16, 0.0), args.reps)
    cub = timeit(lambda: torch.mm(dz.t(), xx), args.reps)
    out.append(("wgrad+sgd", n, n, 1024, ours, cub))
    for kind, m, nn, k, o, c in out:
        fl = 2.0 * m * nn * k
        print(json.dumps({"kind": kind, "M": m, "N": nn, "K": k, "ours_us": round(o, 2),
                          "ours_tflops": round(fl / o / 1e6, 1), "cublas_us": round(c, 2),
                          "cublas_tflops": round(fl / c / 1e6, 1)}))


if __name__ == "__main__":
    main()
