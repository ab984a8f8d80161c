"""Workload for compute-sanitizer (racecheck / synccheck / memcheck) on the
multi-stream executor: W=4 stages, N=2 micro-batches, one epoch per mode,
eager (no graph) and graph-captured, pair-kernel shapes (B=256 rows, widths
>= 256) plus a tiny-net epoch on the single-CTA kernels, and C1 at W=2 / W=1
(the fused two-layer dgrad and forward kernels, `chain2` / `chain1`).

  compute-sanitizer --tool racecheck python tools/sanitize_run.py [mode ...]
  python tools/sanitize_run.py --ipc     # 2-process IPC split on one GPU
"""
from __future__ import annotations

import multiprocessing as mp
import os
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

NETS = {
    "pair": ([256, 384, 256, 512, 256, 10], ["relu", "tanh", "relu", "sigmoid", "linear"], 256),
    "tiny": ([64, 96, 64, 48, 10], ["relu", "relu", "tanh", "linear"], 32),
    "chain2": ([784, 512, 256, 10], ["relu", "relu", "linear"], 256, 2),
    "chain1": ([784, 512, 256, 10], ["relu", "relu", "linear"], 256, 1),
}
W, N, M = 4, 2, 12


def one(kind, mode, graph, rank=0, world=1, blobs_fn=None):
    from paper_2410_14312_b200 import pipesim as P
    widths, acts, B = NETS[kind][:3]
    Wk = NETS[kind][3] if len(NETS[kind]) > 3 else W
    if Wk == 1 and mode != "sequential":
        return np.zeros(1)
    net = P.NetworkSpec(widths, acts, "softmax_cross_entropy")
    s = P.Session(net, Wk, N, B, M, 0.05, mode, use_graph=graph, rank=rank, world=world,
                  transport="ipc")
    s.load_params(P.init_network_params(net, 1))
    x, lab = P.make_classification_task(M * B, widths[0], widths[-1], seed=7, as_labels=True,
                                        dtype=np.float32)
    s.upload(x, lab, y_labels=True)
    if blobs_fn:
        s.ipc_connect(blobs_fn(s.ipc_export()))
    r = s.run_epoch()
    loss = r["mini_loss"].copy()
    s.close()
    return loss


def _ipc_worker(rank, world, port):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)

    def gather(b):
        out = [None] * world
        dist.all_gather_object(out, b)
        return out
    for mode in ("timeprest", "pipedream"):
        loss = one("pair", mode, False, rank, world, gather)
        print(f"rank {rank} {mode} ipc ok, loss[0] {loss[0]:.6f}", flush=True)
    dist.barrier()
    dist.destroy_process_group()


def main():
    args = sys.argv[1:]
    if args and args[0] == "--ipc":
        import socket
        so = socket.socket()
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
        so.close()
        ctx = mp.get_context("spawn")
        ps = [ctx.Process(target=_ipc_worker, args=(r, 2, port)) for r in range(2)]
        for p in ps:
            p.start()
        for p in ps:
            p.join()
        sys.exit(max(p.exitcode for p in ps))
    modes = args or ["timeprest", "pipedream", "sequential"]
    for mode in modes:
        for kind in ("pair", "tiny", "chain2", "chain1"):
            for graph in (False, True):
                loss = one(kind, mode, graph)
                print(f"{mode} {kind} graph={graph} ok, loss[0] {loss[0]:.6f}", flush=True)


if __name__ == "__main__":
    main()
