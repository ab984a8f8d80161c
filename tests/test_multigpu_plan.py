"""Cross-GPU pipeline split, host side (no GPU needed): every rank's
point-to-point program must pair up with its neighbours' — same number of
messages, same sizes, same order per boundary and direction — for every
world size, mode and coalescing setting.  Also run as a real 2-process
gloo job (world_size 2) exchanging the per-rank programs."""
import os
import socket

import pytest

from paper_2410_14312_b200 import pipesim as P

NET16 = P.NetworkSpec([256] * 17, ["relu"] * 15 + ["linear"], "softmax_cross_entropy")
NET_C1 = P.NetworkSpec([784, 512, 256, 10], ["relu", "relu", "linear"], "softmax_cross_entropy")


def _check_pairing(programs, world):
    for r in range(world - 1):
        for direction, src, dst in ((0, r, r + 1), (1, r + 1, r)):
            sent = [b for k, d, p, b in programs[src] if k == "send" and d == direction and p == dst]
            recv = [b for k, d, p, b in programs[dst] if k == "recv" and d == direction and p == src]
            assert sent == recv, (r, direction)
            assert sent, "every boundary carries traffic"
    for r in range(world):  # only neighbours talk
        assert all(abs(p - r) == 1 for _, _, p, _ in programs[r])


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("mode", ["timeprest", "pipedream", "sequential"])
@pytest.mark.parametrize("merge", [0, 1])
def test_transfer_programs_pair_up(world, mode, merge):
    progs = [P.plan_transfers(NET16, 8, 8, 1024, 6, mode, r, world, merge) for r in range(world)]
    _check_pairing(progs, world)
    # message counts: one delta per mini-batch per boundary; activations per
    # coalesced forward group (== micro-batches when merge=1)
    for r in range(world - 1):
        deltas = [m for m in progs[r + 1] if m[0] == "send" and m[1] == 1]
        assert len(deltas) == 6
        acts = [m for m in progs[r] if m[0] == "send" and m[1] == 0]
        if merge == 1 and mode == "timeprest":
            assert len(acts) == 6 * 8
        assert sum(m[3] for m in acts) == 6 * 1024 * 256 * 2  # every row crosses once


def test_c1_two_stages_two_gpus():
    progs = [P.plan_transfers(NET_C1, 2, 4, 256, 12, "timeprest", r, 2) for r in range(2)]
    _check_pairing(progs, 2)
    assert sum(b for k, d, p, b in progs[0] if k == "send") == 12 * 256 * 512 * 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2410_14312_b200 import pipesim as PP
    mine = PP.plan_transfers(NET16, 8, 8, 1024, 4, "timeprest", rank, world)
    ids = [os.urandom(128 * 2 * (world - 1))] if rank == 0 else [None]
    dist.broadcast_object_list(ids, src=0)  # how bench.py shares the NCCL ids
    allp = [None] * world
    dist.all_gather_object(allp, mine)
    ids_all = [None] * world
    dist.all_gather_object(ids_all, ids[0])
    if rank == 0:
        try:
            _check_pairing(allp, world)
            assert all(x == ids_all[0] for x in ids_all)
            q.put("ok")
        except AssertionError as e:  # noqa: PERF203
            q.put(f"fail {e}")
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_two_process_exchange():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(180)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=10) == "ok"


@pytest.mark.parametrize("mode", ["timeprest", "pipedream"])
@pytest.mark.parametrize("W,N", [(2, 4), (4, 2), (8, 8)])
def test_plan_memory_matches_slot_model(mode, W, N):
    """The session's weight-version pool per stage is exactly the slot
    model's peak retained versions (metrics.cpp:73-75 /
    build_retention_timeline), and TiMePReSt never holds more bytes than
    PipeDream (the paper's memory claim)."""
    widths = [64] * (W + 1)
    net = P.NetworkSpec(widths, ["relu"] * (W - 1) + ["linear"], "softmax_cross_entropy")
    M = 2 * (W + N)
    cfg = P.SimConfig(workers=W, micro_batches=N, mini_batches=M, samples_per_mini_batch=8 * N)
    grid = P.build_nf1b_schedule(cfg) if mode == "timeprest" else P.build_1f1b_schedule(cfg)
    tl = P.build_retention_timeline(P.assign_versions(grid, cfg), grid)
    mem = P.plan_memory(net, W, N, 8 * N, M, mode=mode)
    assert mem["pool"].tolist() == list(tl.peak_concurrent)
    assert (mem["weight_bytes"] > 0).all() and (mem["act_bytes"] > 0).all()
    if mode == "pipedream":
        t = P.plan_memory(net, W, N, 8 * N, M, mode="timeprest")
        assert (t["weight_bytes"] <= mem["weight_bytes"]).all()
        assert (t["weight_bytes"] + t["act_bytes"] <= mem["weight_bytes"] + mem["act_bytes"]).all()
    # split across ranks: each rank accounts only for its own stages
    half = P.plan_memory(net, W, N, 8 * N, M, mode=mode, rank=0, world=2)
    assert (half["weight_bytes"][W // 2:] == 0).all()
    assert (half["weight_bytes"][:W // 2] == mem["weight_bytes"][:W // 2]).all()
