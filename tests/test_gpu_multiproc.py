"""Stage split across processes on the real device path: two processes share
cuda:0, each owns half of the pipeline stages, and activations / deltas cross
the process boundary through the CUDA IPC peer-memory transport
(csrc/ipc_p2p.cpp: copy straight into the receiver's slot, device-side
posted/done handshake).  The split run must reproduce the single-process
session bit for bit (same kernels, same inputs, same schedule): per-mini-batch
losses, every stage's final weights and the device version traces.  The same
code path runs one process per GPU over NVLink."""
import multiprocessing as mp
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

NET = ([96, 128, 128, 96, 64, 10], ["relu", "relu", "tanh", "relu", "linear"])
W, N, B, M, LR = 4, 4, 64, 8, 0.05


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _net(kind):
    """(network, initial params, x, labels, per-stage parameter counts)."""
    from paper_2410_14312_b200 import pipesim as P
    if kind == "conv":  # VGG-style conv stages (pooled convs, then linear layers)
        from paper_2410_14312_b200 import convnet as CN
        net = CN.vgg((64, "M", 64, 128, "M"), image=16, classes=10, hidden=64, fc_layers=2)
        x, lab = CN.synthetic_images(M * B, net, seed=7)
        split = net.partition(W)
        sizes, at = [], 0
        for c in split:
            sizes.append(sum(l.param_count() for l in net.layers[at:at + c]))
            at += c
        return net, CN.init_params(net, 1), x, lab, sizes
    net = P.NetworkSpec(*NET, "softmax_cross_entropy")
    x, lab = P.make_classification_task(M * B, NET[0][0], NET[0][-1], seed=7, as_labels=True,
                                        dtype=np.float32)
    return net, P.init_network_params(net, 1), x, lab, \
        [st.param_count() for st in P.partition_model(net, W)]


# split-K forwards follow stages-per-process (session.cu); pin them off so the
# split and single-process runs sum in the same order
_NO_SPLIT = {"PIPESIM_SESSION_SPLIT": "0"}


def _worker(rank, world, port, mode, q, kind="mlp"):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), **_NO_SPLIT)
        import torch.distributed as dist
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2410_14312_b200 import pipesim as P
        net, p0, x, lab, _ = _net(kind)
        s = P.Session(net, W, N, B, M, LR if kind == "mlp" else 0.002, mode, rank=rank,
                      world=world, transport="ipc")
        s.load_params(p0)
        s.upload(x, lab, y_labels=True)
        blobs = [None] * world
        dist.all_gather_object(blobs, s.ipc_export())
        s.ipc_connect(blobs)
        outs = []
        for _ in range(2):
            r = s.run_epoch()
            outs.append((r["mini_loss"].copy(), r["dev_fwd"].copy(), r["dev_bwd"].copy(),
                         r["dev_current"].copy()))
        params = s.read_params()
        s.close()
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, outs, params))
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e), None))


def _single(mode, kind="mlp"):
    from paper_2410_14312_b200 import pipesim as P
    net, p0, x, lab, _ = _net(kind)
    saved = os.environ.get("PIPESIM_SESSION_SPLIT")
    os.environ.update(_NO_SPLIT)
    try:
        s = P.Session(net, W, N, B, M, LR if kind == "mlp" else 0.002, mode)
    finally:
        if saved is None:
            os.environ.pop("PIPESIM_SESSION_SPLIT")
        else:
            os.environ["PIPESIM_SESSION_SPLIT"] = saved
    s.load_params(p0)
    s.upload(x, lab, y_labels=True)
    outs = []
    for _ in range(2):
        r = s.run_epoch()
        outs.append((r["mini_loss"].copy(), r["dev_fwd"].copy(), r["dev_bwd"].copy(),
                     r["dev_current"].copy()))
    params = s.read_params()
    stage_ranges = [(s.stage_first_layer[i], s.stage_layers[i]) for i in range(W)] \
        if hasattr(s, "stage_first_layer") else None
    s.close()
    return outs, params, stage_ranges


@pytest.mark.parametrize("mode,world,kind", [("timeprest", 2, "mlp"), ("pipedream", 2, "mlp"),
                                             ("timeprest", 4, "mlp"), ("sequential", 2, "mlp"),
                                             ("timeprest", 2, "conv"), ("timeprest", 4, "conv")])
def test_multi_process_stage_split_matches_single_process(mode, world, kind):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, q, kind))
             for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    try:
        for _ in range(world):
            rank, outs, params = q.get(timeout=240)
            assert not isinstance(outs, str), f"rank {rank}: {outs}"
            res[rank] = (outs, params)
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    ref_outs, ref_params, _ = _single(mode, kind)
    sizes = _net(kind)[4]
    owner = [s * world // W for s in range(W)]
    for e in range(2):
        # losses come from the rank owning the last stage
        np.testing.assert_array_equal(res[world - 1][0][e][0], ref_outs[e][0])
        for s in range(W):
            r = owner[s]
            if mode != "sequential":  # (sequential has no per-micro forward trace)
                np.testing.assert_array_equal(res[r][0][e][1][:, :, s], ref_outs[e][1][:, :, s])
            np.testing.assert_array_equal(res[r][0][e][2][:, s], ref_outs[e][2][:, s])
            assert res[r][0][e][3][s] == ref_outs[e][3][s]
    off = 0
    for s, n in enumerate(sizes):
        np.testing.assert_array_equal(res[owner[s]][1][off:off + n], ref_params[off:off + n])
        off += n
