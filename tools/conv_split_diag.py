"""Conv pipeline split over processes vs one process, per stage split."""
import multiprocessing as mp
import os
import sys
import numpy as np
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import test_gpu_multiproc as T  # noqa: E402

W, N, B, M = 2, 4, 64, 8


def net_for(split):
    from paper_2410_14312_b200 import convnet as CN
    net = CN.vgg((64, "M", 64, 128, "M"), image=16, classes=10, hidden=64, fc_layers=2)
    net.stage_layers = split
    return net


def worker(rank, world, port, split, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), PIPESIM_SESSION_SPLIT="0")
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2410_14312_b200 import convnet as CN
    from paper_2410_14312_b200 import pipesim as P
    net = net_for(split)
    x, lab = CN.synthetic_images(M * B, net, seed=7)
    s = P.Session(net, len(split), N, B, M, 0.002, rank=rank, world=world, transport="ipc")
    s.load_params(CN.init_params(net, 1))
    s.upload(x, lab, y_labels=True)
    blobs = [None] * world
    dist.all_gather_object(blobs, s.ipc_export())
    s.ipc_connect(blobs)
    r = s.run_epoch()
    q.put((rank, r["mini_loss"].copy(), s.read_params()))
    s.close()
    dist.barrier()
    dist.destroy_process_group()


def single(split):
    os.environ["PIPESIM_SESSION_SPLIT"] = "0"
    from paper_2410_14312_b200 import convnet as CN
    from paper_2410_14312_b200 import pipesim as P
    net = net_for(split)
    x, lab = CN.synthetic_images(M * B, net, seed=7)
    s = P.Session(net, len(split), N, B, M, 0.002)
    s.load_params(CN.init_params(net, 1))
    s.upload(x, lab, y_labels=True)
    r = s.run_epoch()
    return r["mini_loss"].copy(), s.read_params()


if __name__ == "__main__":
    for split in ([1, 4], [2, 3], [3, 2], [4, 1]):
        world = 2
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        port = T._free_port()
        procs = [ctx.Process(target=worker, args=(r, world, port, split, q)) for r in range(world)]
        for p in procs:
            p.start()
        res = {}
        for _ in range(world):
            rank, loss, params = q.get(timeout=240)
            res[rank] = (loss, params)
        for p in procs:
            p.join()
        l0, p0 = single(split)
        print(split, "loss max diff", np.abs(res[1][0] - l0).max(),
              "first differing mini", int(np.argmax(res[1][0] != l0)) if np.any(res[1][0] != l0) else None)
