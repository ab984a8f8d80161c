"""Calibration of the conv pipeline parity bars (GPU box)."""
import sys
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
import test_gpu_convnet as T  # noqa: E402
for storage in ["bf16", "fp64"]:
    for (W, N) in [(2, 2), (3, 4), (5, 2)]:
        net = T._small(); B, M, lr = 8, 2 * (W + N), 0.002
        o, r, g, p = T._run(net, W, N, B, M, lr, storage=storage)
        print(storage, W, N, end=' '); T._check(o, r, g, p, W, M, "timeprest", 1, 1, 10)
    for mode in ["pipedream", "sequential"]:
        net = T._small(); o, r, g, p = T._run(net, 2, 2, 8, 6, 0.002, mode=mode, storage=storage)
        print(storage, mode, end=' '); T._check(o, r, g, p, 2, 6, mode, 1, 1, 10)
    net = T._small(image=32, cfg=(64, "M", 128, 128, "M", 256, "M"), hidden=64)
    o, r, g, p = T._run(net, 3, 2, 4, 10, 0.0005, epochs=2, storage=storage)
    print(storage, "wide", end=' '); T._check(o, r, g, p, 3, 10, "timeprest", 1, 1, 10)
