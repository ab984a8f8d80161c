"""Times the C3 layer-GEMM shapes alone (the bench's `alone_us`: CUDA graph,
weights rotated through HBM) for the current PIPESIM_* environment:
python tools/gemm_probe.py [rows ...]"""
import json
import os
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import bench  # noqa: E402

rows = [int(v) for v in sys.argv[1:]] or [128, 256, 768, 1024]
out = {f"fwd{m}": round(bench.alone_us("fwd", m), 1) for m in rows}
out["dgrad1024"] = round(bench.alone_us("dgrad", 1024), 1)
out["wgrad1024"] = round(bench.alone_us("wgrad", 1024), 1)
env = {k: v for k, v in os.environ.items() if k.startswith("PIPESIM_")}
print(json.dumps({"env": env, "us": out}))
