"""Times the three layer-GEMM shapes of the C3 workload (CUDA events)."""
import json, os, sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import bench
r = bench.kernel_roofline(bench._peaks())
print(os.environ.get("PIPESIM_EPI", "auto"), os.environ.get("PIPESIM_GEMM", "auto"),
      json.dumps({k: round(v["us"], 1) for k, v in r["per_shape"].items()}))
