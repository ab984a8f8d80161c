mkdir -p gpurun_out; o=gpurun_out/exp12.txt; : > $o
PIPESIM_SPLITK=0 python tools/gemm_exp.py >> $o 2>&1
timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_pipeline.py -q -x 2>&1 | tail -2 >> $o
python - >> $o 2>&1 <<'PY'
import sys, numpy as np
sys.path.insert(0, ".")
from paper_2410_14312_b200 import pipesim as P
net = P.NetworkSpec([4096] * 17, ["relu"] * 15 + ["linear"], "softmax_cross_entropy")
for W, N in ((8, 8), (4, 8), (2, 4)):
    B, M = 1024, 2 * (W + N)
    s = P.Session(net, W, N, B, M, 0.05, "timeprest")
    s.load_params(P.init_network_params(net, 1))
    x, lab = P.make_classification_task(M * B, 4096, 4096, seed=7, as_labels=True, dtype=np.float32)
    s.upload(x, lab, y_labels=True)
    s.run_epoch()
    r = s.profile_epoch()
    g = s.run_epoch()
    pr = r["profile"]
    print(W, N, "graph ms", round(g["device_ms"], 2), "profiled ms", round(pr["makespan_ms"], 2), "bubble", round(pr["bubble"], 4), "nodes", len(pr["nodes"]))
    s.close()
PY
cat $o
