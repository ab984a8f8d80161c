mkdir -p gpurun_out; o=gpurun_out/exp16.txt; : > $o
for v in 0 1; do
  PIPESIM_SESSION_SPLIT=$v timeout 300 python bench.py --no-cpu-baseline > gpurun_out/b.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/b.json'));print('split',$v,'bench',d['value'],d['ms_per_step'])" >> $o 2>&1
done
PIPESIM_FWD_MERGE=1 timeout 300 python bench.py --no-cpu-baseline > gpurun_out/b.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/b.json'));print('merge1 bench',d['value'],d['ms_per_step'])" >> $o 2>&1
PIPESIM_FWD_MERGE=1 PIPESIM_SESSION_SPLIT=1 timeout 300 python bench.py --no-cpu-baseline > gpurun_out/b.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/b.json'));print('merge1 split bench',d['value'],d['ms_per_step'])" >> $o 2>&1
python - >> $o 2>&1 <<'PY'
import sys, numpy as np
sys.path.insert(0, ".")
from paper_2410_14312_b200 import pipesim as P
net = P.NetworkSpec([4096] * 17, ["relu"] * 15 + ["linear"], "softmax_cross_entropy")
W, N, B, M = 8, 8, 1024, 32
x, lab = P.make_classification_task(M * B, 4096, 4096, seed=7, as_labels=True, dtype=np.float32)
for kind in ("fwd", "dgrad", "wgrad"):
    s = P.Session(net, W, N, B, M, 0.05, "timeprest", timed_kernel=kind)
    s.load_params(P.init_network_params(net, 1))
    s.upload(x, lab, y_labels=True)
    for _ in range(3): r = s.run_epoch()
    t = s.kernel_times_ms()
    print(kind, "epoch ms", round(r["device_ms"], 2), "launches", len(t), "mean us", round(1000 * float(t.mean()), 2), "sum ms", round(float(t.sum()), 2))
    s.close()
PY
cat $o
