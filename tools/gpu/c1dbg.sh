for v in 1 0; do PIPESIM_SPLIT_MASTER=$v timeout 300 python -m pytest tests/test_gpu_pipeline.py -q -x -k "c1_c2_mnist_shaped" 2>&1 | tail -2; done
python - <<'PY'
import os, sys
sys.path.insert(0,'.')
from paper_2410_14312_b200 import pipesim as P
net = P.NetworkSpec([784, 512, 256, 10], ["relu", "relu", "linear"], "softmax_cross_entropy")
s = P.Session(net, 2, 4, 256, 12, 0.05, "timeprest")
print("arena", s.arena_bytes if hasattr(s, "arena_bytes") else None)
PY
