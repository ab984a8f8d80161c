# 64-wide single-CTA tiles (PIPESIM_BN64): parity with every single-CTA GEMM
# forced to BN=64, then C1 / C2 per-mini-batch time with and without
set -x
PIPESIM_BN64=100000 timeout 900 python -m pytest tests -m gpu -x -q -k "kernel or gemm or session or mlp" 2>&1 | tail -5
for rep in 1 2; do
  for v in 0 8 16; do
    echo "== BN64=$v rep $rep"
    PIPESIM_BN64=$v timeout 300 python tools/c1_timeline.py 2>&1 | head -1
  done
done
