# 64-wide CTA-pair forward tiles (PIPESIM_PAIR_BN64): parity, VGG-16 per-layer
# forward times and the VGG step with and without; the 16x4096 step with and
# without the 64-wide single-CTA tiles (PIPESIM_BN64=0)
set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "conv or fwd or convnet" 2>&1 | tail -3
for v in 0 1; do PIPESIM_PAIR_BN64=$v timeout 300 python tools/vgg_layers.py --n 64 2>&1 | head -3; done
for rep in 1 2; do
  for v in 0 1; do
    echo "== PAIR_BN64=$v rep $rep"
    PIPESIM_PAIR_BN64=$v timeout 600 python tools/vgg_bench.py --W 4 --reps 3 2>&1 | python -c "import sys,json;[print(round(json.loads(l)['images_per_s']), round(json.loads(l)['epoch_ms'],2)) for l in sys.stdin if l.startswith('{')]"
  done
done
for rep in 1 2; do
  for v in 0 8; do
    echo "== BN64=$v rep $rep"
    PIPESIM_BN64=$v PIPESIM_BENCH_VGG=0 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-dropin 2>/dev/null | python -c "import sys,json;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(round(d['value']), d['clocks']['sm_mhz'])"
  done
done
