# 64-wide pair conv dgrad for Cin = 64 (PIPESIM_DGRAD_BN64): parity first
# (under a short timeout), then the VGG layer table and step
set -x
timeout 300 python -m pytest tests/test_gpu_conv.py -x -q -k "dx" 2>&1 | tail -3 || exit 1
timeout 600 python -m pytest tests/test_gpu_conv.py tests/test_gpu_convnet.py -x -q 2>&1 | tail -2
for v in 0 1; do PIPESIM_DGRAD_BN64=$v timeout 300 python tools/vgg_layers.py --n 64 2>&1 | head -2; done
for rep in 1 2; do
  for v in 0 1; do
    echo "== DGRAD_BN64=$v rep $rep"
    PIPESIM_DGRAD_BN64=$v timeout 600 python tools/vgg_bench.py --W 4 --reps 3 2>&1 | python -c "import sys,json;[print(round(json.loads(l)['images_per_s']), round(json.loads(l)['epoch_ms'],2)) for l in sys.stdin if l.startswith('{')]"
  done
done
