# transitive pruning of cross-stream waits (PIPESIM_PRUNE_EDGES): the whole
# GPU suite, then C1 (TiMePReSt, 1F1B) and the 16x4096 step with and without
set -x
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
for rep in 1 2; do
  for v in 0 1; do
    echo "== PRUNE=$v rep $rep"
    PIPESIM_PRUNE_EDGES=$v timeout 300 python tools/c1_timeline.py 2>&1 | head -1
    PIPESIM_PRUNE_EDGES=$v timeout 300 python tools/c1_trace.py --mode pipedream 2>&1 | head -1
    PIPESIM_PRUNE_EDGES=$v PIPESIM_BENCH_VGG=0 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-dropin 2>/dev/null | python -c "import sys,json;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('bench', round(d['value']), d['clocks']['sm_mhz'])"
  done
done
python tools/c1_trace.py > gpurun_out/c1_trace_prune.log 2>&1; head -1 gpurun_out/c1_trace_prune.log
