mkdir -p gpurun_out; o=gpurun_out/exp15.txt; : > $o
for p in 74 60 48 37; do
  echo "pairs $p" >> $o
  PIPESIM_WG_PAIRS=$p python tools/gemm_exp.py >> $o 2>&1
  PIPESIM_WG_PAIRS=$p timeout 300 python bench.py --no-cpu-baseline > gpurun_out/b.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/b.json'));print('bench',d['value'],d['ms_per_step'])" >> $o 2>&1
done
cat $o
