mkdir -p gpurun_out; o=gpurun_out/exp58.txt; : > $o
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -2 >> $o
timeout 300 python tools/fullwidth_check.py >> $o 2>&1
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1i.csv python tools/prof_step.py 4 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_r1i.csv >> $o
for r in 1 2; do
  timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/b58.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/b58.json'));print('bench', round(d['value']), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']), d['clocks']['sm_mhz'])" >> $o
done
cat $o
