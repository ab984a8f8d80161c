mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -2
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1h.csv python tools/prof_step.py 4 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_r1h.csv
