mkdir -p gpurun_out; o=gpurun_out/exp24.txt; : > $o
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3 >> $o
python tools/diag_e2e.py >> $o 2>&1
cat $o
