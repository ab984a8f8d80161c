# compute-sanitizer over the executor with the fused two-layer kernels
mkdir -p gpurun_out/san
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 1200 $CS --tool $tool --target-processes all --print-limit 50 python tools/sanitize_run.py > gpurun_out/san/sanitize_$tool.log 2>&1
  echo $tool rc=$?; tail -3 gpurun_out/san/sanitize_$tool.log
done
