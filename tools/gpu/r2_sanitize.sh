# compute-sanitizer racecheck / synccheck / memcheck over the executor + memory report.
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
python tools/memory_report.py --measure --md gpurun_out/memory_r2.md --json gpurun_out/memory_r2.json > /dev/null 2> gpurun_out/memory_r2.err; echo memreport rc=$?
for tool in racecheck synccheck memcheck; do
  timeout 900 $CS --tool $tool --target-processes all --print-limit 50 python tools/sanitize_run.py > gpurun_out/sanitize_$tool.log 2>&1
  echo $tool rc=$?; tail -3 gpurun_out/sanitize_$tool.log
done
timeout 600 $CS --tool racecheck --target-processes all --print-limit 50 python tools/sanitize_run.py --ipc > gpurun_out/sanitize_racecheck_ipc.log 2>&1; echo racecheck-ipc rc=$?; tail -3 gpurun_out/sanitize_racecheck_ipc.log
timeout 600 $CS --tool memcheck --target-processes all --print-limit 50 python tools/sanitize_run.py --ipc > gpurun_out/sanitize_memcheck_ipc.log 2>&1; echo memcheck-ipc rc=$?; tail -3 gpurun_out/sanitize_memcheck_ipc.log
