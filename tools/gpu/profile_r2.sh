# Round-2 evidence run: tests, smoke, bench, launch list + ncu --set full of
# the step's GEMMs, C5 sweep, other configs, VGG-16 step and layer table.
mkdir -p gpurun_out/r2p
O=gpurun_out/r2p
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -1 $O/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$?; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo bench rc=$?
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_step_m4.csv python tools/prof_step.py 4 > $O/prof_step.log 2>&1; echo ncu-list rc=$?
python tools/launch_summary.py $O/launches_step_m4.csv > $O/launch_summary.txt 2>&1
PIPESIM_SPLITK=0 timeout 400 ncu --set full --clock-control none --import-source on -k regex:gemm -c 3 -o $O/ncu_gemm_r2 python tools/prof_gemm.py fwd1024,dgrad,wgrad 1 > $O/prof_gemm.log 2>&1; echo ncu-full rc=$?
python tools/ncu_summary.py $O/ncu_gemm_r2.ncu-rep > $O/ncu_gemm_r2.md 2>&1
timeout 900 python tools/sweep.py --out $O/sweep_c5_r2.json > $O/sweep_c5_r2.md 2> $O/sweep.err; echo sweep rc=$?
timeout 600 python tools/configs.py --out $O/configs_r2.json > $O/configs_r2.md 2> $O/configs.err; echo configs rc=$?
timeout 600 python tools/vgg_bench.py --W 4 8 --M 16 --profile --out $O/vgg16_bench.json > /dev/null 2> $O/vgg.err; echo vgg rc=$?
timeout 600 python tools/vgg_layers.py --out $O/vgg16_layers_alone.json > /dev/null 2>&1; echo vggl rc=$?
