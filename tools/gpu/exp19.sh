mkdir -p gpurun_out; o=gpurun_out/exp19.txt; : > $o
PIPESIM_SPLITK=0 PIPESIM_FWD_BN=128 python tools/gemm_exp.py >> $o 2>&1
for r in 512 1024; do
PIPESIM_FWD_BN=128 PIPESIM_FWD_BN_ROWS=$r timeout 300 python bench.py --no-cpu-baseline > gpurun_out/b.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/b.json'));print('bn128 rows<=$r bench',d['value'],d['ms_per_step'], d['roofline']['in_step']['fwd'])" >> $o 2>&1
done
cat $o
