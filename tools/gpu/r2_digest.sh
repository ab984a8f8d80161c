# device digest parity + drop-in timing after the fast param path + racecheck re-run
mkdir -p gpurun_out
nproc > gpurun_out/r2d_nproc.txt; free -g >> gpurun_out/r2d_nproc.txt
timeout 900 python -m pytest tests/test_digest.py tests/test_cpp_dropin.py -q -m gpu -x -p no:cacheprovider > gpurun_out/r2d_pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/r2d_pytest.log
python - > gpurun_out/r2d_digest_speed.txt 2>&1 <<'PY'
import ctypes as C, numpy as np
from paper_2410_14312_b200 import _native as N
for n in (1<<20, 1<<24, 268500992):
    v = np.random.default_rng(0).normal(0, 0.02, n).astype(np.float32)
    out = C.create_string_buffer(17); ms = C.c_float()
    for _ in range(2):
        N.check(N.lib().pb_device_digest_f32(v.ctypes.data_as(C.POINTER(C.c_float)), n, out, C.byref(ms)))
    print(n, out.value.decode(), f"{ms.value:.2f} ms", f"{n/ms.value/1e6:.1f} Gvalues/s")
PY
cat gpurun_out/r2d_digest_speed.txt
for c in c1 c3; do timeout 600 tools/bin/dropin_bench $c 3 > gpurun_out/r2d_dropin_$c.json 2> gpurun_out/r2d_dropin_$c.err; echo dropin $c rc=$?; cat gpurun_out/r2d_dropin_$c.json; done
timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_run.py timeprest > gpurun_out/sanitize_racecheck2.log 2>&1; echo racecheck rc=$?; tail -2 gpurun_out/sanitize_racecheck2.log
