# in-epoch digests: parity + full GPU suite + drop-in timing + digest speed
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_digest.py -q -m gpu -x -p no:cacheprovider > gpurun_out/r2e_digest.log 2>&1; echo digest-tests rc=$?; tail -3 gpurun_out/r2e_digest.log
python - > gpurun_out/r2e_digest_speed.txt 2>&1 <<'PY'
import ctypes as C, numpy as np
from paper_2410_14312_b200 import _native as N
for n in (1<<24, 268500992):
    v = np.random.default_rng(0).normal(0, 0.02, n).astype(np.float32)
    out = C.create_string_buffer(17); ms = C.c_float()
    for _ in range(2):
        N.check(N.lib().pb_device_digest_f32(v.ctypes.data_as(C.POINTER(C.c_float)), n, out, C.byref(ms)))
    print(n, out.value.decode(), f"{ms.value:.2f} ms", f"{n/ms.value/1e6:.2f} Gvalues/s")
PY
cat gpurun_out/r2e_digest_speed.txt
for c in c1 c3; do for d in auto final; do timeout 600 tools/bin/dropin_bench $c 3 $d > gpurun_out/r2e_dropin_${c}_$d.json 2> gpurun_out/r2e_dropin_${c}_$d.err; echo dropin $c $d rc=$?; cat gpurun_out/r2e_dropin_${c}_$d.json; done; done
timeout 1500 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/r2e_pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/r2e_pytest.log
