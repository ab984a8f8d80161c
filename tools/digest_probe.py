"""Device digest timing for n fp32 values (ncu target / timing): python tools/digest_probe.py n"""
import ctypes as C, sys
import numpy as np
sys.path.insert(0, ".")
from paper_2410_14312_b200 import _native as N
n = int(sys.argv[1])
v = np.random.default_rng(0).standard_normal(n).astype(np.float32) * 0.01
out = C.create_string_buffer(17)
ms = C.c_float(0)
for _ in range(3):
    N.check(N.lib().pb_device_digest_f32(v.ctypes.data_as(C.POINTER(C.c_float)), n, out, C.byref(ms)))
    print(n, out.value.decode(), "device ms", ms.value)
