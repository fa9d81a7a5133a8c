"""Timing experiment: clock64 phase stamps of CTA 0 of the packed BMM kernel (timing build,
BTNN_LIB=.../libbtnn_cuda_timing.so): start, TMEM alloc, tiles staged, sync, expanded, MMA
issued, MMA done, epilogue done, dealloc."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_16578_b200 import capi  # noqa: E402

lib = capi.lib()
lib.btnn_cuda_debug_bmm_timestamps.argtypes = [C.POINTER(C.c_uint64), C.c_size_t]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
med, mn = C.c_double(), C.c_double()
eng = C.create_string_buffer(16)
capi.check(lib.btnn_cuda_bench_bmm(n, 0, 20, 5, C.byref(med), C.byref(mn), eng, 16, None))
ts = np.zeros(16 + 2048, dtype=np.uint64)
capi.check(lib.btnn_cuda_debug_bmm_timestamps(ts.ctypes.data_as(C.POINTER(C.c_uint64)), ts.size))
t = ts.astype(np.int64)
names = ["start", "staged", "alloc (w0)", "sync", "expanded", "mma-issued", "mma-done", "epilogue", "dealloc"]
print("median call us", med.value / 1e3, "engine", eng.value)
for i in range(1, 9):
    print(f"{names[i]:12s} +{t[i] - t[i - 1]:6d} clk  (cumulative {t[i] - t[0]})")

ctas = ((n + 63) // 64) * ((n + 127) // 128)
g = ts[16:16 + 2 * ctas].astype(np.int64).reshape(ctas, 2)
g0 = g[:, 0].min()
st, en = g[:, 0] - g0, g[:, 1] - g0
print(f"CTAs {ctas}: start spread {st.min()}..{st.max()} ns (median {int(np.median(st))}), "
      f"end {en.min()}..{en.max()} ns, span per CTA median {int(np.median(en - st))} ns")
