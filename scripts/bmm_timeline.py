"""Timing experiment (timing build, BTNN_TC_DBG=16): timeline of CTA 0 of the bmm_pm1 GEMM
(n x n x n packed operands) — producer arrivals, MMA issue and epilogue start per tile."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_16578_b200 import capi  # noqa: E402

lib = capi.lib()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
med, mn, kern = C.c_double(), C.c_double(), C.c_double()
eng = C.create_string_buffer(32)
rb = capi.BenchReadback(None, None, None, C.pointer(kern))
capi.check(lib.btnn_cuda_bench_bmm(n, 0, 5, 2, C.byref(med), C.byref(mn), eng, 32, C.byref(rb)))
ts = np.zeros(4096, dtype=np.uint64)
capi.check(lib.btnn_cuda_debug_tc_timestamps(ts.ctypes.data_as(C.POINTER(C.c_uint64)), 4096))
t = ts.astype(np.int64)
t0 = int(t[t > 0].min())
rel = lambda a: [int(v) - t0 if v else -1 for v in a]
print("call us", med.value / 1e3, "gemm us", kern.value / 1e3, eng.value, capi.last_tc_launch())
print("f  prod_arrive  mma_issue")
for f in range(0, 24):
    print(f, rel([t[f], t[1024 + f]]))
print("epilogue tile starts", rel(t[2048:2056]))
