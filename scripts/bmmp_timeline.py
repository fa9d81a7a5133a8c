"""Timing experiment: per-K-step clock64 stamps of CTA (0, 0) of the pipelined packed BMM
(timing build, BTNN_LIB=.../libbtnn_cuda_timing.so): MMA issue, A / B producer arrive and
empty-wait times. Usage: python scripts/bmmp_timeline.py [n]"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_16578_b200 import capi  # noqa: E402

lib = capi.lib()
lib.btnn_cuda_debug_bmm_timestamps.argtypes = [C.POINTER(C.c_uint64), C.c_size_t]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
capi.set_bmm_kernel(capi.BMM_PIPELINED)
med, mn = C.c_double(), C.c_double()
eng = C.create_string_buffer(24)
capi.check(lib.btnn_cuda_bench_bmm(n, 1, 3, 1, C.byref(med), C.byref(mn), eng, 24, None))
ts = np.zeros(16 + 2048 + 384, dtype=np.uint64)
capi.check(lib.btnn_cuda_debug_bmm_timestamps(ts.ctypes.data_as(C.POINTER(C.c_uint64)), ts.size))
t = ts[16 + 2048:].astype(np.int64).reshape(6, 64)
t0 = t[0][t[0] > 0].min()
print("median call us", med.value / 1e3, eng.value)
print("step: mma_issue | A ready, A empty-done, A arrive | B empty-done, B arrive   (clk rel. to first MMA)")
for s in range(64):
    r = [t[0, s], t[5, s], t[3, s], t[1, s], t[4, s], t[2, s]]
    print(s, [int(x - t0) if x > 0 else -1 for x in r], "dMMA", int(t[0, s] - t[0, s - 1]) if s else 0)

# per-CTA globaltimer start / end (ns) of the first 1024 CTAs (the A-ready row above is
# overwritten by the SM ids of CTAs 0..63 at their end)
g = ts[16:16 + 2048].astype(np.int64).reshape(1024, 2)
ok = (g[:, 0] > 0) & (g[:, 1] > g[:, 0])
st, en = g[ok, 0], g[ok, 1]
dur = en - st
print(f"CTAs {ok.sum()}: duration ns median {np.median(dur):.0f} min {dur.min()} max {dur.max()}")
print(f"span of these CTAs {(en.max() - st.min()) / 1e3:.1f} us; start offsets of CTAs 0..9 (ns):",
      (st[:10] - st.min()).tolist())
o = np.argsort(st)
print("sorted starts (us) every 148th:", [round((st[o][k] - st.min()) / 1e3, 1) for k in range(0, len(o), 148)])
