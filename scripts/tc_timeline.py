"""Timing experiment: per-K-step timeline of CTA 0 of the tensor-core conv kernel
(BTNN_TC_DBG=16), for a ResNet-18 56x56x64 threshold layer at batch 512."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_16578_b200 import capi  # noqa: E402

lib = capi.lib()
hw, n, c, o = (int(v) for v in (sys.argv[1:5] if len(sys.argv) > 4 else (56, 512, 64, 64)))
med, mn = C.c_double(), C.c_double()
eng = C.create_string_buffer(32)
capi.check(lib.btnn_cuda_bench_bconv(hw, n, c, o, 3, 1, 3, 1, C.byref(med), C.byref(mn), eng, 32, None))
ts = np.zeros(4096, dtype=np.uint64)
capi.check(lib.btnn_cuda_debug_tc_timestamps(ts.ctypes.data_as(C.POINTER(C.c_uint64)), 4096))
t0 = int(min(v for v in ts if v > 0))
rel = lambda a: [int(v) - t0 if v else -1 for v in a]
prod, mma, epi, emp = rel(ts[:1024]), rel(ts[1024:2048]), rel(ts[2048:2176]), rel(ts[2176:2304])
print("median us", med.value / 1e3, eng.value)
print("f  prod_arrive  mma_issue  empty_done")
for f in range(0, 60):
    print(f, prod[f], mma[f], emp[f] if f < 128 else None)
print("epilogue tile starts", epi[:12])
steps = [v for v in mma if v >= 0]
print("mma issue deltas (mean over 100..400):", np.diff(steps[100:400]).mean() if len(steps) > 400 else None)
it = ts[2304:2304 + 320].astype(np.int64).reshape(40, 8)
print("producer group 0 thread 0, per-iteration phase durations (clk):")
print(" top->issued issued->cpwait cpwait->expanded expanded->stwait stwait->arrived arrived->emptyok emptyok->sttm sttm->next")
for r in range(39):
    d = np.diff(np.append(it[r], it[r + 1][0]))
    print(r + 10, d.tolist())
h = ts[3072:3072 + 800].astype(np.int64).reshape(100, 8)
if h[:, 0].any():
    hb = h[h > 0].min()
    print("halo units: start freed built | mma_start mma_issued   (clk)")
    for u in range(24):
        print(u, (h[u, :5] - hb).tolist())
