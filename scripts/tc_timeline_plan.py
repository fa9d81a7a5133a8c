"""Timing experiment: timeline of CTA 0 of one tensor-core layer inside a ResNet-18 plan
run (BTNN_TC_DBG=16, BTNN_TC_DBG_NTH = launch index; 19 tensor-core launches per
forward, so the second forward's layer L (1-based conv index) is 19 + L - 1)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_16578_b200 import btnn, capi  # noqa: E402
from paper_2006_16578_b200 import model as M  # noqa: E402
from paper_2006_16578_b200 import weights as W  # noqa: E402

B = 512
m = M.stock_model("resnet18", 224, 224)
ws = W.build_weights(m, W.random_weights(m, 1))
plan = btnn.Plan(m, ws, B)
x = np.random.default_rng(2).standard_normal((B, 224, 224, 3), dtype=np.float32)
plan.run(x)
plan.run(x)
ts = np.zeros(4096, dtype=np.uint64)
capi.check(capi.lib().btnn_cuda_debug_tc_timestamps(ts.ctypes.data_as(C.POINTER(C.c_uint64)), 4096))
t = ts.astype(np.int64)
t0 = t[t > 0].min()
rel = lambda a: [int(v) - t0 if v else -1 for v in a]
print("K-steps: f prod_arrive mma_issue")
for f in range(0, 24):
    print(f, rel([t[f], t[1024 + f]]))
ep = t[3584:3584 + 400].reshape(200, 2)
print("epilogue tiles (start, end, dur):")
for i in range(16):
    if ep[i, 0]:
        print(i, int(ep[i, 0] - t0), int(ep[i, 1] - t0), int(ep[i, 1] - ep[i, 0]))
h = t[3072:3072 + 800].reshape(100, 8)
if h[:, 0].any():
    print("halo units: start freed built | mma_start mma_issued")
    for u in range(12):
        print(u, [int(v - t0) if v else -1 for v in h[u, :5]])
c = t[3968:3968 + 128].reshape(16, 8)
if c[:, 0].any():
    print("epilogue warp 0 chunk phases (clk): ld->tt | tt->loop | loop | ->store | store->issue-done")
    for k in range(12):
        r = c[k]
        print(k + 8, [int(r[1] - r[0]), int(r[3] - r[1]), int(r[4] - r[3]), int(r[5] - r[4]), int(r[6] - r[5])])
m = t[1024:1024 + 512].reshape(16, 32)
if m[:, 0].any() and not t[1024 + 16 * 32:1024 + 16 * 32 + 1].any():
    print("halo MMA issue stamps per tap (clk since the unit's first tap):")
    for u in range(8):
        r = m[u]
        if r[0]:
            print(u, [int(v - r[0]) for v in r[:9]])
p = t[2304:2304 + 320].reshape(40, 8)
if p[:, 0].any():
    print("producer thread 0 per K-step (i = 10..): issue | cp-wait | expand | st-wait+arrive | ->empty-wait | empty-wait | st (clk)")
    for k in range(12):
        r = p[k]
        if r[0]:
            print(k + 10, [int(r[j + 1] - r[j]) for j in range(7)])
