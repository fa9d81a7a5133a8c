"""Timing experiment: per-tile timeline of CTA 0 of the tensor-core first layer
(BTNN_FTC_DBG=1) on a ResNet-18 plan at batch 512."""
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
ts = np.zeros(640, dtype=np.uint64)
capi.check(capi.lib().btnn_cuda_debug_ftc_timestamps(ts.ctypes.data_as(C.POINTER(C.c_uint64)), 640))
t = ts[:512].astype(np.int64).reshape(64, 8)
t0 = t[t > 0].min()
print("tile: bstart bfree bdone | mma_start mma_issued | epi_start epi_done  (clk rel. to first stamp)")
for i in range(40):
    print(i, (t[i, :7] - t0).tolist())

e = ts[512:640].astype(np.int64).reshape(8, 2, 8)
print("epilogue warp 0, tiles 20..27, per group: acc-wait | ld | process | ld | process | tap store | bits (clk)")
for i in range(8):
    print(i + 20, [np.diff(e[i, g, :7]).tolist() for g in range(2)], "gap to next group", int(e[i, 1, 0] - e[i, 0, 6]))
