"""Timing experiment: where the end-to-end plan_run time goes (ResNet-18, batch 512)."""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_16578_b200 import btnn, capi  # noqa: E402
from paper_2006_16578_b200 import model as M  # noqa: E402
from paper_2006_16578_b200 import weights as W  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 512
m = M.stock_model("resnet18", 224, 224)
ws = W.build_weights(m, W.random_weights(m, 1))
plan = btnn.Plan(m, ws, B)
lib = capi.lib()
xh = torch.randn((B, 224, 224, 3), dtype=torch.float32).pin_memory()
lh = torch.empty((B, 1000), dtype=torch.float64).pin_memory()
bh = torch.empty((B,), dtype=torch.int32).pin_memory()
def run():
    capi.check(lib.btnn_cuda_plan_run(plan.h, C.cast(xh.data_ptr(), C.POINTER(C.c_float)), B,
                                      C.cast(lh.data_ptr(), C.POINTER(C.c_double)), C.cast(bh.data_ptr(), C.POINTER(C.c_int32))))
for _ in range(3): run()
t = time.perf_counter()
for _ in range(10): run()
dt = (time.perf_counter() - t) / 10
print(f"plan_run B={B}: {dt*1e3:.2f} ms  ({B/dt:.0f} img/s)")
xd = torch.empty_like(xh, device="cuda")
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(10): xd.copy_(xh, non_blocking=True)
torch.cuda.synchronize()
print(f"H2D alone: {(time.perf_counter()-t)/10*1e3:.2f} ms")
ld = torch.empty((B, 1000), dtype=torch.float64, device="cuda"); bd = torch.empty((B,), dtype=torch.int32, device="cuda")
def dev():
    capi.check(lib.btnn_cuda_plan_run_device(plan.h, 0, C.cast(xd.data_ptr(), C.POINTER(C.c_float)), B,
               C.cast(ld.data_ptr(), C.POINTER(C.c_double)), C.cast(bd.data_ptr(), C.POINTER(C.c_int32)), None))
for _ in range(3): dev()
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(10): dev()
torch.cuda.synchronize()
print(f"graph only: {(time.perf_counter()-t)/10*1e3:.2f} ms")
for b in (32, 48, 72, 104, 152):
    for _ in range(2):
        capi.check(lib.btnn_cuda_plan_run_device(plan.h, 0, C.cast(xd.data_ptr(), C.POINTER(C.c_float)), b,
               C.cast(ld.data_ptr(), C.POINTER(C.c_double)), C.cast(bd.data_ptr(), C.POINTER(C.c_int32)), None))
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(5):
        capi.check(lib.btnn_cuda_plan_run_device(plan.h, 0, C.cast(xd.data_ptr(), C.POINTER(C.c_float)), b,
               C.cast(ld.data_ptr(), C.POINTER(C.c_double)), C.cast(bd.data_ptr(), C.POINTER(C.c_int32)), None))
    torch.cuda.synchronize()
    print(f"graph b={b}: {(time.perf_counter()-t)/5*1e3:.3f} ms")
