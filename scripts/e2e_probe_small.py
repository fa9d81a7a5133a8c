"""Timing experiment: per-call cost of plan_run for a small-input model (MNIST-MLP b1024)."""
import ctypes as C, os, sys, time
import numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2006_16578_b200 import btnn, capi
from paper_2006_16578_b200 import model as M, weights as W
name = sys.argv[1] if len(sys.argv) > 1 else "mnist-mlp"; B = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
m = M.stock_model(name); ws = W.build_weights(m, W.random_weights(m, 1))
plan = btnn.Plan(m, ws, B); lib = capi.lib()
xh = torch.randn((B, m.in_h, m.in_w, m.in_c), dtype=torch.float32).pin_memory()
lh = torch.empty((B, m.classes), dtype=torch.float64).pin_memory(); bh = torch.empty((B,), dtype=torch.int32).pin_memory()
xp, lp, bp = C.cast(xh.data_ptr(), C.POINTER(C.c_float)), C.cast(lh.data_ptr(), C.POINTER(C.c_double)), C.cast(bh.data_ptr(), C.POINTER(C.c_int32))
def tm(f, n=50):
    for _ in range(5): f()
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(n): f()
    torch.cuda.synchronize(); return (time.perf_counter() - t) / n * 1e6
print("plan_run us", tm(lambda: lib.btnn_cuda_plan_run(plan.h, xp, B, lp, bp)))
dx = torch.empty((B, m.in_h, m.in_w, m.in_c), device="cuda"); dl = torch.empty((B, m.classes), dtype=torch.float64, device="cuda"); db = torch.empty((B,), dtype=torch.int32, device="cuda")
s = torch.cuda.current_stream()
def dev(): plan.run_device(dx.data_ptr(), B, dl.data_ptr(), db.data_ptr(), s.cuda_stream); s.synchronize()
print("run_device+sync us", tm(dev))
def h2d(): dx.copy_(xh, non_blocking=True); s.synchronize()
print("h2d+sync us", tm(h2d))
def d2h(): lh.copy_(dl, non_blocking=True); bh.copy_(db, non_blocking=True); s.synchronize()
print("d2h+sync us", tm(d2h))
def ctypes_only(): lib.btnn_cuda_device_count(C.byref(C.c_int()))
print("ctypes call us", tm(ctypes_only))
