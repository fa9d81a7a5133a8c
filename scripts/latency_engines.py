"""Timing experiment: small-batch latency of the ResNet-18 plan per bit-GEMM engine
(device-resident input, graph replay, CUDA events)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_16578_b200 import btnn, capi  # noqa: E402
from paper_2006_16578_b200 import model as M  # noqa: E402
from paper_2006_16578_b200 import weights as W  # noqa: E402

m = M.stock_model("resnet18")
ws = W.build_weights(m, W.random_weights(m, 1))
lib = capi.lib()
for name, eng in (("auto", capi.ENGINE_AUTO), ("popc", capi.ENGINE_POPC)):
    capi.set_engine(eng)
    plan = btnn.Plan(m, ws, 128)
    s = torch.cuda.Stream()
    row = []
    for b in (1, 8, 32, 128):
        xd = torch.randn((b, 224, 224, 3), device="cuda")
        ld = torch.empty((b, 1000), dtype=torch.float64, device="cuda")
        bd = torch.empty((b,), dtype=torch.int32, device="cuda")

        def step():
            capi.check(lib.btnn_cuda_plan_run_device(plan.h, 0, C.cast(xd.data_ptr(), C.POINTER(C.c_float)), b,
                                                     C.cast(ld.data_ptr(), C.POINTER(C.c_double)),
                                                     C.cast(bd.data_ptr(), C.POINTER(C.c_int32)),
                                                     C.c_void_p(s.cuda_stream)))
        for _ in range(3):
            step()
        ts = []
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            step()
            e1.record(s)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        row.append(f"b{b}={np.median(ts) * 1e3:.0f}us")
    plan.set_breakdown(True)
    print(name, " ".join(row), flush=True)
capi.set_engine(capi.ENGINE_AUTO)
