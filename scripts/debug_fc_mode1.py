"""Debug: diff pattern of the stride-1 tensor-core first conv vs the C oracle."""
import ctypes as C, sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__)))); sys.path.insert(0, "tests")
from fixtures import load
from oracle_lib import oracle, ptr
from paper_2006_16578_b200 import btnn as B, capi
d = load("first_conv_pool")
for case in [tuple(int(v) for v in d["f3_case"]), (1, 8, 8, 3, 32, 3, 1, 1), (1, 16, 16, 3, 32, 3, 1, 1)]:
    n, h, w, c, o, k, s, pd = case
    rng = np.random.default_rng(1)
    x = d["f3_x"].reshape(n, h, w, c) if case == tuple(int(v) for v in d["f3_case"]) else rng.standard_normal((n, h, w, c)).astype(np.float32)
    wt = d["f3_w"] if case == tuple(int(v) for v in d["f3_case"]) else np.where(rng.standard_normal(o * k * k * c) >= 0, 1.0, -1.0).astype(np.float32)
    geo = capi.ConvGeom(k, k, s, pd)
    capi.set_engine(capi.ENGINE_TC)
    got = B.first_conv_bwn(x, wt, k, k, o, geo)
    print(case, capi.last_tc_launch())
    P = Q = (h + 2 * pd - k) // s + 1
    want = np.zeros(P * Q * n * o)
    oracle().bo_first_conv_bwn(ptr(np.ascontiguousarray(x), C.c_float), n, h, w, c, ptr(np.ascontiguousarray(wt), C.c_float), k, k, o, C.byref(geo), ptr(want, C.c_double))
    dd = (got - want).reshape(P, Q, n, o)
    bad = np.argwhere(dd != 0)
    print(" bad", len(bad), "of", dd.size)
    for b in bad[:12]:
        print("  pqno", b.tolist(), dd[tuple(b)], want.reshape(P, Q, n, o)[tuple(b)])
    print(" bad (p,q) sites:", sorted(set((int(b[0]), int(b[1])) for b in bad))[:40])
