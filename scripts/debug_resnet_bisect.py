"""Bisect a TC-vs-POPC mismatch over prefixes of the ResNet-18 structure (debug aid)."""
import sys, os
sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.abspath(__file__)))]
import numpy as np
from paper_2006_16578_b200 import btnn as B, capi, model as M, weights as W

toks = ["64C7/4"] + ["64C3"] * 4 + ["128C3/2"] + ["128C3"] * 3 + ["256C3/2"] + ["256C3"] * 3 + ["512C3/2"] + ["512C3"] * 3
hw = int(sys.argv[1]) if len(sys.argv) > 1 else 64
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 3
for k in range(2, len(toks) + 1):
    sc = [(a, a + 2) for a in range(0, 16, 2) if a + 2 < k]
    m = M.make_model("r%d" % k, "-".join(toks[:k]), hw, hw, 3, 10, sc)
    ws = W.build_weights(m, W.random_weights(m, 5))
    x = np.random.default_rng(6).standard_normal((batch, hw, hw, 3), dtype=np.float32)
    out = {}
    for eng in (capi.ENGINE_POPC, capi.ENGINE_TC):
        capi.set_engine(eng)
        p = B.Plan(m, ws, batch)
        out[eng] = p.run(x)
        p.close()
    same = np.array_equal(out[1][0].view(np.uint64), out[2][0].view(np.uint64))
    print(f"depth {k} ({toks[k-1]}, shortcuts {sc[-1:] if sc else []}): {'OK' if same else 'MISMATCH'}", flush=True)
    if not same:
        break
