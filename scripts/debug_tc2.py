"""Localize a TC-vs-POPC mismatch at kernel level (debug aid)."""
import sys, os
sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.abspath(__file__)))]
import numpy as np
from paper_2006_16578_b200 import btnn as B, capi, model as M, weights as W

rng = np.random.default_rng(0)
def both(fn):
    out = []
    for eng in (capi.ENGINE_POPC, capi.ENGINE_TC):
        capi.set_engine(eng)
        out.append(fn())
    capi.set_engine(capi.ENGINE_AUTO)
    return out

for (hw, n, c, o, k, s, p) in [(4, 3, 256, 256, 3, 1, 1), (4, 3, 256, 128, 3, 1, 1), (4, 3, 128, 256, 3, 1, 1),
                               (8, 3, 256, 256, 3, 1, 1), (4, 8, 256, 256, 3, 1, 1), (4, 3, 512, 512, 3, 1, 1),
                               (8, 3, 128, 256, 3, 2, 1), (14, 2, 256, 256, 3, 1, 1), (4, 3, 384, 64, 3, 1, 1),
                               (2, 3, 256, 256, 3, 1, 1), (4, 1, 256, 256, 3, 1, 1), (4, 3, 256, 256, 1, 1, 0)]:
    x = rng.standard_normal((n, hw, hw, c), dtype=np.float32)
    wt = rng.standard_normal(k * k * o * c, dtype=np.float32)
    aw, fw = W.pack_nhwc(x), W.pack_filter(wt, k, k, o, c)
    ad, fd, g = capi.ActDesc(hw, hw, n, c, 0, 8, 128), capi.FilterDesc(k, k, o, c, 0, 8, 128), capi.ConvGeom(k, k, s, p)
    a, b = both(lambda: B.bconv_pm1(ad, aw, fd, fw, g))
    bad = np.nonzero(a != b)[0]
    P = (hw + 2 * p - k) // s + 1
    msg = ""
    if bad.size:
        i = bad[0]
        oo = i % o; nn = (i // o) % n; site = i // (o * n)
        msg = f" first bad idx {i} (site {site} n {nn} o {oo}) popc {a[i]} tc {b[i]}; bad count {bad.size}/{a.size}; bad o set {sorted(set((bad % o).tolist()))[:8]} sites {sorted(set((bad // (o*n)).tolist()))[:10]}"
    print(f"pm1 hw{hw} n{n} c{c} o{o} k{k} s{s}: {'OK' if not bad.size else 'MISMATCH'}{msg}", flush=True)
    gamma, beta = rng.standard_normal(o), rng.standard_normal(o)
    mean, var = rng.standard_normal(o) * 5, rng.uniform(0.25, 2, o)
    rin = rng.standard_normal(P * P * n * o)
    (b1, r1), (b2, r2) = both(lambda: B.bconv_fused(ad, aw, fd, fw, g, bn=(gamma, beta, mean, var), residual_in=rin, want_residual_out=True))
    print(f"   fused bits {'OK' if np.array_equal(b1, b2) else 'MISMATCH'} rout {'OK' if np.array_equal(r1.view(np.uint64), r2.view(np.uint64)) else 'MISMATCH'}", flush=True)
