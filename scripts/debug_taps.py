"""Compare every residual tap between engines for ResNet-18 structures (debug aid)."""
import sys, os
sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.abspath(__file__)))]
import numpy as np
from paper_2006_16578_b200 import btnn as B, capi, model as M, weights as W

for hw, batch in ((64, 3), (32, 2)):
    m = M.stock_model("resnet18", hw, hw)
    ws = W.build_weights(m, W.random_weights(m, 5))
    x = np.random.default_rng(6).standard_normal((batch, hw, hw, 3), dtype=np.float32)
    taps = {}
    for eng in (capi.ENGINE_POPC, capi.ENGINE_TC):
        capi.set_engine(eng)
        p = B.Plan(m, ws, batch)
        p.run(x)
        taps[eng] = {i: p.read_tap(i, batch) for i, l in enumerate(m.layers) if l.residual_out}
        p.close()
    for i in taps[1]:
        a, b = taps[1][i], taps[2][i]
        l = m.layers[i]
        bad = np.nonzero(a.view(np.uint64) != b.view(np.uint64))[0]
        info = ""
        if bad.size:
            O, N = l.out_channels, batch
            info = f" bad {bad.size}/{a.size}; o {sorted(set((bad % O).tolist()))[:6]}..; n {sorted(set(((bad // O) % N).tolist()))}; sites {sorted(set((bad // (O*N)).tolist()))[:8]}; e.g. popc {a[bad[0]]} tc {b[bad[0]]}"
        print(f"hw{hw} tap layer {i} ({l.out_h}x{l.out_w}x{l.out_channels}, rin={l.residual_in}): {'OK' if not bad.size else 'MISMATCH'}{info}", flush=True)
