import os, sys
import numpy as np
sys.path.insert(0, os.getcwd())
from paper_2006_16578_b200 import btnn, capi
from paper_2006_16578_b200 import model as M
from paper_2006_16578_b200 import weights as W
m = M.stock_model("resnet18")
ws = W.build_weights(m, W.random_weights(m, 1))
plan = btnn.Plan(m, ws, 8)
x = np.random.default_rng(1).standard_normal((8, 224, 224, 3), dtype=np.float32)
plan.run(x); plan.set_breakdown(True)
for _ in range(3): plan.run(x)
print([round(v * 1000) for v in plan.layer_ms()], round(sum(plan.layer_ms()) * 1000))
