"""Print the plan tuner's measured candidates per layer of a stock model (ResNet-18 b512 by
default): python scripts/show_choices.py [model] [batch]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_16578_b200 import btnn as B  # noqa: E402
from paper_2006_16578_b200 import model as M  # noqa: E402
from paper_2006_16578_b200 import weights as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "resnet18"
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 512
m = M.stock_model(name)
ws = W.build_weights(m, W.random_weights(m, 1))
p = B.Plan(m, ws, batch)
for i in range(len(m.layers)):
    n, k, ms = p.layer_choice(i)
    if n:
        print(i, "pick", n[k], " ".join(f"{a}:{b:.4f}" for a, b in zip(n, ms)))
