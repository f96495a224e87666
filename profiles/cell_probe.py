"""GPU box: parity probe of one configuration for any cell kind against the reference engine
(default: the GRU draw of verify.hpp check_oracle_agreement that failed, seed 42 draw 1)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")):
    sys.path.insert(0, p)
import numpy as np  # noqa: E402
import oracle  # noqa: E402
from parity import compare, run_device, run_reference  # noqa: E402
from paper_1604_01946_b200 import engine as E  # noqa: E402

kind, L, H, I, B, T = (int(v) for v in (sys.argv[1].split(",") if len(sys.argv) > 1 else (2, 1, 34, 33, 6, 6)))
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 834950173115998881
prec = sys.argv[3] if len(sys.argv) > 3 else "fp32"
c = E.LadderConfig(layers=L, hidden=H, input=I, batch=B, steps=T, seed=seed, kind=kind, opt_level=3)
params = E.init_params(c)
x, dy = E.make_input(c), E.make_dy(c)
ref = run_reference(oracle.Reference(), c, params, x, dy, None, None)
eng = E.Engine(c, precision=prec)
dev = run_device(eng, params, x, dy, None, None)
print(eng.describe())
for r in sorted(compare(dev, ref, c), key=lambda r: -r[1])[:8]:
    print(f"  {r[0]:8s} normwise {r[1]:.3e} scaled-max {r[2]:.3e}")
d, rr = dev["dw"][0], ref["dw"][0]
bad = np.argwhere(np.abs(d - rr) > 1e-3)
print("dW bad entries", len(bad), "of", d.size, bad[:10].tolist())
