"""GPU box: run each GPU-ladder rung once on a small LSTM and report failures (debug aid)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
from paper_1604_01946_b200 import Engine, LadderConfig, init_params, make_dy, make_input  # noqa: E402

dims = [int(v) for v in (sys.argv[1].split(",") if len(sys.argv) > 1 else (2, 64, 64, 16, 5))]
prec = sys.argv[2] if len(sys.argv) > 2 else "fp32"
levels = [int(v) for v in sys.argv[3].split(",")] if len(sys.argv) > 3 else [0, 1, 2, 3, 4]
cfg = LadderConfig(layers=dims[0], hidden=dims[1], input=dims[2], batch=dims[3], steps=dims[4], seed=5)
e = Engine(cfg, precision=prec, schedule="stepwise")
p = init_params(cfg)
e.set_params(p)
e.upload_inputs(make_input(cfg), make_dy(cfg))
ref = e.forward(p, make_input(cfg), False).y
for lv in levels:
    e.ladder_pass(lv)
    e.sync()
    y = np.zeros_like(ref)
    e.read_outputs(y=y)
    print(lv, "normwise vs forward", float(np.linalg.norm(y - ref) / np.linalg.norm(ref)), flush=True)
