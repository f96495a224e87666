"""Run N config-B training passes (default 3) through the device-resident path; the target of
ncu captures (profiles/collect.sh). Usage: python profiles/one_pass.py [bf16|fp32] [N]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1604_01946_b200 import Engine, LadderConfig, init_params, make_dy, make_input  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "bf16"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = LadderConfig(layers=4, hidden=512, input=512, batch=64, steps=100, seed=42)
eng = Engine(cfg, precision=prec)
eng.set_params(init_params(cfg))
eng.upload_inputs(make_input(cfg), make_dy(cfg))
for _ in range(n):
    eng.run_pass(2)
eng.sync()
print("ok", eng.describe())
