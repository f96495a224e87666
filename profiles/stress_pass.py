"""Hang / race stress: run `n` training passes of a config back to back (CUDA graphs) and check
the error flag; run under an outer `timeout`. Usage: python profiles/stress_pass.py B 2000"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1604_01946_b200 import Engine, LadderConfig, init_params, make_dy, make_input  # noqa: E402

c = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "B"]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
cfg = LadderConfig(**c, seed=42)
eng = Engine(cfg, precision="bf16")
print(eng.describe(), flush=True)
eng.set_params(init_params(cfg))
eng.upload_inputs(make_input(cfg), make_dy(cfg))
t0 = time.time()
for i in range(n):
    eng.run_pass(2)
    if i % int(os.environ.get("STRESS_EVERY", "200")) == int(os.environ.get("STRESS_EVERY", "200")) - 1:
        eng.sync()
        print(f"{i + 1} passes, {time.time() - t0:.1f} s", flush=True)
eng.sync()
print("ok", n, "passes", flush=True)
