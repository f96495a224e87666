import os, sys, time
sys.path.insert(0, os.getcwd())
from paper_1604_01946_b200 import Engine, LadderConfig, init_params, make_dy, make_input
import bench
c = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "B"]
cfg = LadderConfig(**c, seed=42)
eng = Engine(cfg, precision="bf16")
print(eng.describe(), flush=True)
eng.set_params(init_params(cfg)); eng.upload_inputs(make_input(cfg), make_dy(cfg))
for i in range(3):
    t0 = time.time(); eng.run_pass(2); eng.sync(); print("pass", i, time.time() - t0, flush=True)
