"""GPU box: config-B parity of the device (fp32 / bf16) against the reference CPU engine, worst
tensors printed -- a quick probe for precision experiments (env knobs such as RW_CL_DEBUG)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
from parity import compare, make_case, run_device, run_reference  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "fp32"
dims = oracle.Dims(*(int(v) for v in (sys.argv[2].split(",") if len(sys.argv) > 2 else (4, 512, 512, 64, 100))))
from paper_1604_01946_b200 import Engine  # noqa: E402
c, params, x, dy, h0, c0 = make_case(dims, seed=42)
ref = run_reference(oracle.Reference(), c, params, x, dy, h0, c0)
eng = Engine(c, precision=prec)
rows = compare(run_device(eng, params, x, dy, h0, c0), ref, c)
rows.sort(key=lambda r: -max(r[1], r[2]))
print(prec, dims, eng.describe()["operands"], os.environ.get("RW_CL_DEBUG", ""))
for r in rows[:6]:
    print(f"  {r[0]:8s} normwise {r[1]:.3e} scaled-max {r[2]:.3e}")
