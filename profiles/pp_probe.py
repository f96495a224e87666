"""GPU box: the layer-pipeline equivalence case of tests/test_pipeline_gpu.py with max |diff| per
output instead of a bitwise assert (debug aid)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np  # noqa: E402
from parity import make_case  # noqa: E402
from oracle import Dims  # noqa: E402
from paper_1604_01946_b200 import Engine  # noqa: E402
from paper_1604_01946_b200.pipeline import PipelineStage, link_in_process  # noqa: E402

dims = Dims(*[int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "4,128,96,32,10").split(",")])
n = int(sys.argv[2]) if len(sys.argv) > 2 else 2
c, params, x, dy, _, _ = make_case(dims, seed=23, bias=True)
H, I, B, T, L = c.hidden, c.input, c.batch, c.steps, c.layers
ref = Engine(c, precision="bf16", schedule="cluster")
ref.set_params(params)
ref.upload_inputs(x, dy)
ref.run_pass(2)
ref.sync()
y_r = np.zeros((H, B * T), np.float32, order="F")
dx_r = np.zeros((I, B * T), np.float32, order="F")
dw_r = [np.zeros((4 * H, I if l == 0 else H), np.float32, order="F") for l in range(L)]
dr_r = [np.zeros((4 * H, H), np.float32, order="F") for _ in range(L)]
db_r = [np.zeros(4 * H, np.float32) for _ in range(L)]
ref.read_outputs(y_r, dx_r, dw_r, dr_r, db_r)
os.environ["RW_PP_RING"] = str(T)
stages = [PipelineStage(c, k, n) for k in range(n)]
for s in stages:
    s.set_params(params)
link_in_process(stages, params)
zx = np.zeros((H, B * T), np.float32, order="F")
for k, s in enumerate(stages):
    s.engine.upload_inputs(x if k == 0 else zx, dy if k == n - 1 else zx)
for s in stages:
    s.engine.run_pass(3)
    s.engine.sync()
for s in reversed(stages):
    s.engine.run_pass(1)
    s.engine.sync()
import ctypes as C  # noqa: E402
F = C.POINTER(C.c_float)


def tape(e, which, l, rows, cols):
    out = np.zeros((rows, cols), np.float32, order="F")
    assert e._L.rw_get_tape(e._ctx, which, l, out.ctypes.data_as(F)) == 0
    return out


names = {1: ("h", H, B * (T + 1)), 2: ("c", H, B * (T + 1)), 3: ("gates", 4 * H, B * T), 4: ("tanhc", H, B * T),
         5: ("dgw", 4 * H, B * T)}
for s in stages:
    for j in range(s.count):
        l = s.first + j
        for w, (nm, r, cc) in names.items():
            a, b = tape(s.engine, w, j, r, cc), tape(ref, w, l, r, cc)
            d = np.abs(a - b)
            print(f"  tape {nm} layer {l}: max diff {d.max():.3e}", "first bad col", (np.argwhere(d > 0)[:1, 1] if d.max() else ""))
for s in stages:
    lo, cnt = s.first, s.count
    y = np.zeros((H, B * T), np.float32, order="F")
    dx = np.zeros((I if s.k == 0 else H, B * T), np.float32, order="F")
    dw = [np.zeros_like(dw_r[l]) for l in range(lo, lo + cnt)]
    dr = [np.zeros_like(dr_r[l]) for l in range(lo, lo + cnt)]
    db = [np.zeros_like(db_r[l]) for l in range(lo, lo + cnt)]
    s.engine.read_outputs(y, dx, dw, dr, db)
    print("stage", s.k, s.engine.describe())
    for j in range(cnt):
        l = lo + j
        print(f"  layer {l}: dW {np.abs(dw[j]-dw_r[l]).max():.3e} (ref max {np.abs(dw_r[l]).max():.3e})"
              f" dR {np.abs(dr[j]-dr_r[l]).max():.3e} db {np.abs(db[j]-db_r[l]).max():.3e}")
        bad = np.argwhere(dw[j] != dw_r[l])
        if len(bad):
            print("    dW bad entries", len(bad), "rows", sorted(set(bad[:, 0].tolist()))[:12], "cols",
                  sorted(set(bad[:, 1].tolist()))[:12])
    if s.k == n - 1:
        print("  y", np.abs(y - y_r).max())
    if s.k == 0:
        print("  dx0", np.abs(dx - dx_r).max())
