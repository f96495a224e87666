"""GPU box: the layer pipeline at config E (8L h2048 mb256 T100, bf16, automatic schedule =
config E's stepwise CTA-pair forward + persistent CTA-pair backward) on ONE GPU, two stages of
4 layers in this process, run one after the other (forward 0, 1; backward 1, 0). Prints one
JSON line: the single context's pass time, the sum of the stages' pass times, and whether y /
dW / dR / db of every layer are bitwise equal to the single context -- a parity check of the
persistent / stepwise hand-off at full scale, not a multi-GPU speed-up. (Both stages in flight
at once on ONE GPU deadlock at this size: the later stage's step kernels fill the SMs while
spinning on counters the earlier stage can then not get SMs to release -- the flag timeout
ends it with an error. On separate GPUs, the deployment, each stage has its own SMs.)
Usage: python profiles/pp_e_probe.py [layers,hidden,input,batch,steps] [precision] [reps] [seq|conc]
conc: both stages in flight at once on their own streams (no host sync between the stages) --
for shapes whose two stages fit on the GPU together (e.g. C1024: 2 x 2 layers, persistent)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np  # noqa: E402
from parity import make_case  # noqa: E402
from oracle import Dims  # noqa: E402
from paper_1604_01946_b200 import Engine  # noqa: E402
from paper_1604_01946_b200.pipeline import PipelineStage, link_in_process  # noqa: E402

dims = Dims(*[int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "8,2048,2048,256,100").split(",")])
prec = sys.argv[2] if len(sys.argv) > 2 else "bf16"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
mode = sys.argv[4] if len(sys.argv) > 4 else "seq"
n = 2
c, params, x, dy, _, _ = make_case(dims, seed=41, bias=True)
H, I, B, T, L = c.hidden, c.input, c.batch, c.steps, c.layers


def outputs(e, lo, cnt, first):
    y = np.zeros((H, B * T), np.float32, order="F")
    dw = [np.zeros((4 * H, I if l == 0 else H), np.float32, order="F") for l in range(lo, lo + cnt)]
    dr = [np.zeros((4 * H, H), np.float32, order="F") for _ in range(cnt)]
    db = [np.zeros(4 * H, np.float32) for _ in range(cnt)]
    e.read_outputs(y=y, dw=dw, dr=dr, db=db)
    return y, dw, dr, db


def timed(fn):
    fn()  # warm-up (graph capture, repack)
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return 1e3 * float(np.median(ts))


ref = Engine(c, precision=prec, schedule="auto")
desc_ref = ref.describe()
ref.set_params(params)
ref.upload_inputs(x, dy)


def single():
    ref.run_pass(2)
    ref.sync()


ms_single = timed(single)
y_r, dw_r, dr_r, db_r = outputs(ref, 0, L, True)
ref.close()

stages = [PipelineStage(c, k, n, precision=prec, schedule="auto") for k in range(n)]
desc_st = [s.engine.describe() for s in stages]
for s in stages:
    s.set_params(params)
link_in_process(stages, params)
zx = np.zeros((H, B * T), np.float32, order="F")
for k, s in enumerate(stages):
    s.engine.upload_inputs(x if k == 0 else zx, dy if k == n - 1 else zx)


def pipelined():
    for s in stages:
        s.engine.run_pass(3)
        if mode == "seq":
            s.engine.sync()
    for s in reversed(stages):
        s.engine.run_pass(1)
        if mode == "seq":
            s.engine.sync()
    for s in stages:
        s.engine.sync()


ms_pp = timed(pipelined)
same = {"y": True, "dW": True, "dR": True, "db": True}
worst = 0.0
for s in stages:
    y, dw, dr, db = outputs(s.engine, s.first, s.count, s.k == 0)
    if s.k == n - 1:
        same["y"] = bool(np.array_equal(y, y_r))
        worst = max(worst, float(np.abs(y - y_r).max()))
    for j in range(s.count):
        l = s.first + j
        same["dW"] &= bool(np.array_equal(dw[j], dw_r[l]))
        same["dR"] &= bool(np.array_equal(dr[j], dr_r[l]))
        same["db"] &= bool(np.array_equal(db[j], db_r[l]))
        worst = max(worst, float(np.abs(dw[j] - dw_r[l]).max()))
flops = 3 * 2 * 4 * H * (I + H) * B * T * L  # forward + backward_data + weight_update
print(json.dumps({"config": dict(layers=L, hidden=H, input=I, batch=B, steps=T), "precision": prec, "mode": mode,
                  "single_ms": round(ms_single, 2), "pipeline_2stage_ms": round(ms_pp, 2),
                  "single_tflops": round(flops / ms_single / 1e9, 1),
                  "pipeline_tflops": round(flops / ms_pp / 1e9, 1),
                  "bitwise_equal": same, "max_abs_diff": worst,
                  "schedules": {"single": desc_ref, "stages": desc_st}}))
