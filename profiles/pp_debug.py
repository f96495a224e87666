"""Layer-pipeline debugging on one GPU: two pipeline stages in one process run one after the
other (RW_PP_RING = T), outputs compared with a single context. Paths are this container's."""
import os, sys, time
import os; os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests"); sys.path.insert(0, "/root/repo/oracle")
import numpy as np
from parity import make_case
from oracle import Dims
from paper_1604_01946_b200.pipeline import PipelineStage, link_in_process
c, params, x, dy, _, _ = make_case(Dims(4, 128, 96, 32, int(os.environ.get("TT", "10"))), seed=23, bias=True)
H, B, T = c.hidden, c.batch, c.steps
order = os.environ.get("ORDER", "01")
stages = [PipelineStage(c, k, 2) for k in range(2)]
for s in stages: s.set_params(params)
link_in_process(stages, params)
zx = np.zeros((H, B * T), np.float32, order="F")
stages[0].engine.upload_inputs(x, zx)
stages[1].engine.upload_inputs(zx, dy)
t0 = time.time()
for ps in os.environ.get("PASS", "2").split(","):
    for k in order:
        stages[int(k)].engine.run_pass(int(ps))
    print("enqueued pass", ps, time.time() - t0, flush=True)
    for k in order:
        try:
            stages[int(k)].engine.sync(); print("stage", k, "ok", time.time() - t0, flush=True)
        except Exception as e:
            print("stage", k, "ERR", e, time.time() - t0, flush=True)

import ctypes as C
for k, st in enumerate(stages):
    out = (C.c_longlong * 16)()
    st.engine._L.rw_pp_debug(st.engine._ctx, out)
    print("stage", k, list(out), flush=True)
