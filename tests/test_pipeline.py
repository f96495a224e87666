"""Host logic of the layer pipeline (CPU): stage split, per-stage configs and the export/link
plan; the exchange itself over a 2-rank gloo group with stub engines."""
import os

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1604_01946_b200.engine import LadderConfig
from paper_1604_01946_b200.pipeline import link_plan, split_layers, stage_config


def test_split_layers():
    assert split_layers(8, 1) == [(0, 8)]
    assert split_layers(8, 2) == [(0, 4), (4, 4)]
    assert split_layers(8, 8) == [(k, 1) for k in range(8)]
    assert split_layers(7, 3) == [(0, 2), (2, 2), (4, 3)]
    assert sum(c for _, c in split_layers(10, 4)) == 10
    with pytest.raises(ValueError):
        split_layers(2, 3)


def test_stage_config_and_plan():
    cfg = LadderConfig(layers=8, hidden=256, input=100, batch=32, steps=10, seed=1)
    c0, c1 = stage_config(cfg, 0, 2), stage_config(cfg, 1, 2)
    assert (c0.layers, c0.input, c1.layers, c1.input) == (4, 100, 4, 256)
    p = [link_plan(k, 3) for k in range(3)]
    assert [(q.export_fwd, q.export_bwd, q.link_next, q.link_prev) for q in p] == [
        (False, True, True, False), (True, True, True, True), (True, False, False, True)]


class _StubEngine:
    def __init__(self, k):
        self.k, self.links = k, []

    def pp_export(self, d):
        return f"stage{self.k}-dir{d}".encode()

    def pp_link(self, d, peer, w=None):
        self.links.append((d, peer, None if w is None else float(w[0][0])))


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1604_01946_b200 import pipeline as P

    class Stage(P.PipelineStage):
        def __init__(self, k, n):  # no device: a stub engine
            self.k, self.n = k, n
            self.first, self.count = P.split_layers(4, n)[k]
            self.engine = _StubEngine(k)
            self.plan = P.link_plan(k, n)
            self.exports = {}

    class Lp:
        def __init__(self, v):
            self.w = [[v]]

    params = [Lp(float(l)) for l in range(4)]
    st = Stage(rank, world)
    P.link_distributed(st, params)
    out[rank] = st.engine.links
    dist.destroy_process_group()


def test_link_distributed_gloo():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    # stage 0 links forward to stage 1's forward export (the h_t hand-off needs no weights)
    assert out[0] == [(0, b"stage1-dir0", None)]
    # stage 1 links backward to stage 0's backward export
    assert out[1] == [(1, b"stage0-dir1", None)]
