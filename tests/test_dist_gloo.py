"""CPU, world_size 2 over gloo: the data-parallel partition of SURVEY §8e.

Each rank runs the (CPU) reference-path restatement on its minibatch shard of the same
sequences; the weight gradients are summed with torch.distributed (the host-side twin of the
library's NCCL all-reduce). The sum must equal the full-batch gradients (up to fp32
summation order), and the per-rank outputs must reassemble the full-batch y / dx0 exactly
(sequences are independent, so those are bitwise).
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from paper_1604_01946_b200.parallel import (  # noqa: E402
    allreduce_gradients, shard_columns, shard_range, unshard_columns)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_range_balanced():
    assert [shard_range(7, r, 3) for r in range(3)] == [(0, 3), (3, 5), (5, 7)]
    assert [shard_range(64, r, 8) for r in range(8)][-1] == (56, 64)
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)


def test_shard_unshard_roundtrip():
    m = np.asfortranarray(np.arange(3 * 5 * 4, dtype=np.float32).reshape(3, 20))
    parts = [shard_columns(m, 5, 4, r, 2) for r in range(2)]
    assert parts[0].shape == (3, 12) and parts[1].shape == (3, 8)
    assert np.array_equal(unshard_columns(parts, 5, 4), m)


def _worker(rank, world, port, result_q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "oracle"))
    import oracle
    from paper_1604_01946_b200.engine import Gradients
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    o = oracle.Restatement()
    full = oracle.Dims(2, 12, 10, 6, 5)
    w, r = o.init_params(full, 9)
    b = [np.zeros(48, np.float32) for _ in range(2)]
    x = o.make_input(full, 9)
    dy = o.make_dy(full, 9)
    b0, b1 = shard_range(full.batch, rank, world)
    mine = oracle.Dims(full.layers, full.hidden, full.input, b1 - b0, full.steps)
    xs = shard_columns(x, full.batch, full.steps, rank, world)
    dys = shard_columns(dy, full.batch, full.steps, rank, world)
    out = o.run(mine, w, r, b, xs, None, None, dys)
    g = Gradients(out["dw"], out["dr"], out["db"], out["dx0"])
    allreduce_gradients(g)
    result_q.put((rank, out["y"], out["dx0"], g.dw, g.dr, g.db))
    dist.barrier()
    dist.destroy_process_group()


def test_data_parallel_gradients_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    import oracle
    o = oracle.Restatement()
    full = oracle.Dims(2, 12, 10, 6, 5)
    w, r = o.init_params(full, 9)
    b = [np.zeros(48, np.float32) for _ in range(2)]
    ref = o.run(full, w, r, b, o.make_input(full, 9), None, None, o.make_dy(full, 9))
    # independent sequences: the shards reassemble the full-batch outputs bitwise
    assert np.array_equal(unshard_columns([t[1] for t in res], 6, 5), ref["y"])
    assert np.array_equal(unshard_columns([t[2] for t in res], 6, 5), ref["dx0"])
    # reduced gradients match the full batch up to summation order, and agree across ranks
    for l in range(2):
        for k, idx in (("dw", 3), ("dr", 4), ("db", 5)):
            got = res[0][idx][l]
            assert np.array_equal(got, res[1][idx][l])
            err = np.linalg.norm(got - ref[k][l]) / np.linalg.norm(ref[k][l])
            assert err < 1e-6, (k, l, err)


def test_bucket_plan_top_layer_first():
    from paper_1604_01946_b200.parallel import bucket_plan
    plan = bucket_plan(3, 4, 5)
    assert [l for l, _ in plan] == [2, 1, 0]
    assert plan[-1][1] == 16 * 5 + 16 * 4 + 16 and plan[0][1] == 16 * 4 * 2 + 16


def _bucket_worker(rank, world, port, result_q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    from paper_1604_01946_b200.engine import Gradients
    from paper_1604_01946_b200.parallel import allreduce_gradients_bucketed
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(100 + rank)
    L, H, I = 3, 8, 6
    mk = lambda r, c: np.asfortranarray(rng.standard_normal((r, c)).astype(np.float32))  # noqa: E731
    g = Gradients([mk(4 * H, I if l == 0 else H) for l in range(L)], [mk(4 * H, H) for _ in range(L)],
                  [rng.standard_normal(4 * H).astype(np.float32) for _ in range(L)])
    mine = Gradients([a.copy(order="F") for a in g.dw], [a.copy(order="F") for a in g.dr], [a.copy() for a in g.db])
    allreduce_gradients_bucketed(g)
    result_q.put((rank, mine, g))
    dist.barrier()
    dist.destroy_process_group()


def test_bucketed_overlapped_allreduce_gloo():
    """World size 2 over gloo: the overlapped per-layer buckets (all in flight at once, top layer
    first, rw_comm_overlap's order) sum to exactly the per-tensor all-reduce."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bucket_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    (_, a, ga), (_, b, gb) = res
    for name in ("dw", "dr", "db"):
        for la, lb, ra, rb in zip(getattr(a, name), getattr(b, name), getattr(ga, name), getattr(gb, name)):
            want = (la.astype(np.float32) + lb.astype(np.float32))
            assert np.array_equal(ra, want) and np.array_equal(rb, want)
