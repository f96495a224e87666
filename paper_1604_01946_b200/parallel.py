"""Multi-GPU partitioning of the LSTM path, host-side logic.

Data parallel: sequences are independent, so the minibatch B is split across ranks; each
rank runs the full forward/backward on its shard and the weight gradients are summed
(NCCL all-reduce inside librnnwave_sm100.so on GPUs; torch.distributed for host arrays, which
is what the gloo CPU tests exercise). The time-major layout puts batch element b of step t
in column t*B + b, so a shard is a strided column gather.
"""
from __future__ import annotations

import numpy as np


def shard_range(batch: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced batch range [b0, b1) of `rank` (the first batch % world ranks
    get one extra sequence)."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} out of range for world size {world}")
    base, extra = divmod(batch, world)
    b0 = rank * base + min(rank, extra)
    return b0, b0 + base + (1 if rank < extra else 0)


def shard_columns(m: np.ndarray, batch: int, steps: int, rank: int, world: int) -> np.ndarray:
    """Columns of a time-major (rows x batch*steps) matrix that belong to `rank`."""
    b0, b1 = shard_range(batch, rank, world)
    cols = (np.arange(steps)[:, None] * batch + np.arange(b0, b1)[None, :]).ravel()
    return np.asfortranarray(m[:, cols])


def unshard_columns(parts: list[np.ndarray], batch: int, steps: int) -> np.ndarray:
    """Inverse of shard_columns over all ranks (rank order)."""
    world = len(parts)
    rows = parts[0].shape[0]
    out = np.zeros((rows, batch * steps), np.float32, order="F")
    for r, p in enumerate(parts):
        b0, b1 = shard_range(batch, r, world)
        cols = (np.arange(steps)[:, None] * batch + np.arange(b0, b1)[None, :]).ravel()
        out[:, cols] = p
    return out


def allreduce_gradients(grads, group=None) -> None:
    """Sum dW/dR/db over the process group in place (host arrays, torch.distributed)."""
    import torch
    import torch.distributed as dist
    for lst in (grads.dw, grads.dr, grads.db):
        for i, a in enumerate(lst):
            t = torch.from_numpy(np.array(a, dtype=np.float32).ravel(order="F"))
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
            lst[i] = np.asfortranarray(t.numpy().reshape(a.shape, order="F"))


def bucket_plan(layers: int, hidden: int, inp: int) -> list[tuple[int, int]]:
    """The overlapped data-parallel all-reduce's buckets (rw_comm_overlap, runtime.cu): one per
    layer, top layer first (its weight-gradient GEMMs finish first), as (layer, fp32 values):
    dW_l (4H x I_l) + dR_l (4H x H) + db_l (4H)."""
    G = 4 * hidden
    return [(l, G * (inp if l == 0 else hidden) + G * hidden + G) for l in range(layers - 1, -1, -1)]


def allreduce_gradients_bucketed(grads, group=None) -> None:
    """Host twin of the overlapped device all-reduce: each layer's bucket (dW, dR, db) is summed
    asynchronously in bucket_plan order, all in flight at once, then waited for; the result
    equals allreduce_gradients bit for bit (same per-tensor sums)."""
    import torch
    import torch.distributed as dist
    L = len(grads.dw)
    plan = bucket_plan(L, grads.dr[0].shape[1], grads.dw[0].shape[1])
    pending = []
    for l, _ in plan:
        for lst in (grads.dw, grads.dr, grads.db):
            a = lst[l]
            t = torch.from_numpy(np.array(a, dtype=np.float32).ravel(order="F"))
            pending.append((lst, l, a.shape, t, dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group, async_op=True)))
    for lst, l, shape, t, work in pending:
        work.wait()
        lst[l] = np.asfortranarray(t.numpy().reshape(shape, order="F"))
