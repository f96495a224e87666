"""Layer pipeline across GPUs ("deep stacks split as a layer pipeline that hands off
h_t per timestep peer-to-peer over NVLink following the paper's wavefront").

Stage k of n owns layers [first_k, first_k + L_k) as an ordinary Engine (input width H for
k > 0). The device side is rw_pp_export / rw_pp_link (include/rnnwave_sm100.h), and the
cross-layer wavefront of the paper (PAPER Listing 4) continues across GPUs step by step:

  forward : stage k's last layer writes each h_t (bf16 operand image, H x B x 2 bytes) into stage
            k+1's layer-input image over NVLink and releases a per-step counter, so stage k+1's
            first layer runs exactly as on one GPU;
  backward: stage k+1 computes W_{first_{k+1}}^T . dG_{first_{k+1}, t} into stage k's last-layer
            ring (its d_above), and stage k copies h_{last_k} into stage k+1's layer input
            (the operand of stage k+1's first-layer dW).

That is the cluster schedule. On the persistent / stepwise schedules (config E: deep stacks at
batch 256, where the cluster schedule does not fit) the hand-off goes through plain operand
planes instead: stage k's last layer stores h_t straight into stage k+1's layer-input planes;
stage k+1's first layer stores its dG_t into stage k's dG-input planes, and stage k's top layer
multiplies them by W_{first_{k+1}}^T (read from stage k+1's parameters over the link) exactly
as the layer below does inside one context. Both directions release system-scope per-step
counters, cumulative over passes.

Exchange order (both the in-process and the torch.distributed variants):
  1. every stage k > 0 exports its forward ring (dir 0), every stage k < n-1 its backward ring
     (dir 1);
  2. stage k < n-1 links forward to stage k+1's export (with W_{first_{k+1}}), stage k > 0 links
     backward to stage k-1's export.
Outputs: y / h_T from the last stage, dx0 from stage 0, each layer's dW/dR/db from its owner.
"""
from __future__ import annotations

import os
from dataclasses import dataclass

# stages in one process (tests) need their streams on distinct hardware queues; effective only
# if set before the process initialises CUDA
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

from .engine import Engine, LadderConfig


def split_layers(layers: int, n: int) -> list[tuple[int, int]]:
    """Contiguous (first, count) per stage, earlier stages taking the remainder (SURVEY §8e:
    stage k owns layers [k L / n, (k + 1) L / n))."""
    if n < 1 or n > layers:
        raise ValueError(f"pipeline: cannot split {layers} layers over {n} stages")
    return [(k * layers // n, (k + 1) * layers // n - k * layers // n) for k in range(n)]


def stage_config(cfg: LadderConfig, k: int, n: int) -> LadderConfig:
    first, count = split_layers(cfg.layers, n)[k]
    c = LadderConfig(**cfg.__dict__)
    c.layers = count
    c.input = cfg.input if k == 0 else cfg.hidden
    return c


@dataclass
class LinkPlan:
    """Which exports a stage makes and which links it needs (host logic, unit-tested on CPU)."""
    export_fwd: bool
    export_bwd: bool
    link_next: bool
    link_prev: bool


def link_plan(k: int, n: int) -> LinkPlan:
    return LinkPlan(export_fwd=k > 0, export_bwd=k < n - 1, link_next=k < n - 1, link_prev=k > 0)


class PipelineStage:
    """One stage: an Engine over the stage's layers plus the boundary links."""

    def __init__(self, cfg: LadderConfig, k: int, n: int, device: int = 0, precision: str = "bf16",
                 schedule: str = "cluster"):
        """schedule: "cluster" (boundary groups), or "persistent" / "stepwise" / "auto" resolving to
        those two (config E's shape): every stage of one pipeline must use the same family, and
        stages below the last need >= 2 layers there (the top layer's backward takes W_next)."""
        self.k, self.n = k, n
        self.first, self.count = split_layers(cfg.layers, n)[k]
        self.full_cfg = cfg
        self.engine = Engine(stage_config(cfg, k, n), precision=precision, schedule=schedule, device=device)
        self.plan = link_plan(k, n)
        self.exports: dict[int, bytes] = {}

    def set_params(self, params) -> None:
        """params: the full model's LayerParams; the stage takes its own slice (the forward
        hand-off sends h_t, so no neighbour's weights are needed)."""
        self.engine.set_params(params[self.first:self.first + self.count])

    def export(self) -> dict[int, bytes]:
        if self.plan.export_fwd:
            self.exports[0] = self.engine.pp_export(0)
        if self.plan.export_bwd:
            self.exports[1] = self.engine.pp_export(1)
        return self.exports

    def link(self, next_exports: dict[int, bytes] | None, prev_exports: dict[int, bytes] | None,
             params) -> None:
        if self.plan.link_next:
            self.engine.pp_link(0, next_exports[0], None)
        if self.plan.link_prev:
            self.engine.pp_link(1, prev_exports[1])


def link_in_process(stages: list[PipelineStage], params) -> None:
    """All stages in one process (tests; several stages may share a GPU)."""
    ex = [s.export() for s in stages]
    for k, s in enumerate(stages):
        s.link(ex[k + 1] if k + 1 < len(stages) else None, ex[k - 1] if k > 0 else None, params)


def link_distributed(stage: PipelineStage, params, group=None) -> None:
    """One stage per rank (torch.distributed, any backend): all-gather the exports (bytes with
    CUDA IPC handles), then link to the neighbours."""
    import torch.distributed as dist
    mine = stage.export()
    allx = [None] * stage.n
    dist.all_gather_object(allx, mine, group=group)
    k = stage.k
    stage.link(allx[k + 1] if k + 1 < stage.n else None, allx[k - 1] if k > 0 else None, params)
