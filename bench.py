#!/usr/bin/env python3
"""bench.py -- LSTM fwd+bwd TFLOPS on B200 (BASELINE.json metric), one JSON line on rank 0.

Workload (BASELINE.json configs[1], the paper's headline case): 4-layer LSTM, h=512, mb=64,
T=100, forward (training) + backward_data + weight_update per step, synthetic SplitMix64
inputs/weights exactly like the reference generators (seed 42). FLOPs follow the
reference convention (cells.hpp:65-68, bench.hpp:55-62, 210-213): GEMM multiply-adds only,
2*4*H*(I+H)*B per cell x L*T x 3 (fwd 1 + bwd 2).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--precision fp32|bf16] [--config B]

The headline line is the fp32-parity mode (the reference computes in fp32; our split-operand
tensor-core products meet its 1e-5 contract); bf16 is reported as a secondary key. Every timed
step re-runs the K7 weight repack (the parameters are marked updated, as after an optimizer
step), like the reference's per-pass pretranspose.
  python bench.py --impl reference ...   (the reference CPU engine, oracle/_ref, host cores)

Under torchrun (N > 1) every rank runs its own independent minibatch of the same shape
(data parallel, weak scaling) and the weight gradients are summed over ranks with NCCL
(all-reduce of dW/dR/db); timing is the max over ranks of CUDA-event device time.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIG_B = dict(layers=4, hidden=512, input=512, batch=64, steps=100)
# BASELINE.json configs by SURVEY §8(d) letter; only B is the bench line, the others are sweep /
# parity cases (--config for the profiles/ sweep tables).
CONFIGS = {
    "A": dict(layers=1, hidden=512, input=512, batch=64, steps=100),
    "B": CONFIG_B,
    "C128": dict(layers=4, hidden=128, input=128, batch=64, steps=100),
    "C256": dict(layers=4, hidden=256, input=256, batch=64, steps=100),
    "C1024": dict(layers=4, hidden=1024, input=1024, batch=64, steps=100),
    "C2048": dict(layers=4, hidden=2048, input=2048, batch=64, steps=100),
    "D1": dict(layers=1, hidden=1024, input=1024, batch=16, steps=200),
    "D4": dict(layers=4, hidden=1024, input=1024, batch=16, steps=200),
    "E": dict(layers=8, hidden=2048, input=2048, batch=256, steps=100),
}
METRIC = "LSTM fwd+bwd TFLOPS (h=512, mb=64, 4 layers, T=100) and % of B200 TC peak"


def pass_flops(c: dict, mult: int = 3) -> int:
    f = 0
    for l in range(c["layers"]):
        il = c["input"] if l == 0 else c["hidden"]
        f += 2 * 4 * c["hidden"] * (il + c["hidden"]) * c["batch"] * c["steps"]
    return f * mult


# weights re-read every step (the streaming schedules) still come from L2 (126 MB) when they
# fit in it; the cluster / persistent-resident schedules keep them in shared memory
L2_WEIGHT_BYTES = 100 * 1024 * 1024


def recurrent_bytes(c: dict, fwd: bool, planes: int = 1) -> int:
    """Algorithmic HBM bytes of one recurrent launch: the 16-bit weight
    operand planes (bf16: one; fp32-parity: hi + lo) -- once per pass when they fit on chip or
    in L2, else once per step (config E: 512 MB of bf16 [W|R] per wavefront step, far beyond
    smem + L2) -- plus the fp32 tapes each cell must write (forward: gates x4, c, h, tanh c + the
    16-bit h operand planes) or read and write (backward: gates x4, tanh c, c read; dG fp32 x4 +
    the 16-bit dG operand planes x4 written)."""
    L, H, I, B, T = c["layers"], c["hidden"], c["input"], c["batch"], c["steps"]
    if fwd:
        w = sum(4 * H * ((I if l == 0 else H) + H) * 2 for l in range(L))
        steps, cell = T, 4 * (4 + 3) + 2 * planes
    else:
        w = sum(4 * H * (H + (H if l < L - 1 else 0)) * 2 for l in range(L))
        steps, cell = T + 1, 4 * (4 + 2) + 4 * 4 + 4 * 2 * planes
    w *= planes
    wt = w if w <= L2_WEIGHT_BYTES else w * steps
    return wt + L * T * H * B * cell


def ncu_traffic(kernel_prefix: str, config: str, precision: str = "bf16"):
    """DRAM bytes (read + write) of the kernel from the newest committed ncu --set full capture
    of this config and precision (profiles/r02/ncu_summary_<config>_<precision>.json, else the
    round-1 bf16 captures profiles/r01/ncu_summary_<config>_v{3,2}.json), or None."""
    summ = None
    cands = [("r02", f"ncu_summary_{config}_{precision}.json")]
    if precision == "bf16":
        cands += [("r01", f"ncu_summary_{config}_{v}.json") for v in ("v3", "v2")]
    for rd, name in cands:
        try:
            summ = json.load(open(os.path.join(ROOT, "profiles", rd, name)))
            break
        except (OSError, ValueError):
            continue
    if summ is None:
        return None
    unit = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for rows in summ.values():
        for r in rows:
            if isinstance(r, dict) and r.get("kernel", "").startswith(f"void {kernel_prefix}") and "dram_read" in r:
                tot = 0.0
                for k in ("dram_read", "dram_write"):
                    v, u = r[k].split()
                    tot += float(v) * unit.get(u, 1)
                return tot
    return None


def measured_peaks() -> tuple[dict, str]:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        return json.load(open(p)), "measured"
    except (OSError, ValueError):
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region: NVML polled every 5 ms
    from a thread (nvidia-smi -lms cannot go below ~100 ms, longer than a short timed region);
    falls back to nvidia-smi when NVML is unavailable."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4}

    def __init__(self, gpu: int):
        self.gpu, self.rows, self.stop = gpu, [], threading.Event()
        self.nvml = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nvml = None
        self.t = threading.Thread(target=self._poll, daemon=True)
        self.t.start()
        return self

    def _poll(self):
        while not self.stop.is_set():
            try:
                if self.nvml:
                    sm = self.nvml.nvmlDeviceGetClockInfo(self.h, self.nvml.NVML_CLOCK_SM)
                    r = self.nvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                    self.rows.append((sm, self.max_mhz, r))
                else:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), "--query-gpu=clocks.sm,clocks.max.sm",
                                          "--format=csv,noheader,nounits"], capture_output=True, text=True)
                    sm, mx = (float(v) for v in out.stdout.split(","))
                    self.rows.append((sm, mx, 0))
            except Exception:
                pass
            time.sleep(0.005)

    def __exit__(self, *a):
        self.stop.set()
        self.t.join(2)

    def summary(self) -> dict:
        sm = [r[0] for r in self.rows]
        reasons = sorted({n for r in self.rows for n, bit in self.REASONS.items() if r[2] & bit})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(r[1] for r in self.rows) if self.rows else None, "reasons": reasons,
                "samples": len(self.rows), "source": "nvml 5 ms" if self.nvml else "nvidia-smi"}


# ----------------------------------------------------------------------------- shared
def job_flops(args, world: int) -> int:
    """FLOPs of one step of the whole job: weak scaling runs `world` full minibatches, strong
    scaling splits one across the ranks. `--pass fwd` (inference forward) counts 1x, both 3x
    (bench.hpp:55-62)."""
    f = pass_flops(CONFIGS[args.config], 1 if getattr(args, "pass_", "both") == "fwd" else 3)
    return f if args.scaling == "strong" else f * world


def workload_name(key: str, c: dict, pass_: str = "both") -> str:
    base = f"{c['layers']}L h{c['hidden']} mb{c['batch']} T{c['steps']} LSTM " + (
        "fwd+bwd" if pass_ == "both" else "forward (inference)")
    return base + (" (BASELINE configs[1])" if key == "B" and pass_ == "both" else f" (sweep config {key})")


def config_dict(key: str, c: dict, world: int, pass_: str = "both") -> dict:
    """The `config` object both arms print (identical keys, so the driver can match them)."""
    return {"workload": workload_name(key, c, pass_), "model": f"lstm-{c['layers']}x{c['hidden']}",
            "global_batch": c["batch"] * world, "seq_len": c["steps"], "layers": c["layers"],
            "hidden": c["hidden"], "parallelism": f"dp{world}" if world > 1 else "single",
            "l2": "flushed (256 MiB write) between timed steps",
            "per_step_work": ("K7 repack (params updated in place) + forward (training) + backward_data + "
                              "weight_update, like the reference's time_level pass" if pass_ == "both" else
                              "K7 repack (params updated in place) + inference forward, like the reference's "
                              "time_level Forward pass")}


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ----------------------------------------------------------------------------- reference arm
def run_reference(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle  # the reference CPU engine (oracle/_ref) -- checker/baseline leg only
    R = oracle.Reference()
    c = dict(CONFIGS[args.config])  # the same workload as our arm's line
    d = oracle.Dims(**c)
    cores = os.cpu_count() or 1
    pk = 0 if args.pass_ == "fwd" else 2  # bench::PassKind Forward / Both
    flops = pass_flops(c, 1 if pk == 0 else 3)
    # one pass of the reference engine at O6 ~ seconds; bound the run to a few minutes
    est = R.time(d, seed=42, pass_kind=pk, reps=1, warmup=0, workers=cores)["median_us"] * 1e-6
    budget = 150.0
    reps = max(1, min(args.steps, int(budget / max(est, 1e-3))))
    warm = max(args.warmup, 3) if est * (reps + max(args.warmup, 3)) < 1.5 * budget else 1
    t = R.time(d, seed=42, pass_kind=pk, reps=reps, warmup=warm, workers=cores)
    sec = t["median_us"] * 1e-6
    tflops = flops / sec / 1e12
    line = {
        "impl": "reference", "metric": METRIC, "value": tflops, "unit": "TFLOP/s",
        "n_gpus": args.gpus, "steps": reps, "warmup": warm, "ms_per_step": sec * 1e3,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (SplitMix64 seed 42, reference generators)",
        # the same job description as our arm's line (weak scaling: N minibatches, which the CPU
        # engine processes at its per-minibatch rate)
        "config": config_dict(args.config, c, 1 if args.scaling == "strong" else args.gpus, args.pass_),
        "cpu_baseline": {"value": tflops, "unit": "TFLOP/s", "cores": cores, "kind": "reference",
                         "sample": f"{reps} full config-{args.config} passes (median), O6, {cores} workers",
                         "cpu": cpu_model(), "lib": os.path.basename(R.path)},
        "e2e": {"value": tflops, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- our arm
def measure(args, precision: str, world: int, rank: int, local: int, with_e2e: bool = True) -> dict:
    """Time one precision mode: K timed steps (repack + fwd + bwd + weight update), per-phase
    device times, and the end-to-end host-buffer training call. Returns a partial line."""
    import numpy as np
    import torch
    from paper_1604_01946_b200 import Engine, LadderConfig, init_params, make_dy, make_input

    c = dict(CONFIGS[args.config])
    if args.scaling == "strong" and world > 1:  # the global minibatch split across the ranks
        from paper_1604_01946_b200.parallel import shard_range
        b0, b1 = shard_range(c["batch"], rank, world)
        c["batch"] = b1 - b0
    cfg = LadderConfig(**c, seed=42 + rank, opt_level=6, batch_steps=2, workers=1)
    eng = Engine(cfg, precision=precision, schedule=args.schedule, device=local)
    params = init_params(LadderConfig(**{**c, "batch": CONFIGS[args.config]["batch"]}, seed=42))
    x = make_input(cfg)
    dy = make_dy(cfg)
    eng.set_params(params)
    eng.upload_inputs(x, dy)
    if world > 1:
        from paper_1604_01946_b200.engine import nccl_unique_id
        import torch.distributed as dist
        box = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=0)
        eng.init_comm(rank, world, box[0])
        eng.comm_overlap(True)  # per-layer buckets all-reduced inside the pass, overlapped
    stream = torch.cuda.Stream()
    sh = stream.cuda_stream

    # L2 flush buffer (> 126 MB L2) written between timed steps, outside the events
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")

    fwd_only = getattr(args, "pass_", "both") == "fwd"
    pass_kind = 0 if fwd_only else 2  # 0: inference forward (config A's "forward" line), 2: fwd + bwd

    def step():
        eng.params_updated()  # the parameters changed (optimizer): K7 repack inside the pass
        eng.run_pass(pass_kind, sh)
        if world > 1 and not fwd_only:
            eng.allreduce_grads(sh)

    with torch.cuda.stream(stream):
        for _ in range(max(args.warmup, 3)):
            step()
        eng.sync()
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()

        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(args.steps)]
        eng.launch_count(reset=True)
        with ClockSampler(local) as clk:
            for i in range(args.steps):
                flush.zero_()
                ev[i][0].record(stream)
                step()
                ev[i][1].record(stream)
            torch.cuda.synchronize()
            eng.sync()
        launches = eng.launch_count(reset=True) // args.steps
        step_ms = [a.elapsed_time(b) for a, b in ev]
        total_ms = sum(step_ms)
        if world > 1:
            t = torch.tensor([total_ms], device="cuda")
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            total_ms = t.item()
        ms = total_ms / args.steps

        # ---- per-phase device times (CUDA events on the launching stream) for the roofline
        eng.set_profiling(True)
        eng.phase_times(reset=True)
        nprof = max(3, min(args.steps, 10))
        for _ in range(nprof):
            flush.zero_()
            eng.params_updated()
            eng.run_pass(pass_kind, sh)
        eng.sync()
        ph = eng.phase_times(reset=True)
        eng.set_profiling(False)

        e2e = None
        if with_e2e and fwd_only:
            # inference through the public API with host buffers: upload x (pinned), forward, read y
            yh = torch.zeros(c["batch"] * c["steps"], c["hidden"], dtype=torch.float32).pin_memory().numpy().T
            xh = torch.from_numpy(np.asfortranarray(x).ravel(order="F")).pin_memory()
            e2e_steps = max(10, min(args.steps, 50))

            def infer():
                eng.params_updated()
                eng.upload_inputs_ptr(xh.data_ptr(), 0)
                eng.run_pass(0)
                eng.read_outputs(y=yh)

            for _ in range(3):
                infer()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(e2e_steps):
                infer()
            e2e_ms = (time.perf_counter() - t0) * 1e3 / e2e_steps
            e2e = {"value": job_flops(args, world) / (e2e_ms * 1e-3) / 1e12, "unit": "TFLOP/s",
                   "ms_per_step": e2e_ms, "h2d_bytes_per_step": xh.numel() * 4, "d2h_bytes_per_step": yh.size * 4,
                   "path": "C-ABI rw_upload_inputs (pinned host x) -> rw_run_pass(0) (K7 repack + inference "
                           "forward) -> rw_read_outputs(y) on the host"}
        elif with_e2e:
            def pinned(rows, cols=None):
                """Column-major float32 host array in pinned (page-locked) memory."""
                if cols is None:
                    return torch.zeros(rows, dtype=torch.float32).pin_memory().numpy()
                return torch.zeros(cols, rows, dtype=torch.float32).pin_memory().numpy().T

            y = pinned(c["hidden"], c["batch"] * c["steps"])
            dx0 = pinned(c["input"], c["batch"] * c["steps"])
            dw = [pinned(4 * c["hidden"], c["input"] if l == 0 else c["hidden"]) for l in range(c["layers"])]
            dr = [pinned(4 * c["hidden"], c["hidden"]) for _ in range(c["layers"])]
            db = [pinned(4 * c["hidden"]) for _ in range(c["layers"])]
            xh = torch.from_numpy(np.asfortranarray(x).ravel(order="F")).pin_memory()
            dyh = torch.from_numpy(np.asfortranarray(dy).ravel(order="F")).pin_memory()
            h2d = xh.numel() * 4 + dyh.numel() * 4
            d2h = (y.size + dx0.size + sum(a.size for a in dw) + sum(a.size for a in dr)
                   + sum(a.size for a in db)) * 4
            # the public training call with host buffers: rw_train_step uploads x/dy, runs the
            # pass (repack of the updated parameters included, + the DP all-reduce) and reads y,
            # dx0, dW, dR, db back, pipelined so the next step's uploads and this step's read-back
            # overlap compute; wall clock over the whole sequence including the final wait
            e2e_steps = max(10, min(args.steps, 50))
            xn, dyn = xh.numpy(), dyh.numpy()
            for _ in range(3):
                eng.params_updated()
                eng.train_step(xn, dyn, y, dx0, dw, dr, db)
            eng.train_wait()
            torch.cuda.synchronize()
            if world > 1:
                torch.distributed.barrier()
            t0 = time.perf_counter()
            for _ in range(e2e_steps):
                eng.params_updated()
                eng.train_step(xn, dyn, y, dx0, dw, dr, db)
            eng.train_wait()
            e2e_ms = (time.perf_counter() - t0) * 1e3 / e2e_steps
            if world > 1:
                t = torch.tensor([e2e_ms], device="cuda")
                torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
                e2e_ms = t.item()
            e2e = {"value": job_flops(args, world) / (e2e_ms * 1e-3) / 1e12, "unit": "TFLOP/s",
                   "ms_per_step": e2e_ms, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                   "path": "C-ABI rw_train_step (pinned host x, dy -> K7 repack + forward + backward_data"
                           " + weight_update -> y, dx0, dW, dR, db on the host; uploads/read-back"
                           " pipelined against compute)"}
    desc = eng.describe()
    eng.close()
    return {"ms": ms, "ph": ph, "launches": launches, "clocks": clk.summary(), "e2e": e2e, "desc": desc}


def roofline(args, m: dict, precision: str) -> tuple[dict, dict]:
    c = dict(CONFIGS[args.config])
    peaks, peak_src = measured_peaks()
    desc, ph = m["desc"], m["ph"]
    planes = 1 if precision == "bf16" else 2  # fp32-parity: hi and lo operand planes
    # dominant kernel: the longer of the two recurrent (persistent / stepwise / cluster) phases
    fwd_ms = ph["fwd_recurrent"][0] / max(ph["fwd_recurrent"][1], 1)
    bwd_ms = ph["bwd_recurrent"][0] / max(ph["bwd_recurrent"][1], 1)
    L, H, I, B, T = c["layers"], c["hidden"], c["input"], c["batch"], c["steps"]
    fwd_fl = pass_flops(c, 1)  # [W|R].[x;h] for every cell
    bwd_fl = sum(2 * 4 * H * (H + (H if l < L - 1 else 0)) * B * (T + 1)
                 for l in range(L))  # W_{l+1}^T and R_l^T per cell (+ the dh0 step)
    kern = {"cluster": ("k_cl_fwd", "k_cl_bwd"), "persistent": ("k_lstm_fwd", "k_lstm_bwd"),
            "layerseq": ("k_gemm_p + k_lstm_fwd", "k_gemm_p + k_lstm_bwd"),
            "stepwise": ("k_lstm_fwd", "k_lstm_bwd")}
    kf = kern.get(desc["fwd_schedule"], ("k_lstm_fwd",))[0]
    kb = kern.get(desc["bwd_schedule"], ("", "k_lstm_bwd"))[1]
    if bwd_ms >= fwd_ms and getattr(args, "pass_", "both") != "fwd":
        dom, dom_ms, dom_fl = f"{kb} (fused recurrent backward, {desc['bwd_schedule']})", bwd_ms, bwd_fl
        dom_k, dom_by = kb, recurrent_bytes(c, False, planes)
    else:
        dom, dom_ms, dom_fl = f"{kf} (fused recurrent forward, {desc['fwd_schedule']})", fwd_ms, fwd_fl
        dom_k, dom_by = kf, recurrent_bytes(c, True, planes)
    achieved = dom_fl / (dom_ms * 1e-3) / 1e12
    # burst peak for a kernel timed alone; the sustained (power-capped) one once the kernel runs
    # long enough to hit the power limit (>= 10 ms)
    peak_burst = peaks.get("bf16_tflops", 1590.0)
    peak_sus = peaks.get("bf16_tflops_sustained", 1400.0)
    long_kernel = dom_ms >= 10.0
    peak = peak_sus if long_kernel else peak_burst
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    hbm_bound = dom_by / (hbm_peak * 1e9) > dom_fl / (peak * 1e12)
    traffic = ncu_traffic(dom_k.split()[0], args.config, precision)
    note = ("fp32-parity: each product is 3 tensor-core MMAs on split operands (hi.hi + hi.lo + "
            "lo.hi), so the attainable ceiling is peak/3; frac is against the full dense bf16 peak"
            if precision == "fp32" else "bf16 operands, fp32 accumulation")
    if hbm_bound:
        r = {"kernel": dom, "bound": "hbm", "achieved": dom_by / (dom_ms * 1e-3) / 1e9, "peak": hbm_peak,
             "unit": "GB/s", "frac": dom_by / (dom_ms * 1e-3) / 1e9 / hbm_peak, "traffic": traffic,
             "peak_source": f"{peak_src} HBM copy bandwidth (MEASURED_PEAKS.json)",
             "algorithmic_bytes_per_launch": dom_by, "tensor_tflops": achieved,
             "tensor_frac": achieved / peak, "avg_launch_ms": dom_ms, "note": note}
    else:
        r = {"kernel": dom, "bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
             "frac": achieved / peak, "traffic": traffic,
             "peak_source": f"{peak_src} bf16 dense {'sustained' if long_kernel else 'burst'} (MEASURED_PEAKS.json)",
             "algorithmic_flops_per_launch": dom_fl, "algorithmic_bytes_per_launch": dom_by,
             "hbm_frac": dom_by / (dom_ms * 1e-3) / 1e9 / hbm_peak, "avg_launch_ms": dom_ms, "note": note}
    crit = {"steps_fwd": T + L - 1, "steps_bwd": T + L,
            "us_per_step_fwd": 1e3 * fwd_ms / (T + L - 1), "us_per_step_bwd": 1e3 * bwd_ms / (T + L)}
    return r, crit


def run_ours(args) -> None:
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    c = dict(CONFIGS[args.config])
    m = measure(args, args.precision, world, rank, local)
    # the other precision mode, same workload, as a secondary key (bf16 is narrower arithmetic
    # than the reference's fp32: never the headline)
    other = "bf16" if args.precision == "fp32" else "fp32"
    m2 = None if args.single_precision else measure(args, other, world, rank, local, with_e2e=True)
    if rank != 0:
        return
    peaks, _ = measured_peaks()
    peak_burst = peaks.get("bf16_tflops", 1590.0)
    peak_sus = peaks.get("bf16_tflops_sustained", 1400.0)
    rf, crit = roofline(args, m, args.precision)
    cpu_base = None
    if not args.no_cpu_baseline and args.config in ("A", "B"):
        cpu_base = cpu_baseline(args.config, args.pass_)
    value = job_flops(args, world) / (m["ms"] * 1e-3) / 1e12
    dtype = {"bf16": "bf16", "fp32": "tf32x3 (fp32-parity)"}
    operands = {"tf32x3": "3xTF32 split operands", "fp16x2": "fp16x2 split operands (hi + lo, 3 MMAs)",
                "bf16": "bf16 operands"}
    cfgd = config_dict(args.config, c, 1 if args.scaling == "strong" else world, args.pass_)
    cfgd.update({"precision": args.precision, "schedule": m["desc"],
                 "operands": operands.get(m["desc"]["operands"], m["desc"]["operands"]),
                 "pct_of_bf16_peak": 100.0 * value / world / peak_burst,
                 "pct_of_bf16_peak_sustained": 100.0 * value / world / peak_sus})
    line = {
        "metric": METRIC,
        "value": value,
        "unit": "TFLOP/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": max(args.warmup, 3),
        "ms_per_step": m["ms"],
        "higher_is_better": True,
        "scaling": args.scaling,
        "vs_baseline": None,
        "dtype": dtype[args.precision],
        "data": "synthetic (SplitMix64 seed 42 weights, streams 1000/1001 inputs: the reference generators)",
        "config": cfgd,
        "e2e": m["e2e"],
        "roofline": rf,
        "phases_ms": {k: v[0] / max(v[1], 1) for k, v in m["ph"].items()},
        # SURVEY §8d's latency bound: the wavefront's dependent steps (T + L - 1 per direction,
        # + the dh0 step backward) and the measured time per step of each recurrent phase
        "critical_path": crit,
        "gpu_launches": m["launches"],
        "clocks": m["clocks"],
        "cpu_baseline": cpu_base,
    }
    if m2 is not None:
        rf2, crit2 = roofline(args, m2, other)
        v2 = job_flops(args, world) / (m2["ms"] * 1e-3) / 1e12
        line[other] = {"dtype": dtype[other], "value": v2, "unit": "TFLOP/s", "ms_per_step": m2["ms"],
                       "e2e": m2["e2e"], "schedule": m2["desc"], "roofline": rf2, "critical_path": crit2,
                       "phases_ms": {k: v[0] / max(v[1], 1) for k, v in m2["ph"].items()},
                       "pct_of_bf16_peak": 100.0 * v2 / world / peak_burst, "gpu_launches": m2["launches"],
                       "clocks": m2["clocks"]}
    print(json.dumps(line), flush=True)


def cpu_baseline(key: str = "B", pass_: str = "both") -> dict | None:
    """The reference CPU engine on the host cores, bounded sample of the same workload: P = all
    host threads and P = min(nproc, 2L) (the reference CLI's default worker count,
    rnnwave.cpp:30-37)."""
    try:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import oracle
        R = oracle.Reference()
        kind = "reference"
    except Exception:
        return None
    c = CONFIGS[key]
    d = oracle.Dims(**c)
    cores = os.cpu_count() or 1
    pk, mult = (0, 1) if pass_ == "fwd" else (2, 3)
    t = R.time(d, seed=42, pass_kind=pk, reps=3, warmup=1, workers=cores)
    sec = t["median_us"] * 1e-6
    p2 = min(cores, 2 * c["layers"])
    t2 = R.time(d, seed=42, pass_kind=pk, reps=3, warmup=1, workers=p2)
    sec2 = t2["median_us"] * 1e-6
    what = "fwd+bwd" if pass_ == "both" else "inference forward"
    return {"value": pass_flops(c, mult) / sec / 1e12, "unit": "TFLOP/s", "cores": cores,
            "kind": kind, "ms_per_step": sec * 1e3, "cpu": cpu_model(),
            "sample": f"3 full config-{key} {what} passes after 1 warm-up (median), O6, workers=cores",
            "default_workers": {"workers": p2, "value": pass_flops(c, mult) / sec2 / 1e12, "ms_per_step": sec2 * 1e3,
                                "why": "min(nproc, 2L), the reference CLI default (rnnwave.cpp:30-37)"}}


# ----------------------------------------------------------------------------- GPU ladder
LADDER_LABELS = ["Naive", "Grouped GEMMs", "Streamed GEMMs", "Fused point-wise", "Pre-transpose",
                 "Batching inputs", "Overlapping layers"]  # bench.hpp:30-32


def write_ladder_csv(f, c: dict, rows: list, reps: int, warmup: int, precision: str) -> None:
    """The reference's write_ladder_csv schema (bench.hpp:226-242): the same two comment lines
    (plus the device and precision), the same header and %.3f columns."""
    f.write(f"# rnnwave run-ladder: cell=lstm layers={c['layers']} hidden={c['hidden']} input={c['input']} "
            f"batch={c['batch']} steps={c['steps']} batch_steps=2 workers=1 seed=42 pass=fwd reps={reps} "
            f"warmup={warmup} device=B200 precision={precision}\n")
    f.write("# us_per_cell is the median over reps; gflops counts GEMM multiply-adds only "
            "(2*G*H*(I+H)*B per cell, pass multiplier fwd=1 bwd=2 both=3)\n")
    f.write("opt_level,label,us_per_cell,speedup_vs_naive,gflops,equiv_ok\n")
    for r in rows:
        f.write(f"{r['opt_level']},{r['label']},{r['us_per_cell']:.3f},{r['speedup_vs_naive']:.3f},"
                f"{r['gflops']:.3f},{'true' if r['equiv_ok'] else 'false'}\n")


def run_ladder(args) -> None:
    """The reference's run_ladder (bench.hpp:176-224) on the GPU: the seven rungs of the paper's
    Table 1 as device variants (runtime.cu run_ladder_forward: O0-O4 on a stepwise context, O5 the
    layer-sequential schedule, O6 the automatic wavefront), forward pass, median over reps, each
    rung checked against O0 (equiv_ok: y within the precision's tolerance -- the reference's check
    is bitwise, a tensor-core build's is a tolerance) and written in write_ladder_csv's schema
    (bench.hpp:226-242)."""
    import numpy as np
    import torch
    from paper_1604_01946_b200 import Engine, LadderConfig, init_params, make_dy, make_input
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from parity import TOL, errors
    torch.cuda.set_device(0)
    c = dict(CONFIGS[args.config])
    cfg = LadderConfig(**c, seed=42, opt_level=6, batch_steps=2, workers=1)
    params = init_params(cfg)
    x, dy = make_input(cfg), make_dy(cfg)
    engines = {"stepwise": Engine(cfg, precision=args.precision, schedule="stepwise"),
               "layerseq": Engine(cfg, precision=args.precision, schedule="layerseq"),
               "auto": Engine(cfg, precision=args.precision, schedule="auto")}
    for e in engines.values():
        e.set_params(params)
        e.upload_inputs(x, dy)
    stream = torch.cuda.Stream()
    sh = stream.cuda_stream

    def run(level):
        if level <= 4:
            engines["stepwise"].ladder_pass(level, sh)
            return engines["stepwise"]
        e = engines["layerseq" if level == 5 else "auto"]
        e.run_pass(0, sh)
        return e

    cells = c["layers"] * c["steps"]
    flop_cell = 2 * 4 * c["hidden"] * (c["input"] + c["hidden"]) * c["batch"]
    rows, y0, naive = [], None, None
    with torch.cuda.stream(stream):
        for level in range(7):
            for _ in range(max(args.warmup, 2)):
                e = run(level)
            e.sync()
            y = np.zeros((c["hidden"], c["batch"] * c["steps"]), np.float32, order="F")
            e.read_outputs(y=y)
            if y0 is None:
                y0 = y
            nw, sm = errors(y, y0)
            tol = TOL[args.precision]
            equiv = nw <= tol[0] and sm <= tol[1]
            reps = max(3, min(args.steps, 20))
            ts = []
            for _ in range(reps):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                run(level)
                b.record(stream)
                b.synchronize()
                ts.append(a.elapsed_time(b) * 1e3)
            med = statistics.median(ts)
            us_cell = round(med / cells, 3)
            if naive is None:
                naive = us_cell
            rows.append({"opt_level": level, "label": LADDER_LABELS[level], "us_per_cell": us_cell,
                         "speedup_vs_naive": round(naive / us_cell, 3) if us_cell else 0.0,
                         "gflops": flop_cell / (us_cell * 1000.0), "equiv_ok": bool(equiv),
                         "y_normwise_vs_O0": nw, "schedule": engines["auto"].describe()["fwd_schedule"]
                         if level == 6 else ("layerseq" if level == 5 else "stepwise")})
    out = args.ladder_csv or os.path.join(ROOT, "gpurun_out", f"ladder_{args.config}_{args.precision}.csv")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    with open(out, "w") as f:
        write_ladder_csv(f, c, rows, reps=max(3, min(args.steps, 20)), warmup=max(args.warmup, 2),
                         precision=args.precision)
    print(json.dumps({"ladder": rows, "csv": out, "config": workload_name(args.config, c),
                      "precision": args.precision}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--precision", default="fp32", choices=["bf16", "fp32"],
                    help="headline precision: fp32 = the reference's fp32 contract (split-operand "
                         "tensor-core products, parity <= 1e-5); the other mode is a secondary key")
    ap.add_argument("--single-precision", action="store_true", help="skip the secondary precision")
    ap.add_argument("--schedule", default="auto", choices=["auto", "stepwise", "persistent", "cluster", "layerseq"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--pass", dest="pass_", default="both", choices=["both", "fwd"],
                    help="both: training step (the headline); fwd: inference forward (SURVEY 8d config A)")
    ap.add_argument("--ladder", action="store_true", help="the GPU optimisation ladder (O0-O6) in the "
                    "reference's run-ladder CSV schema instead of the bench line")
    ap.add_argument("--ladder-csv", default=None)
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="multi-GPU: weak = every rank its own full minibatch (data parallel); strong = "
                         "the configuration's minibatch split across the ranks (e.g. --config E, B = 256)")
    ap.add_argument("--config", default="B", choices=sorted(CONFIGS),
                    help="SURVEY §8(d) config; B (the headline) unless sweeping")
    args = ap.parse_args()
    if args.ladder:
        run_ladder(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
