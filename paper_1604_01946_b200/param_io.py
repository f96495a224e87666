"""The reference's binary parameter file (proj/include/rnnwave/param_io.hpp:18-151), so that
`save-params` artifacts of the reference CLI load bit-exactly into a device context (SURVEY §8f,
"next" row 3).

Layout (param_io.hpp:18-26): 16 bytes magic "RNNWAVE1" + 8 zero bytes; five little-endian
uint32 -- kind (0 rnn-tanh, 1 rnn-relu, 2 gru, 3 lstm), layers, hidden, input, batch hint; then
per layer W ((G*H) x I_l), R ((G*H) x H), bias (G*H) as raw little-endian float32, column-major.
Errors keep the reference's messages (std::runtime_error -> RuntimeError, invalid_argument ->
ValueError).
"""
from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np

from .engine import CELL_NAMES, LadderConfig, LayerParams, gate_count

MAGIC = b"RNNWAVE1" + b"\0" * 8


@dataclass
class ParamFileHeader:
    """param_io.hpp:33-39."""
    kind: int = 3
    layers: int = 0
    hidden: int = 0
    input: int = 0
    batch_hint: int = 0


def param_file_size(h: ParamFileHeader) -> int:
    """param_io.hpp:41-50."""
    gh = gate_count(h.kind) * h.hidden
    total = 16 + 20
    for l in range(h.layers):
        il = h.input if l == 0 else h.hidden
        total += 4 * (gh * il + gh * h.hidden + gh)
    return total


def save_params(path: str, header: ParamFileHeader, params: list[LayerParams]) -> None:
    """param_io.hpp:70-92."""
    if len(params) != header.layers:
        raise ValueError(f"save_params: header says {header.layers} layers, got {len(params)}")
    try:
        f = open(path, "wb")
    except OSError:
        raise RuntimeError(f"save_params: cannot open {path}") from None
    with f:
        f.write(MAGIC)
        f.write(struct.pack("<5I", header.kind, header.layers, header.hidden, header.input, header.batch_hint))
        for p in params:
            for a in (p.w, p.r):
                f.write(np.asarray(a, dtype="<f4").tobytes(order="F"))
            f.write(np.asarray(p.bias, dtype="<f4").tobytes())


def load_params(path: str) -> tuple[ParamFileHeader, list[LayerParams]]:
    """param_io.hpp:99-133."""
    try:
        f = open(path, "rb")
    except OSError:
        raise RuntimeError(f"load_params: cannot open {path}") from None
    with f:
        data = f.read()
    if len(data) < 16 or data[:16] != MAGIC:
        raise RuntimeError(f"load_params: {path} is not a parameter file (bad magic)")
    names = ["kind", "layers", "hidden", "input", "batch hint"]
    vals = []
    for i, n in enumerate(names):
        off = 16 + 4 * i
        if off + 4 > len(data):
            raise RuntimeError(f"param file: truncated while reading {n}")
        vals.append(struct.unpack_from("<I", data, off)[0])
        if i == 0 and vals[0] > 3:
            raise RuntimeError(f"load_params: unknown cell kind {vals[0]}")
    h = ParamFileHeader(*vals)
    if h.layers <= 0 or h.hidden <= 0 or h.input <= 0:
        raise RuntimeError("load_params: non-positive dimensions in header")
    gh = gate_count(h.kind) * h.hidden
    off = 36
    params = []

    def take(n, what):
        nonlocal off
        if off + 4 * n > len(data):
            raise RuntimeError(f"param file: truncated while reading {what}")
        a = np.frombuffer(data, dtype="<f4", count=n, offset=off).astype(np.float32)
        off += 4 * n
        return a

    for l in range(h.layers):
        il = h.input if l == 0 else h.hidden
        w = take(gh * il, f"layer {l} W").reshape((gh, il), order="F")
        r = take(gh * h.hidden, f"layer {l} R").reshape((gh, h.hidden), order="F")
        b = take(gh, f"layer {l} bias")
        params.append(LayerParams(np.asfortranarray(w), np.asfortranarray(r), b))
    return h, params


def check_matches(h: ParamFileHeader, cfg: LadderConfig) -> None:
    """param_io.hpp:136-148."""
    if h.kind != cfg.kind:
        raise RuntimeError(f"param file: cell kind is {CELL_NAMES.get(h.kind, '?')} but the configuration expects "
                           f"{CELL_NAMES.get(cfg.kind, '?')}")
    for what, got, want in (("layer count", h.layers, cfg.layers), ("hidden size", h.hidden, cfg.hidden),
                            ("input size", h.input, cfg.input)):
        if got != want:
            raise RuntimeError(f"param file: {what} is {got} but the configuration expects {want}")
