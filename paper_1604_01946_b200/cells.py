"""The free functions of the reference's cell and GEMM layers on the device (Python mirror of
include/rnnwave/cells.hpp and gemm.hpp): ``pointwise_forward`` (cells.hpp:181-333),
``pointwise_backward`` (cells.hpp:349-562) and ``gemm`` (gemm.hpp:339-347), with the
reference's argument meaning, dimension checks and messages. Arrays are float32 matrices
(column-major copies are made as needed); outputs are written in place like the reference's
spans. All three run on the sm_100a kernels of librnnwave_sm100 (rw_pointwise_forward /
rw_pointwise_backward / rw_gemm); there is no host fallback.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .engine import gate_count

_F = C.POINTER(C.c_float)


def _check(status: int) -> None:
    if status == 0:
        return
    msg = _lib.load().rw_last_error(None).decode()
    raise (ValueError if status == _lib.RW_EINVAL else RuntimeError)(msg)


def _dims(a, rows: int, cols: int, what: str) -> None:
    if a.shape != (rows, cols):
        raise ValueError(f"cells: {what} is {a.shape[0]}x{a.shape[1]}, expected {rows}x{cols}")


def _in(a):
    return None if a is None else np.asfortranarray(a, dtype=np.float32)


def _p(a):
    return None if a is None else a.ctypes.data_as(_F)


class _Out:
    """A column-major float32 scratch for an output array, copied back into it afterwards."""

    def __init__(self, a):
        self.a = a
        self.buf = None if a is None else np.zeros(a.shape, np.float32, order="F")

    def ptr(self):
        return _p(self.buf)

    def back(self):
        if self.a is not None:
            self.a[...] = self.buf


def pointwise_forward(kind: int, fused: bool, zw, zr, bias, h_prev, c_prev, h_out, c_out=None,
                      gates=None, tanh_c=None, zr_h=None) -> None:
    """cells.hpp:181-333. ``gates`` / ``tanh_c`` / ``zr_h`` are the training save slots (None:
    inference); the RNN kinds save nothing (their saved state is h_out)."""
    h_prev = _in(h_prev)
    hidden, batch = h_prev.shape
    G = gate_count(kind)
    zw, zr = _in(zw), _in(zr)
    _dims(zw, G * hidden, batch, "zw")
    _dims(zr, G * hidden, batch, "zr")
    _dims(h_out, hidden, batch, "h_out")
    if kind == 3:
        _dims(c_prev, hidden, batch, "c_prev")
        _dims(c_out, hidden, batch, "c_out")
    elif c_prev is not None:
        raise ValueError("cells: cell state supplied for a cell kind without one")
    rnn = kind in (0, 1)
    outs = [_Out(h_out), _Out(c_out if kind == 3 else None), _Out(None if rnn else gates),
            _Out(tanh_c if kind == 3 else None), _Out(zr_h if kind == 2 else None)]
    b = np.ascontiguousarray(bias, dtype=np.float32)
    _check(_lib.load().rw_pointwise_forward(kind, 1 if fused else 0, hidden, batch, _p(zw), _p(zr), _p(b),
                                            _p(h_prev), _p(_in(c_prev)), *[o.ptr() for o in outs]))
    for o in outs:
        o.back()


def pointwise_backward(kind: int, fused: bool, gates, tanh_c, zr_h, h_prev, c_prev, d_above, dh_carry,
                       dc_carry, dgw, dgr, dh_local, dc_prev=None, db=None) -> None:
    """cells.hpp:349-562; ``gates`` is the saved gates (the post-activation h for the RNN kinds),
    ``db`` an optional float32 accumulator of G*H (+= row sums of dgw)."""
    d_above = _in(d_above)
    hidden, batch = d_above.shape
    G = gate_count(kind)
    _dims(dgw, G * hidden, batch, "dgw")
    _dims(dh_carry, hidden, batch, "dh_carry")
    _dims(dh_local, hidden, batch, "dh_local")
    if gates is None:
        raise ValueError("cells: backward requires saved state from a training forward")
    if kind == 3:
        _dims(dc_carry, hidden, batch, "dc_carry")
        _dims(dc_prev, hidden, batch, "dc_prev")
    if kind == 2:
        if dgr is None or dgr is dgw:
            raise ValueError("cells: GRU needs distinct dgw and dgr blocks")
        _dims(dgr, G * hidden, batch, "dgr")
    outs = [_Out(dgw), _Out(dgr if kind == 2 else None), _Out(dh_local), _Out(dc_prev if kind == 3 else None)]
    dbb = None
    if db is not None:
        dbb = np.ascontiguousarray(db, dtype=np.float32).copy()
    lstm, gru = kind == 3, kind == 2
    _check(_lib.load().rw_pointwise_backward(
        kind, 1 if fused else 0, hidden, batch, _p(_in(gates)), _p(_in(tanh_c) if lstm else None),
        _p(_in(zr_h) if gru else None), _p(_in(h_prev) if gru else None), _p(_in(c_prev) if lstm else None),
        _p(d_above), _p(_in(dh_carry)), _p(_in(dc_carry) if lstm else None), *[o.ptr() for o in outs], _p(dbb)))
    for o in outs:
        o.back()
    if db is not None:
        db[...] = dbb.reshape(db.shape)


def gemm(trans_a: bool, trans_b: bool, a, b, c, alpha: float, beta: float) -> None:
    """gemm.hpp:339-347: c = alpha op(a) op(b) + beta c (in place), fp32-parity tensor-core GEMM."""
    a, b = _in(a), _in(b)
    am, ak = (a.shape[1], a.shape[0]) if trans_a else a.shape
    bk, bn = (b.shape[1], b.shape[0]) if trans_b else b.shape
    if ak != bk:
        raise ValueError(f"gemm: op(A) is {am}x{ak} but op(B) is {bk}x{bn}; inner dimensions differ")
    if c.shape != (am, bn):
        raise ValueError(f"gemm: C is {c.shape[0]}x{c.shape[1]} but op(A)*op(B) is {am}x{bn}")
    if am == 0 or bn == 0:
        return
    out = _Out(c)
    out.buf[...] = c
    _check(_lib.load().rw_gemm(1 if trans_a else 0, 1 if trans_b else 0, am, bn, ak, alpha, _p(a), max(a.shape[0], 1),
                               _p(b), max(b.shape[0], 1), beta, out.ptr(), am))
    out.back()
