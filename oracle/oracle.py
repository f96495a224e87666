"""ctypes loaders for the CPU checkers (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
import this module. The product path (paper_1604_01946_b200 + librnnwave_sm100.so)
never imports it: it is the checker, not the thing measured or shipped.

Two checkers:
  * ``Restatement`` -- oracle/lstm_oracle.c, the C restatement of the reference LSTM path
    (bitwise equal to the reference engine on the same host libm).
  * ``Reference``   -- oracle/_ref/librwref_v*.so, a shim over the UNMODIFIED reference
    engine compiled from /root/reference/proj/include (see oracle/Makefile). Provides the
    reference Engine pipeline, its fp64 oracle and its bench::time_level timer.

Arrays are numpy float32, column-major flattened exactly like rnnwave::Matrix
(element (r, c) at c*rows + r); we carry them as 2-D arrays in Fortran order.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_F = C.POINTER(C.c_float)
_D = C.POINTER(C.c_double)
_PF = C.POINTER(_F)
_PD = C.POINTER(_D)


@dataclass
class Dims:
    layers: int
    hidden: int
    input: int
    batch: int
    steps: int
    kind: int = 3  # the reference's CellKind: 0 rnn-tanh, 1 rnn-relu, 2 gru, 3 lstm

    def input_width(self, l: int) -> int:
        return self.input if l == 0 else self.hidden


def gate_count(kind: int) -> int:
    """config.hpp:19-28: RNN 1, GRU 3, LSTM 4 (kind in the reference's CellKind order)."""
    return {0: 1, 1: 1, 2: 3, 3: 4}[kind]


def _dims(cfg) -> Dims:
    return Dims(cfg.layers, cfg.hidden, cfg.input, cfg.batch, cfg.steps)


def fmat(rows: int, cols: int, dtype=np.float32) -> np.ndarray:
    return np.zeros((rows, cols), dtype=dtype, order="F")


def _fp(a):
    if a is None:
        return None
    assert a.flags.f_contiguous or a.ndim == 1, "expected Fortran-ordered array"
    return a.ctypes.data_as(_F if a.dtype == np.float32 else _D)


def _arr(ptrs, typ=_F):
    if ptrs is None:
        return None
    return (typ * len(ptrs))(*ptrs)


def build(quiet: bool = True) -> None:
    """make -C oracle (restatement always; reference shim when /root/reference exists)."""
    out = subprocess.run(["make", "-C", HERE, "all"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


# --------------------------------------------------------------------------------------
class _RwoDims(C.Structure):
    _fields_ = [("layers", C.c_int), ("hidden", C.c_int), ("input", C.c_int),
                ("batch", C.c_int), ("steps", C.c_int)]


class Restatement:
    """oracle/lstm_oracle.c through ctypes."""

    def __init__(self):
        path = os.path.join(HERE, "_build", "librwo.so")
        if not os.path.exists(path):
            build()
        self.lib = C.CDLL(path)
        L = self.lib
        L.rwo_fill_symmetric.argtypes = [C.c_uint64, C.c_uint64, C.c_double, _F, C.c_int64]
        L.rwo_init_params.argtypes = [C.POINTER(_RwoDims), C.c_uint64, _PF, _PF]
        L.rwo_make_input.argtypes = [C.POINTER(_RwoDims), C.c_uint64, _F]
        L.rwo_make_dy.argtypes = [C.POINTER(_RwoDims), C.c_uint64, _F]
        L.rwo_flop_count_cell.argtypes = [C.c_int, C.c_int, C.c_int]
        L.rwo_flop_count_cell.restype = C.c_int64
        L.rwo_forward.argtypes = [C.POINTER(_RwoDims), _PF, _PF, _PF, _F, _PF, _PF, C.c_int,
                                  _PF, _PF, _PF, _PF, _F]
        L.rwo_backward_data.argtypes = [C.POINTER(_RwoDims), _PF, _PF, _PF, _PF, _PF, _PF, _F,
                                        _PF, _F, _PF, _PF]
        L.rwo_weight_update.argtypes = [C.POINTER(_RwoDims), _F, _PF, _PF, _PF, _PF, _PF]

    def fill_symmetric(self, seed, stream, rng, n):
        out = np.zeros(n, np.float32)
        self.lib.rwo_fill_symmetric(seed, stream, rng, _fp(out), n)
        return out

    def init_params(self, cfg, seed):
        d = _dims(cfg)
        G = 4 * d.hidden
        w = [fmat(G, d.input_width(l)) for l in range(d.layers)]
        r = [fmat(G, d.hidden) for _ in range(d.layers)]
        self.lib.rwo_init_params(C.byref(_RwoDims(d.layers, d.hidden, d.input, d.batch, d.steps)), seed,
                                 _arr([_fp(a) for a in w]), _arr([_fp(a) for a in r]))
        return w, r

    def make_input(self, cfg, seed):
        d = _dims(cfg)
        x = fmat(d.input, d.batch * d.steps)
        self.lib.rwo_make_input(C.byref(_RwoDims(d.layers, d.hidden, d.input, d.batch, d.steps)), seed, _fp(x))
        return x

    def make_dy(self, cfg, seed):
        d = _dims(cfg)
        dy = fmat(d.hidden, d.batch * d.steps)
        self.lib.rwo_make_dy(C.byref(_RwoDims(d.layers, d.hidden, d.input, d.batch, d.steps)), seed, _fp(dy))
        return dy

    def flop_count_cell(self, hidden, inp, batch):
        return int(self.lib.rwo_flop_count_cell(hidden, inp, batch))

    def run(self, cfg, w, r, b, x, h0=None, c0=None, dy=None, training=True):
        """Forward (+ backward_data + weight_update when dy is given). Returns a dict of
        Fortran-ordered float32 arrays named like the reference fields."""
        if getattr(cfg, "kind", 3) != 3:
            raise NotImplementedError("the C restatement covers the LSTM path; use Reference for GRU / RNN")
        d = _dims(cfg)
        H, B, T, G = d.hidden, d.batch, d.steps, 4 * d.hidden
        L = d.layers
        dd = C.byref(_RwoDims(d.layers, d.hidden, d.input, d.batch, d.steps))
        training = training or dy is not None
        out = {
            "h_seq": [fmat(H, B * (T + 1)) for _ in range(L)],
            "c_seq": [fmat(H, B * (T + 1)) for _ in range(L)],
            "gates_seq": [fmat(G, B * T) for _ in range(L)] if training else None,
            "tanh_c_seq": [fmat(H, B * T) for _ in range(L)] if training else None,
            "y": fmat(H, B * T),
        }
        P = lambda lst: _arr([_fp(a) for a in lst]) if lst is not None else None  # noqa: E731
        self.lib.rwo_forward(dd, P(w), P(r), P(b), _fp(x), P(h0), P(c0), int(training),
                             P(out["h_seq"]), P(out["c_seq"]), P(out["gates_seq"]),
                             P(out["tanh_c_seq"]), _fp(out["y"]))
        if dy is None:
            return out
        out["dgw_seq"] = [fmat(G, B * T) for _ in range(L)]
        out["dx0"] = fmat(d.input, B * T)
        out["dh0"] = [fmat(H, B) for _ in range(L)]
        out["dc0"] = [fmat(H, B) for _ in range(L)]
        self.lib.rwo_backward_data(dd, P(w), P(r), P(out["h_seq"]), P(out["c_seq"]),
                                   P(out["gates_seq"]), P(out["tanh_c_seq"]), _fp(dy),
                                   P(out["dgw_seq"]), _fp(out["dx0"]), P(out["dh0"]),
                                   P(out["dc0"]))
        out["dw"] = [fmat(G, d.input_width(l)) for l in range(L)]
        out["dr"] = [fmat(G, H) for _ in range(L)]
        out["db"] = [np.zeros(G, np.float32) for _ in range(L)]
        self.lib.rwo_weight_update(dd, _fp(x), P(out["h_seq"]), P(out["dgw_seq"]),
                                   P(out["dw"]), P(out["dr"]), P(out["db"]))
        return out


# --------------------------------------------------------------------------------------
def _cpu_isa_level() -> int:
    try:
        flags = open("/proc/cpuinfo").read()
    except OSError:
        return 2
    if " avx512f" in flags and " avx512bw" in flags and " avx512vl" in flags:
        return 4
    if " avx2" in flags and " fma" in flags and " bmi2" in flags:
        return 3
    return 2


def reference_path() -> str | None:
    lvl = _cpu_isa_level()
    for v in range(lvl, 1, -1):
        p = os.path.join(HERE, "_ref", f"librwref_v{v}.so")
        if os.path.exists(p):
            return p
    return None


class Reference:
    """Shim over the unmodified reference engine (oracle/_ref)."""

    def __init__(self, path: str | None = None):
        path = path or reference_path()
        if path is None:
            if os.path.isdir("/root/reference/proj/include"):
                build()
                path = reference_path()
            if path is None:
                raise FileNotFoundError("oracle/_ref/librwref_v*.so not built")
        self.path = path
        self.lib = C.CDLL(path)
        L = self.lib
        L.rwref_init_params.argtypes = [C.POINTER(C.c_int), C.c_uint64, _PF, _PF]
        L.rwref_make_input.argtypes = [C.POINTER(C.c_int), C.c_uint64, _F, _F]
        L.rwref_flop_count_cell.argtypes = [C.c_int, C.c_int, C.c_int]
        L.rwref_flop_count_cell.restype = C.c_longlong
        L.rwref_run.argtypes = [C.POINTER(C.c_int), C.c_uint64, _PF, _PF, _PF, _F, _PF, _PF, _F,
                                C.c_int, _F, _PF, _PF, _PF, _PF, _PF, _F, _PF, _PF, _PF, _PF,
                                _PF, C.c_char_p, C.c_int]
        L.rwref_oracle.argtypes = [C.POINTER(C.c_int), _PF, _PF, _PF, _F, _F, _D, _PD, _PD,
                                   _PD, _D, _PD, _PD, C.c_char_p, C.c_int]
        L.rwref_time.argtypes = [C.POINTER(C.c_int), C.c_uint64, C.c_int, C.c_int, C.c_int,
                                 _D, _D, _D, C.c_char_p, C.c_int]
        L.rwref_pointwise_forward.argtypes = [C.c_int] * 4 + [_F] * 10 + [C.c_char_p, C.c_int]
        L.rwref_pointwise_backward.argtypes = [C.c_int] * 4 + [_F] * 13 + [C.c_char_p, C.c_int]

    def _call(self, fn, *args):
        err = C.create_string_buffer(512)
        if fn(*args, err, 512) != 0:
            raise ValueError(err.value.decode())

    def pointwise_forward(self, kind, fused, zw, zr, bias, h_prev, c_prev, training=True):
        """cells.hpp:181 through the unmodified reference; returns dict of outputs."""
        H, B = h_prev.shape
        G = gate_count(kind)
        o = {"h": fmat(H, B)}
        if kind == 3:
            o["c"] = fmat(H, B)
        if training and kind in (2, 3):
            o["gates"] = fmat(G * H, B)
        if training and kind == 3:
            o["tanh_c"] = fmat(H, B)
        if training and kind == 2:
            o["zr_h"] = fmat(H, B)
        self._call(self.lib.rwref_pointwise_forward, kind, int(fused), H, B, _fp(zw), _fp(zr),
                   _fp(np.ascontiguousarray(bias, np.float32)), _fp(h_prev), _fp(c_prev), _fp(o["h"]),
                   _fp(o.get("c")), _fp(o.get("gates")), _fp(o.get("tanh_c")), _fp(o.get("zr_h")))
        return o

    def pointwise_backward(self, kind, fused, gates, tanh_c, zr_h, h_prev, c_prev, d_above, dh_carry,
                           dc_carry, db=None):
        """cells.hpp:349 through the unmodified reference; returns dict of outputs (db: in place)."""
        H, B = d_above.shape
        G = gate_count(kind)
        o = {"dgw": fmat(G * H, B), "dh_local": fmat(H, B)}
        if kind == 2:
            o["dgr"] = fmat(G * H, B)
        if kind == 3:
            o["dc_prev"] = fmat(H, B)
        self._call(self.lib.rwref_pointwise_backward, kind, int(fused), H, B, _fp(gates), _fp(tanh_c),
                   _fp(zr_h), _fp(h_prev), _fp(c_prev), _fp(d_above), _fp(dh_carry), _fp(dc_carry),
                   _fp(o["dgw"]), _fp(o.get("dgr")), _fp(o["dh_local"]), _fp(o.get("dc_prev")), _fp(db))
        return o

    @staticmethod
    def _cfg(cfg, opt_level=6, batch_steps=None, workers=None):
        s = batch_steps if batch_steps is not None else min(2, cfg.steps)
        wk = workers if workers is not None else min(os.cpu_count() or 1, 2 * cfg.layers)
        kind = getattr(cfg, "kind", 3)  # the reference's CellKind (3 = LSTM)
        arr = (C.c_int * 9)(cfg.layers, cfg.hidden, cfg.input, cfg.batch, cfg.steps,
                            opt_level, s, wk, kind)
        return arr

    def init_params(self, cfg, seed):
        G = gate_count(getattr(cfg, "kind", 3)) * cfg.hidden
        w = [fmat(G, cfg.input if l == 0 else cfg.hidden) for l in range(cfg.layers)]
        r = [fmat(G, cfg.hidden) for _ in range(cfg.layers)]
        self.lib.rwref_init_params(self._cfg(cfg), seed, _arr([_fp(a) for a in w]),
                                   _arr([_fp(a) for a in r]))
        return w, r

    def make_input(self, cfg, seed):
        x = fmat(cfg.input, cfg.batch * cfg.steps)
        self.lib.rwref_make_input(self._cfg(cfg), seed, _fp(x), None)
        return x

    def make_dy(self, cfg, seed):
        dy = fmat(cfg.hidden, cfg.batch * cfg.steps)
        self.lib.rwref_make_input(self._cfg(cfg), seed, None, _fp(dy))
        return dy

    def flop_count_cell(self, hidden, inp, batch):
        return int(self.lib.rwref_flop_count_cell(hidden, inp, batch))

    def run(self, cfg, w, r, b, x, h0=None, c0=None, dy=None, training=True, tapes=True,
            opt_level=6, workers=None):
        H, B, T, L = cfg.hidden, cfg.batch, cfg.steps, cfg.layers
        kind = getattr(cfg, "kind", 3)
        G = gate_count(kind) * H
        training = training or dy is not None
        out = {"y": fmat(H, B * T)}
        # tapes: True = every tape, "states" = h_seq / c_seq only (full-size parity runs)
        if tapes:
            out["h_seq"] = [fmat(H, B * (T + 1)) for _ in range(L)]
            if kind == 3:
                out["c_seq"] = [fmat(H, B * (T + 1)) for _ in range(L)]
            if training and tapes is True:
                out["gates_seq"] = [fmat(G, B * T) for _ in range(L)]
                out["tanh_c_seq"] = [fmat(H, B * T) for _ in range(L)]
        if dy is not None:
            if tapes is True:
                out["dgw_seq"] = [fmat(G, B * T) for _ in range(L)]
            out["dx0"] = fmat(cfg.input, B * T)
            out["dh0"] = [fmat(H, B) for _ in range(L)]
            out["dc0"] = [fmat(H, B) for _ in range(L)] if kind == 3 else []
            out["dw"] = [fmat(G, cfg.input if l == 0 else H) for l in range(L)]
            out["dr"] = [fmat(G, H) for _ in range(L)]
            out["db"] = [np.zeros(G, np.float32) for _ in range(L)]
        P = lambda k: _arr([_fp(a) for a in out[k]]) if out.get(k) else None  # noqa: E731
        Q = lambda lst: _arr([_fp(a) for a in lst]) if lst is not None else None  # noqa: E731
        err = C.create_string_buffer(512)
        rc = self.lib.rwref_run(self._cfg(cfg, opt_level, workers=workers), 0, Q(w), Q(r), Q(b),
                                _fp(x), Q(h0), Q(c0), _fp(dy), int(training), _fp(out["y"]),
                                P("h_seq"), P("c_seq"), P("gates_seq"), P("tanh_c_seq"),
                                P("dgw_seq"), _fp(out.get("dx0")), P("dh0"), P("dc0"),
                                P("dw"), P("dr"), P("db"), err, 512)
        if rc != 0:
            raise ValueError(err.value.decode())
        return out

    def oracle(self, cfg, w, r, b, x, dy=None):
        """The reference fp64 oracle (oracle.hpp) on the same float parameters."""
        H, B, T, G, L = cfg.hidden, cfg.batch, cfg.steps, 4 * cfg.hidden, cfg.layers
        f64 = lambda r_, c_: np.zeros((r_, c_), np.float64, order="F")  # noqa: E731
        out = {"y": f64(H, B * T)}
        if dy is not None:
            out["dw"] = [f64(G, cfg.input if l == 0 else H) for l in range(L)]
            out["dr"] = [f64(G, H) for _ in range(L)]
            out["db"] = [np.zeros(G, np.float64) for _ in range(L)]
            out["dx0"] = f64(cfg.input, B * T)
            out["dh0"] = [f64(H, B) for _ in range(L)]
            out["dc0"] = [f64(H, B) for _ in range(L)]
        Q = lambda lst: _arr([_fp(a) for a in lst]) if lst is not None else None  # noqa: E731
        QD = lambda k: _arr([_fp(a) for a in out[k]], _D) if k in out else None  # noqa: E731
        err = C.create_string_buffer(512)
        rc = self.lib.rwref_oracle(self._cfg(cfg), Q(w), Q(r), Q(b), _fp(x), _fp(dy),
                                   _fp(out["y"]), QD("dw"), QD("dr"), QD("db"),
                                   _fp(out.get("dx0")), QD("dh0"), QD("dc0"), err, 512)
        if rc != 0:
            raise ValueError(err.value.decode())
        return out

    def time(self, cfg, seed=42, pass_kind=2, reps=3, warmup=1, opt_level=6, workers=None,
             batch_steps=None):
        med, mean, mn = C.c_double(), C.c_double(), C.c_double()
        err = C.create_string_buffer(512)
        rc = self.lib.rwref_time(self._cfg(cfg, opt_level, batch_steps, workers), seed,
                                 pass_kind, reps, warmup, C.byref(med), C.byref(mean),
                                 C.byref(mn), err, 512)
        if rc != 0:
            raise ValueError(err.value.decode())
        return {"median_us": med.value, "mean_us": mean.value, "min_us": mn.value}
