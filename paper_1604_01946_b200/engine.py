"""Host-side mirror of the reference rnnwave C++ API (proj/include/rnnwave), backed by the
sm_100a library through its C-ABI.

Same names, argument meaning and error behaviour as the reference, so parity tests read like
the reference's own tests:

    LadderConfig      config.hpp:49-97   (validate() raises ValueError with the same text)
    LayerParams       params.hpp:18-25
    init_params       params.hpp:31-51   (SplitMix64 streams 2l / 2l+1, U[-1/sqrt(H), 1/sqrt(H)])
    pretranspose      params.hpp:55-61
    make_input/make_dy verify.hpp:38-44  (streams 1000 / 1001)
    Engine.forward / backward_data / weight_update   engine.hpp:82-217
    ForwardTape / ForwardResult / BackwardState / Gradients   engine.hpp:36-67
    flop_count        cells.hpp:65-68

Matrices are numpy float32 arrays in Fortran (column-major) order with shape (rows, cols),
i.e. exactly rnnwave::Matrix's memory layout. std::invalid_argument maps to ValueError and
std::runtime_error to RuntimeError.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib

_F = C.POINTER(C.c_float)

CELL_LSTM = 3
CELL_NAMES = {0: "rnn-tanh", 1: "rnn-relu", 2: "gru", 3: "lstm"}


def _fp(a):
    return None if a is None else a.ctypes.data_as(_F)


def fmat(rows: int, cols: int) -> np.ndarray:
    return np.zeros((rows, cols), dtype=np.float32, order="F")


def as_matrix(a, rows: int | None = None, cols: int | None = None) -> np.ndarray:
    a = np.asarray(a, dtype=np.float32)
    if a.ndim == 1 and rows is not None and cols is not None and a.size == rows * cols:
        a = a.reshape((rows, cols), order="F")
    return np.asfortranarray(a)


# ------------------------------------------------------------------ config / params
@dataclass
class LadderConfig:
    layers: int = 1
    hidden: int = 1
    input: int = 1
    batch: int = 1
    steps: int = 1
    kind: int = CELL_LSTM
    opt_level: int = 0
    batch_steps: int = 1
    workers: int = 1
    seed: int = 0

    def input_width(self, layer: int) -> int:
        return self.input if layer == 0 else self.hidden

    def effective_batch_steps(self) -> int:
        return 1 if self.opt_level < 5 else min(self.batch_steps, self.steps)

    def num_blocks(self) -> int:
        s = self.effective_batch_steps()
        return (self.steps + s - 1) // s

    def validate(self) -> None:
        for name in ("layers", "hidden", "input", "batch", "steps", "batch_steps", "workers"):
            v = getattr(self, name)
            if v <= 0:
                raise ValueError(f"LadderConfig: {name} must be positive, got {v}")
        if self.opt_level < 0 or self.opt_level > 6:
            raise ValueError(f"LadderConfig: opt_level must be in 0..6, got {self.opt_level}")
        if self.batch_steps > self.steps:
            raise ValueError(f"LadderConfig: batch_steps {self.batch_steps} exceeds steps {self.steps}")


def gate_count(kind: int) -> int:
    return {0: 1, 1: 1, 2: 3, 3: 4}[kind]


@dataclass
class LayerParams:
    w: np.ndarray
    r: np.ndarray
    bias: np.ndarray
    wt: np.ndarray | None = None
    rt: np.ndarray | None = None
    transposed: bool = False


_GOLDEN = np.uint64(0x9E3779B97F4A7C15)


def _mix(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def splitmix_symmetric(seed: int, stream: int, rng: float, n: int) -> np.ndarray:
    """n draws of SplitMix64 stream `stream` of `seed` mapped to U[-rng, rng] (rng.hpp:13-48)."""
    with np.errstate(over="ignore"):
        s0 = _mix(np.array([np.uint64(seed) + np.uint64(stream) * _GOLDEN], dtype=np.uint64))[0]
        idx = np.arange(1, n + 1, dtype=np.uint64)
        z = _mix(s0 + idx * _GOLDEN)
    u = (z >> np.uint64(11)).astype(np.float64) * 2.0**-53
    return ((2.0 * u - 1.0) * rng).astype(np.float32)


def init_params(cfg: LadderConfig) -> list[LayerParams]:
    cfg.validate()
    gh = gate_count(cfg.kind) * cfg.hidden
    rng = 1.0 / np.sqrt(float(cfg.hidden))
    out = []
    for l in range(cfg.layers):
        w = splitmix_symmetric(cfg.seed, 2 * l, rng, gh * cfg.input_width(l))
        r = splitmix_symmetric(cfg.seed, 2 * l + 1, rng, gh * cfg.hidden)
        out.append(LayerParams(w.reshape((gh, cfg.input_width(l)), order="F"),
                               r.reshape((gh, cfg.hidden), order="F"),
                               np.zeros(gh, np.float32)))
    return out


def pretranspose(params: list[LayerParams]) -> None:
    for p in params:
        p.wt = np.asfortranarray(p.w.T)
        p.rt = np.asfortranarray(p.r.T)
        p.transposed = True


def random_matrix(rows: int, cols: int, seed: int, stream: int) -> np.ndarray:
    return splitmix_symmetric(seed, stream, 1.0, rows * cols).reshape((rows, cols), order="F")


def make_input(cfg: LadderConfig) -> np.ndarray:
    return random_matrix(cfg.input, cfg.batch * cfg.steps, cfg.seed, 1000)


def make_dy(cfg: LadderConfig) -> np.ndarray:
    return random_matrix(cfg.hidden, cfg.batch * cfg.steps, cfg.seed, 1001)


def flop_count(kind: int, hidden: int, inp: int, batch: int) -> int:
    return 2 * gate_count(kind) * hidden * (inp + hidden) * batch


# ------------------------------------------------------------------ results
class _LazySeq:
    """Per-layer tape tensors materialised from the device on first access."""

    def __init__(self, fetch, n):
        self._fetch, self._n, self._cache = fetch, n, {}

    def __len__(self):
        return self._n

    def __getitem__(self, l):
        if l < 0:
            l += self._n
        if not 0 <= l < self._n:
            raise IndexError(l)
        if l not in self._cache:
            self._cache[l] = self._fetch(l)
        return self._cache[l]

    def __iter__(self):
        return (self[l] for l in range(self._n))


@dataclass
class ForwardTape:
    cfg: LadderConfig
    training: bool
    _engine: "Engine | None" = None
    _id: int = 0
    _x0: np.ndarray | None = None

    @property
    def x0(self) -> np.ndarray:
        return self._x0

    def _seq(self, which, rows, cols):
        eng, tid = self._engine, self._id

        def fetch(l):
            eng._require_current(tid)
            out = fmat(rows, cols)
            eng._check(eng._L.rw_get_tape(eng._ctx, which, l, _fp(out)))
            return out
        return _LazySeq(fetch, self.cfg.layers)

    @property
    def h_seq(self):
        c = self.cfg
        if "_h" not in self.__dict__:
            self.__dict__["_h"] = self._seq(_lib.RW_TAPE_H, c.hidden, c.batch * (c.steps + 1))
        return self.__dict__["_h"]

    @property
    def c_seq(self):
        c = self.cfg
        if c.kind != CELL_LSTM:  # engine.hpp:264: LSTM only
            return []
        if "_c" not in self.__dict__:
            self.__dict__["_c"] = self._seq(_lib.RW_TAPE_C, c.hidden, c.batch * (c.steps + 1))
        return self.__dict__["_c"]

    @property
    def gates_seq(self):
        c = self.cfg
        if not self.training:
            return []
        if "_g" not in self.__dict__:
            self.__dict__["_g"] = self._seq(_lib.RW_TAPE_GATES, gate_count(c.kind) * c.hidden, c.batch * c.steps)
        return self.__dict__["_g"]

    @property
    def tanh_c_seq(self):
        c = self.cfg
        if not self.training or c.kind != CELL_LSTM:
            return []
        if "_t" not in self.__dict__:
            self.__dict__["_t"] = self._seq(_lib.RW_TAPE_TANH_C, c.hidden, c.batch * c.steps)
        return self.__dict__["_t"]

    @property
    def zrh_seq(self):
        """GRU: R_n h_{t-1} per step (engine.hpp:44)."""
        c = self.cfg
        if not self.training or c.kind != 2:
            return []
        if "_z" not in self.__dict__:
            self.__dict__["_z"] = self._seq(_lib.RW_TAPE_ZRH, c.hidden, c.batch * c.steps)
        return self.__dict__["_z"]


@dataclass
class TraceRecord:
    """sched::TraceRecord (scheduler.hpp:180-192); phase "INPUT_GEMM" | "RECURRENT_STEP"."""
    task_id: int
    layer: int
    block: int
    step_k: int
    phase: str
    worker: int
    start_ns: int
    end_ns: int


@dataclass
class ForwardResult:
    y: np.ndarray
    tape: ForwardTape


@dataclass
class BackwardState:
    dx0: np.ndarray
    dh0: list
    dc0: list
    _engine: "Engine | None" = None
    _id: int = 0

    def _dseq(self, which):
        eng, tid, c = self._engine, self._id, self._engine.cfg

        def fetch(l):
            eng._require_current(tid)
            out = fmat(gate_count(c.kind) * c.hidden, c.batch * c.steps)
            eng._check(eng._L.rw_get_tape(eng._ctx, which, l, _fp(out)))
            return out
        return _LazySeq(fetch, c.layers)

    @property
    def dgw_seq(self):
        if "_dg" not in self.__dict__:
            self.__dict__["_dg"] = self._dseq(_lib.RW_TAPE_DGW)
        return self.__dict__["_dg"]

    @property
    def dgr_seq(self):
        """GRU: the R-side gate gradients (engine.hpp:57); empty for LSTM / RNN."""
        if self._engine.cfg.kind != 2:
            return []
        if "_dr" not in self.__dict__:
            self.__dict__["_dr"] = self._dseq(_lib.RW_TAPE_DGR)
        return self.__dict__["_dr"]


@dataclass
class Gradients:
    dw: list = field(default_factory=list)
    dr: list = field(default_factory=list)
    db: list = field(default_factory=list)
    dx0: np.ndarray | None = None


# ------------------------------------------------------------------ engine
PRECISIONS = {"bf16": _lib.RW_PREC_BF16, "fp32": _lib.RW_PREC_FP32}
SCHEDULES = {"auto": _lib.RW_SCHED_AUTO, "stepwise": _lib.RW_SCHED_STEPWISE,
             "persistent": _lib.RW_SCHED_PERSISTENT, "cluster": _lib.RW_SCHED_CLUSTER,
             "layerseq": _lib.RW_SCHED_LAYERSEQ}


def nccl_unique_id() -> bytes:
    L = _lib.load()
    buf = C.create_string_buffer(128)
    if L.rw_nccl_unique_id(buf) != 0:
        raise RuntimeError(L.rw_create_error().decode() or "ncclGetUniqueId failed")
    return buf.raw


class Engine:
    """rnnwave::Engine on one B200. precision: 'fp32' (the fp32-parity split-operand mode, the
    default like the fp32 reference) or 'bf16'; schedule: 'auto' | 'stepwise' | 'persistent' |
    'cluster' | 'layerseq'. Cell kinds: LSTM on every schedule; GRU (linear before reset) and
    vanilla RNN (tanh / relu) on the cluster schedule (cells.hpp)."""

    def __init__(self, cfg: LadderConfig, precision: str = "fp32", schedule: str = "auto",
                 device: int = 0):
        self.cfg = LadderConfig(**cfg.__dict__)
        self.cfg.validate()
        if self.cfg.kind not in CELL_NAMES:
            raise ValueError(f"LadderConfig: cell kind must be 0 (rnn-tanh), 1 (rnn-relu), 2 (gru) or 3 (lstm), "
                             f"got {self.cfg.kind}")
        self.precision = precision
        self.schedule = schedule
        self._L = _lib.load()
        c = self.cfg
        rc = _lib.rw_config(c.layers, c.hidden, c.input, c.batch, c.steps, c.kind, c.opt_level,
                            c.batch_steps, c.workers, c.seed, PRECISIONS[precision],
                            SCHEDULES[schedule])
        h = C.c_void_p()
        st = self._L.rw_create(C.byref(rc), device, C.byref(h))
        if st != 0:
            msg = self._L.rw_create_error().decode()
            raise (ValueError if st == _lib.RW_EINVAL else RuntimeError)(msg)
        self._ctx = h
        self._tape_id = 0
        self._bwd_id = 0

    def __del__(self):
        ctx = getattr(self, "_ctx", None)
        if ctx:
            self._L.rw_destroy(ctx)
            self._ctx = None

    def close(self):
        self.__del__()

    def config(self) -> LadderConfig:
        return self.cfg

    def set_trace_sink(self, sink) -> None:
        """engine.hpp:79-80: when set (a list), every forward / backward_data replaces its contents
        with the pass's schedule trace -- TraceRecord(task_id, layer, block, step_k, phase,
        worker, start_ns, end_ns) per device task, ids of build_graph(L, T, 1)
        (scheduler.hpp:96-155, 180-192; rw_trace_records)."""
        self._trace_sink = sink
        self._check(self._L.rw_trace_enable(self._ctx, 1 if sink is not None else 0))

    def trace_records(self, direction: int) -> list:
        """The last pass's trace of one direction (0 forward, 1 backward)."""
        n = C.c_int()
        self._check(self._L.rw_trace_records(self._ctx, direction, None, 0, C.byref(n)))
        buf = (_lib.rw_trace_record * max(n.value, 1))()
        self._check(self._L.rw_trace_records(self._ctx, direction, buf, n.value, C.byref(n)))
        return [TraceRecord(r.task_id, r.layer, r.block, r.step_k,
                            "INPUT_GEMM" if r.phase == 0 else "RECURRENT_STEP", r.worker,
                            r.start_ns, r.end_ns) for r in buf[:n.value]]

    def _deposit_trace(self, direction: int) -> None:
        sink = getattr(self, "_trace_sink", None)
        if sink is not None:
            sink[:] = self.trace_records(direction)

    # -- plumbing
    def _check(self, status: int) -> None:
        if status == 0:
            return
        msg = self._L.rw_last_error(self._ctx).decode()
        raise (ValueError if status == _lib.RW_EINVAL else RuntimeError)(msg)

    def _require_current(self, tid: int) -> None:
        if tid != self._tape_id:
            raise ValueError("engine: stale tape, the device no longer holds this tape")

    def _check_params(self, params) -> None:
        c = self.cfg
        if len(params) != c.layers:
            raise ValueError(f"engine: expected {c.layers} layer parameter sets, got {len(params)}")
        gh = gate_count(c.kind) * c.hidden
        for l, p in enumerate(params):
            if (p.w.shape != (gh, c.input_width(l)) or p.r.shape != (gh, c.hidden)
                    or np.asarray(p.bias).size != gh):
                raise ValueError(f"engine: layer {l} parameter shapes do not match the configuration")

    def load_params_file(self, path: str):
        """Load a reference `save-params` file (param_io.hpp) into this context; returns the
        parameters (needed again by forward / backward_data, as in the reference API)."""
        from . import param_io
        h, params = param_io.load_params(path)
        param_io.check_matches(h, self.cfg)
        self.set_params(params)
        return params

    def set_params(self, params) -> None:
        self._check_params(params)
        for l, p in enumerate(params):
            w = as_matrix(p.w)
            r = as_matrix(p.r)
            b = np.ascontiguousarray(p.bias, dtype=np.float32)
            self._check(self._L.rw_set_params(self._ctx, l, _fp(w), _fp(r), _fp(b)))

    # -- reference API
    def forward(self, params, x, training: bool, h0=None, c0=None) -> ForwardResult:
        c = self.cfg
        bt = c.batch * c.steps
        x = as_matrix(x)
        if x.shape != (c.input, bt):
            raise ValueError(f"forward: x is {x.shape[0]}x{x.shape[1]}, expected {c.input}x{bt}")
        self.set_params(params)
        if c.opt_level >= 4:
            pretranspose(params)
        if h0 is not None and len(h0) != c.layers:
            raise ValueError("forward: h0 must supply one matrix per layer")
        if c0 is not None and c.kind != CELL_LSTM:
            raise ValueError("forward: c0 supplied for a cell kind without cell state")
        hs = [as_matrix(m, c.hidden, c.batch) for m in h0] if h0 is not None else None
        cs = [as_matrix(m, c.hidden, c.batch) for m in c0] if c0 is not None else None
        arr = lambda lst: (_F * c.layers)(*[_fp(a) for a in lst]) if lst is not None else None  # noqa: E731
        y = fmat(c.hidden, bt)
        tid = C.c_uint64()
        self._check(self._L.rw_forward(self._ctx, _fp(x), int(bool(training)), arr(hs), arr(cs),
                                       _fp(y), C.byref(tid)))
        self._tape_id = tid.value
        self._deposit_trace(0)
        tape = ForwardTape(LadderConfig(**c.__dict__), bool(training), self, tid.value, x.copy(order="F"))
        return ForwardResult(y, tape)

    def _check_tape(self, tape: ForwardTape) -> None:
        if not tape.training:
            raise ValueError("engine: tape was recorded without training mode")
        t, c = tape.cfg, self.cfg
        if (t.layers, t.hidden, t.input, t.batch, t.steps, t.kind) != (
                c.layers, c.hidden, c.input, c.batch, c.steps, c.kind):
            raise ValueError("engine: stale tape, network dimensions differ")
        if tape._engine is not self or tape._id != self._tape_id:
            raise ValueError("engine: stale tape, the device no longer holds this tape")

    def backward_data(self, params, tape: ForwardTape, dy) -> BackwardState:
        c = self.cfg
        self._check_params(params)
        self._check_tape(tape)
        bt = c.batch * c.steps
        dy = as_matrix(dy)
        if dy.shape != (c.hidden, bt):
            raise ValueError(f"backward_data: dy is {dy.shape[0]}x{dy.shape[1]}, expected {c.hidden}x{bt}")
        if c.opt_level >= 4:
            pretranspose(params)
        dx0 = fmat(c.input, bt)
        dh0 = [fmat(c.hidden, c.batch) for _ in range(c.layers)]
        dc0 = [fmat(c.hidden, c.batch) for _ in range(c.layers)] if c.kind == CELL_LSTM else []  # engine.hpp:318
        arr = lambda lst: (_F * c.layers)(*[_fp(a) for a in lst]) if lst else None  # noqa: E731
        self._check(self._L.rw_backward_data(self._ctx, tape._id, _fp(dy), _fp(dx0), arr(dh0), arr(dc0)))
        self._bwd_id = tape._id
        self._deposit_trace(1)
        return BackwardState(dx0, dh0, dc0, self, tape._id)

    def weight_update(self, tape: ForwardTape, state: BackwardState) -> Gradients:
        c = self.cfg
        self._check_tape(tape)
        if state._id != tape._id or len(state.dh0) != c.layers:
            raise ValueError("weight_update: backward state layer count mismatch")
        gh = gate_count(c.kind) * c.hidden
        dw = [fmat(gh, c.input_width(l)) for l in range(c.layers)]
        dr = [fmat(gh, c.hidden) for _ in range(c.layers)]
        db = [np.zeros(gh, np.float32) for _ in range(c.layers)]
        arr = lambda lst: (_F * c.layers)(*[_fp(a) for a in lst])  # noqa: E731
        self._check(self._L.rw_weight_update(self._ctx, tape._id, arr(dw), arr(dr), arr(db)))
        return Gradients(dw, dr, db, state.dx0)

    # -- device-resident timed path (bench)
    def upload_inputs(self, x, dy=None) -> None:
        x = as_matrix(x)
        dy = as_matrix(dy) if dy is not None else None
        self._check(self._L.rw_upload_inputs(self._ctx, _fp(x), _fp(dy)))

    def upload_inputs_ptr(self, x_ptr: int, dy_ptr: int) -> None:
        """rw_upload_inputs on raw (e.g. pinned) host pointers."""
        self._check(self._L.rw_upload_inputs(self._ctx, C.cast(C.c_void_p(x_ptr), _F),
                                             C.cast(C.c_void_p(dy_ptr), _F)))

    def read_outputs(self, y=None, dx0=None, dw=None, dr=None, db=None) -> None:
        arr = lambda lst: (_F * self.cfg.layers)(*[_fp(a) for a in lst]) if lst is not None else None  # noqa: E731
        self._check(self._L.rw_read_outputs(self._ctx, _fp(y), _fp(dx0), arr(dw), arr(dr), arr(db)))

    def train_step(self, x, dy, y=None, dx0=None, dw=None, dr=None, db=None) -> None:
        """rw_train_step: pipelined host round trip (outputs complete after train_wait)."""
        arr = lambda lst: (_F * self.cfg.layers)(*[_fp(a) for a in lst]) if lst is not None else None  # noqa: E731
        self._check(self._L.rw_train_step(self._ctx, _fp(x), _fp(dy), _fp(y), _fp(dx0), arr(dw), arr(dr), arr(db)))

    def train_wait(self) -> None:
        self._check(self._L.rw_train_wait(self._ctx))

    def init_comm(self, rank: int, world: int, unique_id: bytes) -> None:
        """Join the NCCL data-parallel group (one context per GPU)."""
        self._check(self._L.rw_comm_init(self._ctx, world, rank, unique_id))

    def comm_overlap(self, on: bool = True) -> None:
        """Sum each layer's gradient bucket inside the pass, overlapped (rw_comm_overlap)."""
        self._check(self._L.rw_comm_overlap(self._ctx, int(bool(on))))

    def allreduce_grads(self, stream: int | None = None) -> None:
        self._check(self._L.rw_allreduce_grads(self._ctx, C.c_void_p(stream or 0)))

    # -- layer pipeline (rw_pp_*)
    def pp_export(self, direction: int) -> bytes:
        """Descriptor of this stage's boundary ring (0: forward ring of the first layer, also its
        layer-input buffer; 1: backward ring of the last layer), to hand to the neighbour."""
        r = _lib.rw_pp_ring()
        self._check(self._L.rw_pp_export(self._ctx, direction, C.byref(r)))
        return bytes(r)

    def pp_link(self, direction: int, peer: bytes, w_next=None) -> None:
        """0: link to the next stage's forward export (h_t hand-off; w_next: the next stage's
        first-layer W as a host array -- cluster: unused; persistent / stepwise: packed into the
        top layer's backward image, None = read the next stage's live W_0 over the link);
        1: link to the previous stage's backward export."""
        r = _lib.rw_pp_ring.from_buffer_copy(peer)
        w = as_matrix(w_next) if w_next is not None else None
        self._check(self._L.rw_pp_link(self._ctx, direction, C.byref(r), _fp(w)))

    def pp_set_next_w(self, w_next) -> None:
        """rw_pp_set_next_w: after the next stage's parameters changed (persistent / stepwise:
        re-pack W_next, optionally from a new host array; cluster: a validated no-op)."""
        w = as_matrix(w_next) if w_next is not None else None
        self._check(self._L.rw_pp_set_next_w(self._ctx, _fp(w)))

    def launch_count(self, reset: bool = False) -> int:
        n = C.c_longlong()
        self._check(self._L.rw_launch_count(self._ctx, C.byref(n), int(reset)))
        return n.value

    def run_pass(self, kind: int, stream: int | None = None) -> None:
        self._check(self._L.rw_run_pass(self._ctx, kind, C.c_void_p(stream or 0)))

    def params_updated(self) -> None:
        """The device parameters changed in place: the next pass repacks them (K7)."""
        self._check(self._L.rw_params_updated(self._ctx))

    def ladder_pass(self, level: int, stream: int | None = None) -> None:
        """One inference forward pass of GPU ladder rung 0..4 (rw_ladder_pass; stepwise context)."""
        self._check(self._L.rw_ladder_pass(self._ctx, level, C.c_void_p(stream or 0)))

    def sync(self) -> None:
        self._check(self._L.rw_sync(self._ctx))

    def set_profiling(self, on: bool) -> None:
        self._check(self._L.rw_set_profiling(self._ctx, int(on)))

    def phase_times(self, reset: bool = True):
        ms = (C.c_double * 6)()
        n = (C.c_int * 6)()
        self._check(self._L.rw_phase_times(self._ctx, ms, n, 6, int(reset)))
        names = ["repack", "fwd_recurrent", "bwd_recurrent", "weight_grad_gemm", "dx0_gemm", "db_reduce"]
        return {k: (ms[i], n[i]) for i, k in enumerate(names)}

    def describe(self) -> dict:
        a, b, k1, k2 = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        self._check(self._L.rw_describe(self._ctx, C.byref(a), C.byref(b), C.byref(k1), C.byref(k2)))
        names = {1: "stepwise", 2: "persistent", 3: "cluster", 4: "layerseq"}
        pair, bn = C.c_int(), C.c_int()
        self._check(self._L.rw_describe_variants(self._ctx, C.byref(pair), C.byref(bn)))
        fmt = C.c_int()
        self._check(self._L.rw_describe_precision(self._ctx, C.byref(fmt)))
        return {"fwd_schedule": names[a.value], "bwd_schedule": names[b.value],
                "operands": {0: "bf16", 1: "tf32x3", 2: "fp16x2"}[fmt.value],
                "fwd_ksplit": k1.value, "bwd_ksplit": k2.value, "fwd_pair": pair.value & 1,
                "bwd_pair": (pair.value >> 1) & 1, "wgrad_bn": bn.value,
                "layerseq_persistent": [(pair.value >> 2) & 1, (pair.value >> 3) & 1]}
