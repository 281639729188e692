"""Python mirror of the reference's quasar API (proj/include/quasar) on the B200 engine.

Names, argument meaning and error behaviour follow the reference so tests read like its
Catch2 suites. Everything computes through libqsr.so (CUDA, sm_100a); nothing here falls
back to the CPU. Reference citations are file:line under proj/include/quasar/.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import Iterable, List, Optional, Sequence, Tuple

import numpy as np

from . import _lib
from ._lib import (ENTRY_DTYPE, GATE_DTYPE, CudaError, InvalidArgument, LogicError,  # noqa: F401
                   OutOfRange, QasmError, QuasarError, check, lib, ptr)

__all__ = [
    "GateKind", "Gate", "Circuit", "generate_random", "ScheduleMode", "Window", "Schedule",
    "schedule_windows", "Layout", "Tableau", "RandomStream", "Philox", "MeasurementRecord",
    "PivotList", "PhaseTimers", "RunReport", "SingleShotResult", "apply_window", "measure_window",
    "find_probabilistic", "find_and_compact_pivots", "parallel_ge", "swap_anti_commuting",
    "inject_x", "deterministic_outcome", "run_single_shot", "FrameTableau", "init_frames",
    "apply_window_frames", "ShotRecord", "measure_sample", "sample", "Engine", "ShardedEngine",
    "shard_range", "nccl_unique_id", "sample_shard", "parse_qasm", "emit_qasm", "QasmError",
    "validate_schedule", "set_num_threads", "check_group_validity",
    "kStreamMeasure", "kStreamFrames", "kStreamGenerator", "kGeBlockTargets",
    "InvalidArgument", "OutOfRange", "LogicError", "CudaError", "QuasarError",
]

kStreamMeasure, kStreamFrames, kStreamGenerator = 0, 1, 2   # rng.hpp:98-100
kGeBlockTargets = 256                                       # measure.hpp:152


class GateKind(enum.IntEnum):  # circuit.hpp:29-42
    X = 0
    Y = 1
    Z = 2
    H = 3
    S = 4
    SDG = 5
    CX = 6
    CY = 7
    CZ = 8
    SWAP = 9
    ISWAP = 10
    MEASURE = 11


def gate_arity(kind: int) -> int:  # circuit.hpp:44-55
    return 2 if kind in (GateKind.CX, GateKind.CY, GateKind.CZ, GateKind.SWAP, GateKind.ISWAP) else 1


@dataclass(frozen=True)
class Gate:  # circuit.hpp:85-99
    kind: GateKind
    q0: int = 0
    q1: int = 0

    def arity(self) -> int:
        return gate_arity(self.kind)

    def is_measure(self) -> bool:
        return self.kind == GateKind.MEASURE

    def __eq__(self, o) -> bool:
        if not isinstance(o, Gate):
            return NotImplemented
        return self.kind == o.kind and self.q0 == o.q0 and (self.arity() == 1 or self.q1 == o.q1)

    def __hash__(self):
        return hash((int(self.kind), self.q0, self.q1 if self.arity() == 2 else 0))


def gates_array(gates) -> np.ndarray:
    """Sequence of Gate / (kind, q0[, q1]) tuples, or a GATE_DTYPE array -> GATE_DTYPE array."""
    if isinstance(gates, np.ndarray) and gates.dtype.names == GATE_DTYPE.names:
        if gates.dtype.itemsize == 12 and gates.dtype.fields == GATE_DTYPE.fields:
            return np.ascontiguousarray(gates)
        # numpy may repack structured arrays (e.g. np.concatenate drops the padding)
        a = np.zeros(len(gates), dtype=GATE_DTYPE)
        for f in GATE_DTYPE.names:
            a[f] = gates[f]
        return a
    gates = list(gates)
    a = np.zeros(len(gates), dtype=GATE_DTYPE)
    for i, g in enumerate(gates):
        if isinstance(g, Gate):
            a[i] = (int(g.kind), g.q0, g.q1 if g.arity() == 2 else 0)
        else:
            a[i] = (int(g[0]), g[1], g[2] if len(g) > 2 else 0)
    return a


def gates_list(a: np.ndarray) -> List[Gate]:
    return [Gate(GateKind(int(k)), int(q0), int(q1) if gate_arity(int(k)) == 2 else 0)
            for k, q0, q1 in zip(a["kind"], a["q0"], a["q1"])]


class Circuit:
    """Circuit{num_qubits, gates} (circuit.hpp:101-126). Gates are held by the native
    library (a 180k x 1000 circuit is 124 M gates)."""

    def __init__(self, num_qubits: int = 0, gates=(), *, _handle=None):
        if _handle is not None:
            self._h = _handle
        else:
            arr = gates_array(gates)
            h = C.c_void_p()
            check(lib.qsr_circuit_create(num_qubits, ptr(arr), len(arr), C.byref(h)))
            self._h = h

    def __del__(self):
        if getattr(self, "_h", None):
            lib.qsr_circuit_destroy(self._h)
            self._h = None

    def _info(self):
        nq, ng, nm = C.c_uint32(), C.c_uint64(), C.c_uint64()
        check(lib.qsr_circuit_info(self._h, C.byref(nq), C.byref(ng), C.byref(nm)))
        return nq.value, ng.value, nm.value

    @property
    def num_qubits(self) -> int:
        return self._info()[0]

    @property
    def num_clbits(self) -> int:  # circuit.hpp:103-105 (labels only; not part of ==)
        v = C.c_uint32()
        check(lib.qsr_circuit_clbits(self._h, C.byref(v)))
        return v.value

    @num_clbits.setter
    def num_clbits(self, v: int) -> None:
        check(lib.qsr_circuit_set_clbits(self._h, int(v)))

    def measure_count(self) -> int:
        return self._info()[2]

    def __len__(self) -> int:
        return self._info()[1]

    @property
    def gate_array(self) -> np.ndarray:
        """Zero-copy GATE_DTYPE view of the native gate list (valid while self lives)."""
        n = len(self)
        if n == 0:
            return np.zeros(0, dtype=GATE_DTYPE)
        p = lib.qsr_circuit_gates(self._h)
        buf = (C.c_uint8 * (12 * n)).from_address(p)
        buf._owner = self  # the view keeps the native circuit alive
        return np.frombuffer(buf, dtype=GATE_DTYPE, count=n)

    @property
    def gates(self) -> List[Gate]:
        return gates_list(self.gate_array)

    def __eq__(self, o) -> bool:
        return (self.num_qubits == o.num_qubits and len(self) == len(o)
                and bool(np.array_equal(self.gate_array, o.gate_array)))


def generate_random(n: int, depth: int, seed: int, measure_prob: float) -> Circuit:
    """generate_random (circuit.hpp:132-173), generated natively (same Philox draws)."""
    h = C.c_void_p()
    check(lib.qsr_generate_random(n, depth, seed, float(measure_prob), C.byref(h)))
    return Circuit(_handle=h)


class ScheduleMode(enum.IntEnum):  # schedule.hpp:37
    single_shot = 0
    sampling = 1


@dataclass
class Window:  # schedule.hpp:32-35
    gates: list = field(default_factory=list)
    is_measurement: bool = False

    def array(self) -> np.ndarray:
        return gates_array(self.gates)


class Schedule:
    """Schedule (schedule.hpp:39-42): flattened windows held natively."""

    def __init__(self, windows: Optional[Sequence[Window]] = None, mode=ScheduleMode.single_shot,
                 *, _handle=None):
        if _handle is not None:
            self._h = _handle
            return
        windows = list(windows or [])
        arrs = [w.array() for w in windows]
        gates = gates_array(np.concatenate(arrs)) if arrs else np.zeros(0, dtype=GATE_DTYPE)
        offsets = np.zeros(len(windows) + 1, dtype=np.uint64)
        offsets[1:] = np.cumsum([len(a) for a in arrs]) if arrs else []
        flags = np.array([1 if w.is_measurement else 0 for w in windows], dtype=np.uint8)
        h = C.c_void_p()
        check(lib.qsr_schedule_create(ptr(gates), ptr(offsets, C.c_uint64), ptr(flags, C.c_uint8),
                                      len(windows), int(mode), C.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None):
            lib.qsr_schedule_destroy(self._h)
            self._h = None

    def _info(self):
        nw, ng, mode = C.c_uint64(), C.c_uint64(), C.c_int()
        check(lib.qsr_schedule_info(self._h, C.byref(nw), C.byref(ng), C.byref(mode)))
        return nw.value, ng.value, mode.value

    @property
    def mode(self) -> ScheduleMode:
        return ScheduleMode(self._info()[2])

    def arrays(self) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
        nw, ng, _ = self._info()
        if ng:
            g = np.frombuffer((C.c_uint8 * (12 * ng)).from_address(lib.qsr_schedule_gates(self._h)),
                              dtype=GATE_DTYPE, count=ng).copy()
        else:
            g = np.zeros(0, dtype=GATE_DTYPE)
        off = np.frombuffer((C.c_uint64 * (nw + 1)).from_address(lib.qsr_schedule_offsets(self._h)),
                            dtype=np.uint64).copy()
        if nw:
            fl = np.frombuffer((C.c_uint8 * nw).from_address(lib.qsr_schedule_is_measurement(self._h)),
                               dtype=np.uint8).copy()
        else:
            fl = np.zeros(0, dtype=np.uint8)
        return g, off, fl

    @property
    def windows(self) -> List[Window]:
        g, off, fl = self.arrays()
        return [Window(gates_list(g[off[w]:off[w + 1]]), bool(fl[w])) for w in range(len(fl))]

    def __len__(self):
        return self._info()[0]


def schedule_windows(circuit: Circuit, mode=ScheduleMode.single_shot) -> Schedule:
    """schedule_windows (schedule.hpp:51-137): identical windows, computed in O(G)."""
    h = C.c_void_p()
    check(lib.qsr_schedule_windows(circuit._h, int(mode), C.byref(h)))
    return Schedule(_handle=h)


def schedule_to_text(schedule: Schedule) -> str:  # schedule.hpp:235-249
    return _lib.text(lib.qsr_schedule_text, schedule._h).decode()


def validate_schedule(circuit: Circuit, schedule: Schedule) -> str:  # schedule.hpp:143-233
    return _lib.text(lib.qsr_validate_schedule, circuit._h, schedule._h).decode()


def parse_qasm(text) -> Circuit:
    """parse_qasm (qasm.hpp:159-252). Raises QasmError (with .line / .column) like the reference."""
    data = text.encode() if isinstance(text, str) else bytes(text)
    h, err = C.c_void_p(), _lib.QasmError_t()
    st = lib.qsr_parse_qasm(data, len(data), C.byref(h), C.byref(err))
    if st == _lib.PARSE_ERROR:
        raise QasmError((lib.qsr_last_error() or b"").decode(errors="replace"), err.line, err.column)
    check(st)
    return Circuit(_handle=h)


def emit_qasm(circuit: Circuit) -> str:  # qasm.hpp:254-271
    return _lib.text(lib.qsr_emit_qasm, circuit._h).decode()


def check_group_validity(t: "Tableau") -> str:  # tableau.hpp:184-213
    return t.check_group_validity()


def set_num_threads(threads: int) -> None:  # parallel.hpp:151 (host passes; 0 = hardware default)
    lib.qsr_set_num_threads(int(threads))


class Layout(enum.IntEnum):  # tableau.hpp:30
    ColumnMajor = 0
    RowMajor = 1


class Philox:  # rng.hpp:28-55
    @staticmethod
    def block(ctr: Sequence[int], key: Sequence[int]) -> Tuple[int, int, int, int]:
        c = (C.c_uint32 * 4)(*ctr)
        k = (C.c_uint32 * 2)(*key)
        o = (C.c_uint32 * 4)()
        lib.qsr_philox_block(c, k, o)
        return tuple(o)

    @staticmethod
    def word_at(seed: int, stream: int, ctx: int, index: int) -> int:
        return int(lib.qsr_philox_word(seed, stream, ctx, index))


class RandomStream:
    """RandomStream (rng.hpp:61-95); `index` is public so the engine can advance it by the
    coins a measurement window consumed."""

    def __init__(self, seed: int, stream: int, ctx: int = 0):
        self._seed, self.stream, self.ctx, self.index = seed, stream, ctx, 0

    def seed(self) -> int:
        return self._seed

    def next_word(self) -> int:
        w = Philox.word_at(self._seed, self.stream, self.ctx, self.index)
        self.index += 1
        return w

    def next_bit(self) -> int:
        return self.next_word() & 1

    def next_below(self, bound: int) -> int:
        if bound <= 1:
            return 0
        limit = (bound * ((2 ** 64 - 1) // bound)) & (2 ** 64 - 1)
        while True:
            w = self.next_word()
            if w < limit:
                return w % bound


@dataclass
class Entry:  # measure.hpp:42-46
    qubit: int
    outcome: bool
    deterministic: bool


class MeasurementRecord:  # measure.hpp:41-65
    def __init__(self, entries: Optional[List[Entry]] = None):
        self.entries: List[Entry] = list(entries or [])

    @staticmethod
    def from_array(a: np.ndarray) -> "MeasurementRecord":
        return MeasurementRecord([Entry(int(q), bool(o), bool(d))
                                  for q, o, d in zip(a["qubit"], a["outcome"], a["deterministic"])])

    def array(self) -> np.ndarray:
        a = np.zeros(len(self.entries), dtype=ENTRY_DTYPE)
        for i, e in enumerate(self.entries):
            a[i] = (e.qubit, int(e.outcome), int(e.deterministic))
        return a

    def per_qubit(self) -> List[Tuple[int, bool]]:
        out: List[Tuple[int, bool]] = []
        pos = {}
        for e in self.entries:
            if e.qubit not in pos:
                pos[e.qubit] = len(out)
                out.append((e.qubit, e.outcome))
            else:
                out[pos[e.qubit]] = (e.qubit, e.outcome)
        return out


@dataclass
class PivotList:  # measure.hpp:36-39
    entries: List[int]
    count: int


@dataclass
class PhaseTimers:  # measure.hpp:87-100 (device time from CUDA events)
    to_seconds: float = 0.0
    t_seconds: float = 0.0
    cmp_seconds: float = 0.0
    ge_seconds: float = 0.0


@dataclass
class RunReport:  # simulator.hpp:27-34
    timers: PhaseTimers = field(default_factory=PhaseTimers)
    gate_count: int = 0
    measure_count: int = 0
    probabilistic_count: int = 0
    window_count: int = 0
    total_seconds: float = 0.0

    @staticmethod
    def from_c(r: _lib.Report_t) -> "RunReport":
        t = r.timers
        return RunReport(PhaseTimers(t.to_seconds, t.t_seconds, t.cmp_seconds, t.ge_seconds),
                         r.gate_count, r.measure_count, r.probabilistic_count, r.window_count,
                         r.total_seconds)


class Tableau:
    """Device-resident Tableau<uint64_t> (tableau.hpp:62-350). Host views (x_plane(), ...)
    are downloads in the reference's storage layout."""

    w = 64

    def __init__(self, n: int, device: int = 0, *, _handle=None):
        if _handle is not None:
            self._h = _handle
        else:
            h = C.c_void_p()
            check(lib.qsr_tableau_create(n, device, C.byref(h)))
            self._h = h

    def __del__(self):
        if getattr(self, "_h", None):
            lib.qsr_tableau_destroy(self._h)
            self._h = None

    # ---- construction
    @staticmethod
    def basis_state(initstate: Sequence[bool], device: int = 0) -> "Tableau":
        t = Tableau(len(initstate), device)
        bits = np.asarray([1 if b else 0 for b in initstate], dtype=np.uint8)
        check(lib.qsr_tableau_basis_state(t._h, ptr(bits, C.c_uint8)))
        return t

    @staticmethod
    def zero_state(n: int, device: int = 0) -> "Tableau":
        t = Tableau(n, device)
        check(lib.qsr_tableau_basis_state(t._h, None))
        return t

    @staticmethod
    def from_planes(n: int, x: np.ndarray, z: np.ndarray, s: np.ndarray,
                    layout: Layout = Layout.ColumnMajor, device: int = 0) -> "Tableau":
        t = Tableau(n, device)
        t.upload(x, z, s, layout)
        return t

    def copy(self) -> "Tableau":
        h = C.c_void_p()
        check(lib.qsr_tableau_clone(self._h, C.byref(h)))
        return Tableau(0, _handle=h)

    # ---- geometry
    def _info(self):
        n, k, npad, lay = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_int()
        check(lib.qsr_tableau_info(self._h, C.byref(n), C.byref(k), C.byref(npad), C.byref(lay)))
        return n.value, k.value, npad.value, lay.value

    def num_qubits(self) -> int:
        return self._info()[0]

    def num_words(self) -> int:
        return self._info()[1]

    def padded_qubits(self) -> int:
        return self._info()[2]

    def layout(self) -> Layout:
        return Layout(self._info()[3])

    def plane_words(self) -> int:
        _, k, npad, _ = self._info()
        return npad * 2 * k

    def storage_words(self) -> int:
        return 2 * self.plane_words() + 2 * self.num_words()

    # ---- host transfer (reference storage layout)
    def planes(self) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
        pw = self.plane_words()
        x = np.empty(pw, dtype=np.uint64)
        z = np.empty(pw, dtype=np.uint64)
        s = np.empty(2 * self.num_words(), dtype=np.uint64)
        check(lib.qsr_tableau_download(self._h, ptr(x, C.c_uint64), ptr(z, C.c_uint64),
                                       ptr(s, C.c_uint64)))
        return x, z, s

    def x_plane(self) -> np.ndarray:
        return self.planes()[0]

    def z_plane(self) -> np.ndarray:
        return self.planes()[1]

    def signs(self) -> np.ndarray:
        return self.planes()[2]

    def upload(self, x, z, s, layout: Layout = Layout.ColumnMajor) -> None:
        x = np.ascontiguousarray(x, dtype=np.uint64)
        z = np.ascontiguousarray(z, dtype=np.uint64)
        s = np.ascontiguousarray(s, dtype=np.uint64)
        if x.size != self.plane_words() or z.size != self.plane_words() or s.size != 2 * self.num_words():
            raise InvalidArgument("upload: plane sizes do not match the tableau")
        check(lib.qsr_tableau_upload(self._h, ptr(x, C.c_uint64), ptr(z, C.c_uint64),
                                     ptr(s, C.c_uint64), int(layout)))

    def __eq__(self, o) -> bool:  # tableau.hpp:250-253
        if not isinstance(o, Tableau):
            return NotImplemented
        if self.num_qubits() != o.num_qubits() or self.layout() != o.layout():
            return False
        a, b = self.planes(), o.planes()
        return all(np.array_equal(u, v) for u, v in zip(a, b))

    # ---- logical views (host side, for tests / debugging)
    def _bits(self):
        n, k, npad, lay = self._info()
        x, z, s = self.planes()
        return n, k, npad, lay, x, z, s

    def get_generator(self, g: int) -> "PauliString":
        n, k, npad, lay, x, z, s = self._bits()
        if g >= 2 * n:
            raise OutOfRange("get_generator: index out of range")
        return _generator(n, k, npad, lay, x, z, s, g)

    def dump(self) -> str:
        n, k, npad, lay, x, z, s = self._bits()
        return "".join(_generator(n, k, npad, lay, x, z, s, g).str() + "\n" for g in range(2 * n))

    def sign_bit(self, g: int) -> bool:
        n, k = self.num_qubits(), self.num_words()
        s = self.signs()
        half, idx = (0, g) if g < n else (k, g - n)
        return bool((int(s[half + idx // 64]) >> (idx % 64)) & 1)

    def check_group_validity(self) -> str:  # tableau.hpp:184-213 (device kernel)
        return _lib.text(lib.qsr_tableau_check_validity, self._h).decode()

    def transpose_in_place(self) -> None:  # tableau.hpp:166-176
        check(lib.qsr_transpose_in_place(self._h))


@dataclass
class PauliString:  # tableau.hpp:34-44
    negative: bool
    paulis: str

    def str(self) -> str:
        return ("-" if self.negative else "+") + self.paulis


def _generator(n, k, npad, lay, x, z, s, g) -> PauliString:
    half, idx = (0, g) if g < n else (k, g - n)
    neg = bool((int(s[half + idx // 64]) >> (idx % 64)) & 1)
    q = np.arange(n)
    if lay == Layout.ColumnMajor:
        j = half + idx // 64
        xb = (x[q * 2 * k + j] >> np.uint64(idx % 64)) & np.uint64(1)
        zb = (z[q * 2 * k + j] >> np.uint64(idx % 64)) & np.uint64(1)
    else:
        col = g if g < n else npad + (g - n)
        xb = (x[(q // 64) * 2 * npad + col] >> (q % 64).astype(np.uint64)) & np.uint64(1)
        zb = (z[(q // 64) * 2 * npad + col] >> (q % 64).astype(np.uint64)) & np.uint64(1)
    letters = np.array(list("IXZY"))[(xb + 2 * zb).astype(np.int64)]
    return PauliString(neg, "".join(letters))


def _window_gates(window) -> Tuple[np.ndarray, bool]:
    if isinstance(window, Window):
        return window.array(), window.is_measurement
    return gates_array(window), False


def apply_window(tableau: Tableau, window: Window) -> None:
    """apply_window (gates.hpp:147-197)."""
    arr, is_meas = _window_gates(window)
    if is_meas:
        raise InvalidArgument("apply_window: window contains measurements")
    check(lib.qsr_apply_window(tableau._h, ptr(arr), len(arr)))


def find_probabilistic(t: Tableau, window: Window) -> List[int]:  # measure.hpp:104-126
    arr, _ = _window_gates(window)
    out = np.empty(len(arr), dtype=np.int64)
    check(lib.qsr_find_probabilistic(t._h, ptr(arr), len(arr), ptr(out, C.c_int64)))
    return [int(v) for v in out]


def find_and_compact_pivots(t: Tableau, q: int, scratch=None) -> PivotList:  # measure.hpp:130-150
    n = t.num_qubits()
    e = np.empty(n, dtype=np.int64)
    cnt = C.c_uint64()
    check(lib.qsr_find_and_compact_pivots(t._h, q, ptr(e, C.c_int64), C.byref(cnt)))
    return PivotList([int(v) for v in e], cnt.value)


def parallel_ge(t: Tableau, pivots: PivotList, scratch=None,
                block_targets: int = kGeBlockTargets) -> None:  # measure.hpp:161-273
    e = np.asarray(pivots.entries[:max(pivots.count, 0)], dtype=np.int64)
    if e.size == 0:
        e = np.zeros(1, dtype=np.int64)
    check(lib.qsr_parallel_ge(t._h, ptr(e, C.c_int64), pivots.count, block_targets))


def swap_anti_commuting(t: Tableau, p: int, q: int, scratch=None) -> None:  # measure.hpp:279-332
    check(lib.qsr_swap_anti_commuting(t._h, p, q))


def inject_x(t: Tableau, p: int) -> None:  # measure.hpp:335-338
    check(lib.qsr_inject_x(t._h, p))


def deterministic_outcome(t: Tableau, q: int, scratch=None) -> bool:  # measure.hpp:343-376
    o = C.c_uint8()
    check(lib.qsr_deterministic_outcome(t._h, q, C.byref(o)))
    return bool(o.value)


def measure_window(t: Tableau, window: Window, rng: RandomStream, record: MeasurementRecord,
                   scratch=None, timers: Optional[PhaseTimers] = None) -> None:
    """measure_window (measure.hpp:381-442); coins come from rng (stream kStreamMeasure)."""
    arr, is_meas = _window_gates(window)
    if not is_meas:
        raise InvalidArgument("measure_window: not a measurement window")
    out = np.zeros(len(arr), dtype=ENTRY_DTYPE)
    ct = _lib.Timers_t() if timers is not None else None
    if rng.stream == kStreamMeasure and rng.ctx == 0:
        idx = C.c_uint64(rng.index)  # coins drawn on the device at the stream's position
        check(lib.qsr_measure_window(t._h, ptr(arr), len(arr), rng.seed(), C.byref(idx), ptr(out),
                                     C.byref(ct) if ct is not None else None))
        rng.index = idx.value
    else:  # any other stream: draw the window's coins here, consume exactly what was used
        coins = np.array([Philox.word_at(rng.seed(), rng.stream, rng.ctx, rng.index + i) & 1
                          for i in range(len(arr))], dtype=np.uint8)
        used = C.c_uint64(0)
        check(lib.qsr_measure_window_coins(t._h, ptr(arr), len(arr), ptr(coins, C.c_uint8), len(coins),
                                           C.byref(used), ptr(out), C.byref(ct) if ct is not None else None))
        rng.index += used.value
    record.entries.extend(MeasurementRecord.from_array(out).entries)
    if timers is not None:
        timers.t_seconds += ct.t_seconds
        timers.cmp_seconds += ct.cmp_seconds
        timers.ge_seconds += ct.ge_seconds


@dataclass
class SingleShotResult:  # simulator.hpp:39-44
    tableau: Tableau
    record: MeasurementRecord
    report: RunReport
    record_array: Optional[np.ndarray] = None


def run_single_shot(circuit: Circuit, schedule: Optional[Schedule] = None, seed: int = 0,
                    device: int = 0) -> SingleShotResult:
    """run_single_shot<uint64_t>(circuit[, schedule], seed) (simulator.hpp:46-76)."""
    if isinstance(schedule, int) and not isinstance(schedule, Schedule):
        schedule, seed = None, schedule
    nm = circuit.measure_count()
    rec = np.zeros(max(nm, 1), dtype=ENTRY_DTYPE)
    rep = _lib.Report_t()
    h = C.c_void_p()
    check(lib.qsr_run_single_shot(circuit._h, schedule._h if schedule is not None else None,
                                  seed, device, C.byref(h), ptr(rec), C.byref(rep)))
    rec = rec[:nm]
    return SingleShotResult(Tableau(0, _handle=h), MeasurementRecord.from_array(rec),
                            RunReport.from_c(rep), rec)


class Engine:
    """Device-resident single-shot engine (the bench's `value` path): schedule uploaded once,
    every run() is a full run_single_shot on HBM-resident inputs."""

    def __init__(self, circuit: Circuit, schedule: Optional[Schedule] = None, device: int = 0):
        h = C.c_void_p()
        check(lib.qsr_engine_create(circuit._h, schedule._h if schedule is not None else None,
                                    device, C.byref(h)))
        self._h = h
        self._nm = circuit.measure_count()

    def __del__(self):
        if getattr(self, "_h", None):
            lib.qsr_engine_destroy(self._h)
            self._h = None

    def run(self, seed: int) -> float:
        ms = C.c_double()
        check(lib.qsr_engine_run(self._h, seed, C.byref(ms)))
        return ms.value

    def stats(self) -> dict:
        g, gl, t, m, l = C.c_double(), C.c_uint64(), C.c_double(), C.c_double(), C.c_uint64()
        check(lib.qsr_engine_stats(self._h, C.byref(g), C.byref(gl), C.byref(t), C.byref(m), C.byref(l)))
        b = C.c_double()
        check(lib.qsr_engine_gate_bytes(self._h, C.byref(b)))
        return {"gate_ms": g.value, "gate_launches": gl.value, "transpose_ms": t.value,
                "measure_ms": m.value, "launches": l.value, "gate_bytes": b.value}

    def record(self) -> np.ndarray:
        rec = np.zeros(max(self._nm, 1), dtype=ENTRY_DTYPE)
        check(lib.qsr_engine_record(self._h, ptr(rec)))
        return rec[:self._nm]

    def sample(self, shots: int, seed: int, record: bool = True, world: int = 1, rank: int = 0):
        """sample(circuit, shots, seed) (frames.hpp:163-204) on the resident schedule: returns
        (ShotRecord or None, device ms); world > 1: shot-word slice `rank` (sample_shard).
        record=False leaves the shot record on the device."""
        h = C.c_void_p()
        ms = C.c_double()
        check(lib.qsr_engine_sample(self._h, shots, seed, world, rank, C.byref(h), C.byref(ms)))
        f = FrameTableau(h)
        return (f.record() if record else None), ms.value

    def frames_stats(self) -> Tuple[float, float]:
        """(algorithmic bytes, device ms) of the last sample()'s frames windows."""
        b, ms = C.c_double(), C.c_double()
        check(lib.qsr_engine_frames_bytes(self._h, C.byref(b), C.byref(ms)))
        return b.value, ms.value

    def profile(self, seed: int) -> dict:
        """One extra run with CUDA events around every k_batch_absorb launch (not a timed run)."""
        p = _lib.KernelProfile_t()
        check(lib.qsr_engine_profile(self._h, seed, C.byref(p)))
        return {f: getattr(p, f) for f, _ in p._fields_}

    def tableau_planes(self, n: int) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
        k = (n + 63) // 64
        x = np.empty(64 * k * 2 * k, dtype=np.uint64)
        z = np.empty_like(x)
        s = np.empty(2 * k, dtype=np.uint64)
        check(lib.qsr_engine_tableau(self._h, ptr(x, C.c_uint64), ptr(z, C.c_uint64), ptr(s, C.c_uint64)))
        return x, z, s


# ---- generator-row-sharded engine ------------------------------------
def shard_range(n: int, world: int, rank: int) -> Tuple[int, int]:
    """Generator-word range (j0, kg) of shard `rank` of `world` for n qubits (host only)."""
    j0, kg = C.c_uint64(), C.c_uint64()
    check(lib.qsr_shard_range(n, world, rank, C.byref(j0), C.byref(kg)))
    return j0.value, kg.value


def _pin_nccl() -> None:
    """libqsr binds the NCCL already mapped into the process. Importing torch first maps
    torch's bundled NCCL, so libqsr and torch.distributed share one NCCL (loading the older
    system libnccl.so.2 first would break torch's own import later in the process)."""
    try:
        import torch  # noqa: F401
    except ImportError:
        pass


def nccl_unique_id() -> bytes:
    """ncclUniqueId (128 bytes) for the sharded engine's NCCL exchange; rank 0 creates it."""
    _pin_nccl()
    buf = (C.c_uint8 * 128)()
    check(lib.qsr_nccl_unique_id(buf))
    return bytes(buf)


class ShardedEngine:
    """run_single_shot on a tableau split by generator-words over `world` shards.

    exchange="local": all shards in this process on `device` (the multi-GPU protocol on one
    GPU). exchange="nccl": this process drives shard `rank` (one process per GPU); every rank
    passes the same 128-byte `nccl_id` and the constructor is collective."""

    def __init__(self, circuit: Circuit, world: int, device: int = 0, exchange: str = "local",
                 rank: int = 0, nccl_id: Optional[bytes] = None, schedule: Optional[Schedule] = None,
                 *, streamed_seed: Optional[int] = None):
        """streamed_seed: run_single_shot(circuit, seed) end to end at construction (the streamed
        driver, qsr_sharded_run_circuit; one shard per process) instead of building the resident
        engine; record() / tableau_planes() then read that run's result."""
        cfg = _lib.ShardConfig_t()
        cfg.world, cfg.rank, cfg.device = world, rank, device
        cfg.exchange = {"local": _lib.EXCHANGE_LOCAL, "nccl": _lib.EXCHANGE_NCCL}[exchange]
        self._id = None
        if exchange == "nccl":
            _pin_nccl()
        if nccl_id is not None:
            self._id = (C.c_uint8 * 128).from_buffer_copy(nccl_id)
            cfg.nccl_id = C.cast(self._id, C.POINTER(C.c_uint8))
        h = C.c_void_p()
        self._nm = circuit.measure_count()
        self.device_ms = None
        if streamed_seed is None:
            check(lib.qsr_sharded_create(circuit._h, schedule._h if schedule is not None else None,
                                         C.byref(cfg), C.byref(h)))
        else:
            self._streamed_record = np.zeros(max(self._nm, 1), dtype=ENTRY_DTYPE)
            ms = C.c_double()
            check(lib.qsr_sharded_run_circuit(circuit._h, C.byref(cfg), streamed_seed, ptr(self._streamed_record),
                                              C.byref(h), C.byref(ms)))
            self.device_ms = ms.value
        self._h = h
        self.n = circuit.num_qubits
        self.world, self.rank, self.exchange = world, rank, exchange

    def __del__(self):
        if getattr(self, "_h", None):
            lib.qsr_sharded_destroy(self._h)
            self._h = None

    def run(self, seed: int) -> float:
        ms = C.c_double()
        check(lib.qsr_sharded_run(self._h, seed, C.byref(ms)))
        return ms.value

    def stats(self) -> dict:
        g, gl, t, m, l = C.c_double(), C.c_uint64(), C.c_double(), C.c_double(), C.c_uint64()
        check(lib.qsr_sharded_stats(self._h, C.byref(g), C.byref(gl), C.byref(t), C.byref(m), C.byref(l)))
        b = C.c_double()
        check(lib.qsr_sharded_gate_bytes(self._h, C.byref(b)))
        return {"gate_ms": g.value, "gate_launches": gl.value, "transpose_ms": t.value,
                "measure_ms": m.value, "launches": l.value, "gate_bytes": b.value}

    def record(self) -> np.ndarray:
        rec = np.zeros(max(self._nm, 1), dtype=ENTRY_DTYPE)
        check(lib.qsr_sharded_record(self._h, ptr(rec)))
        return rec[:self._nm]

    def tableau_planes(self, x=None, z=None, s=None):
        """Reference-layout CM planes; only this process's shard columns are written (all of
        them with exchange="local"). Pass zero-filled buffers to combine ranks by XOR/OR."""
        k = (self.n + 63) // 64
        if x is None:
            x = np.zeros(64 * k * 2 * k, dtype=np.uint64)
            z = np.zeros_like(x)
            s = np.zeros(2 * k, dtype=np.uint64)
        check(lib.qsr_sharded_tableau(self._h, ptr(x, C.c_uint64), ptr(z, C.c_uint64), ptr(s, C.c_uint64)))
        return x, z, s


# ---- Pauli frames (frames.hpp:32-204) -------------------------------------------------
class FrameTableau:
    w = 64

    def __init__(self, handle):
        self._h = handle

    def __del__(self):
        if getattr(self, "_h", None):
            lib.qsr_frames_destroy(self._h)
            self._h = None

    def _info(self):
        n, shots, kf = C.c_uint64(), C.c_uint64(), C.c_uint64()
        check(lib.qsr_frames_info(self._h, C.byref(n), C.byref(shots), C.byref(kf)))
        return n.value, shots.value, kf.value

    @property
    def n(self):
        return self._info()[0]

    @property
    def shots(self):
        return self._info()[1]

    @property
    def kf(self):
        return self._info()[2]

    def index(self, q: int, j: int) -> int:
        return q * self.kf + j

    def planes(self) -> Tuple[np.ndarray, np.ndarray]:
        n, _, kf = self._info()
        xf = np.empty(n * kf, dtype=np.uint64)
        zf = np.empty(n * kf, dtype=np.uint64)
        check(lib.qsr_frames_download(self._h, ptr(xf, C.c_uint64), ptr(zf, C.c_uint64)))
        return xf, zf

    @property
    def xf(self) -> np.ndarray:
        return self.planes()[0]

    @property
    def zf(self) -> np.ndarray:
        return self.planes()[1]

    def upload(self, xf, zf) -> None:
        xf = np.ascontiguousarray(xf, dtype=np.uint64)
        zf = np.ascontiguousarray(zf, dtype=np.uint64)
        check(lib.qsr_frames_upload(self._h, ptr(xf, C.c_uint64), ptr(zf, C.c_uint64)))

    def record(self, out: Optional[np.ndarray] = None) -> "ShotRecord":
        """The ShotRecord (frames.hpp:97-107). `out`: an optional uint64 host buffer of at least
        rows x kf words (e.g. PinnedBuffer(...).array) the words are downloaded into; the
        record's `words` is then a view of it."""
        nrows = C.c_uint64()
        check(lib.qsr_frames_record(self._h, C.byref(nrows), None, None))
        _, shots, kf = self._info()
        measured = np.zeros(nrows.value, dtype=np.uint32)
        if out is not None:
            if out.dtype != np.uint64 or not out.flags.c_contiguous or out.size < nrows.value * kf:
                raise ValueError("record: out must be a contiguous uint64 array of >= rows x kf words")
            words = out[:nrows.value * kf]
        else:
            words = np.zeros(nrows.value * kf, dtype=np.uint64)
        if nrows.value:
            check(lib.qsr_frames_record(self._h, C.byref(nrows), ptr(measured, C.c_uint32),
                                        ptr(words, C.c_uint64)))
        return ShotRecord(shots, kf, [int(q) for q in measured], words)


def init_frames(n: int, shots: int, seed: int, device: int = 0, word_bits: int = 64) -> FrameTableau:
    """init_frames<W> (frames.hpp:46-72), W = word_bits; the device layout stays 64-bit words."""
    h = C.c_void_p()
    check(lib.qsr_init_frames_word(n, shots, seed, word_bits, device, C.byref(h)))
    return FrameTableau(h)


def apply_window_frames(f: FrameTableau, window: Window) -> None:
    arr, is_meas = _window_gates(window)
    check(lib.qsr_apply_window_frames(f._h, ptr(arr), len(arr), int(is_meas)))


@dataclass
class ShotRecord:  # frames.hpp:97-107
    shots: int = 0
    kf: int = 0
    measured: List[int] = field(default_factory=list)
    words: np.ndarray = field(default_factory=lambda: np.zeros(0, dtype=np.uint64))

    def bit(self, row: int, shot: int) -> bool:
        return bool((int(self.words[row * self.kf + shot // 64]) >> (shot % 64)) & 1)

    def row_bytes(self, word_bits: int = 64) -> np.ndarray:
        """[rows, ceil(shots/W)*W/8] little-endian bytes = the reference's ShotRecord<W> rows."""
        rb = -(-self.shots // word_bits) * word_bits // 8
        b = np.ascontiguousarray(self.words.astype("<u8")).view(np.uint8)
        return b.reshape(len(self.measured), self.kf * 8)[:, :rb]


def measure_sample(f: FrameTableau, window: Window, record=None, seed: int = 0, epoch: int = 1) -> None:
    """measure_sample (frames.hpp:111-158); the ShotRecord lives in the frames object
    (read it with f.record())."""
    arr, is_meas = _window_gates(window)
    check(lib.qsr_measure_sample(f._h, ptr(arr), len(arr), int(is_meas), seed, epoch))


def sample(circuit: Circuit, shots: int, seed: int, report: Optional[RunReport] = None,
           device: int = 0, word_bits: int = 64, out: Optional[np.ndarray] = None) -> ShotRecord:
    """sample<W>(circuit, shots, seed, report) (frames.hpp:163-204), W = word_bits in {8, 16, 32,
    64}. The record keeps 64-bit words; ShotRecord.row_bytes(W) gives the reference's W rows.
    `out`: optional host buffer for the record words (FrameTableau.record)."""
    h = C.c_void_p()
    rep = _lib.Report_t()
    check(lib.qsr_sample_word(circuit._h, shots, seed, word_bits, device, C.byref(h), C.byref(rep)))
    f = FrameTableau(h)
    if report is not None:
        r = RunReport.from_c(rep)
        report.__dict__.update(r.__dict__)
    return f.record(out)


class PinnedBuffer:
    """Page-locked host memory from libqsr (qsr_host_alloc): device->host downloads into it run
    at PCIe speed, where a fresh pageable numpy array costs page faults and a staged copy."""

    def __init__(self, nbytes: int, dtype=np.uint64):
        self._p = C.c_void_p()
        check(lib.qsr_host_alloc(max(int(nbytes), 8), C.byref(self._p)))
        n = max(int(nbytes), 8) // np.dtype(dtype).itemsize
        buf = (C.c_char * (n * np.dtype(dtype).itemsize)).from_address(self._p.value)
        self.array = np.frombuffer(buf, dtype=dtype, count=n)

    def __del__(self):
        if getattr(self, "_p", None) and self._p.value:
            self.array = None
            lib.qsr_host_free(self._p)
            self._p = C.c_void_p()


def sample_shard(circuit: Circuit, shots: int, seed: int, world: int, rank: int,
                 report: Optional[RunReport] = None, device: int = 0,
                 out: Optional[np.ndarray] = None) -> Tuple[int, ShotRecord]:
    """sample() sharded by shot: this rank's shot-word slice. Returns (w0, record) where the
    record's rows hold the slice's kf = nw words (global words w0 .. w0+nw-1)."""
    h = C.c_void_p()
    rep = _lib.Report_t()
    check(lib.qsr_sample_shard(circuit._h, shots, seed, world, rank, device, C.byref(h), C.byref(rep)))
    f = FrameTableau(h)
    if report is not None:
        r = RunReport.from_c(rep)
        report.__dict__.update(r.__dict__)
    j0, nw = C.c_uint64(), C.c_uint64()
    check(lib.qsr_frames_shot_words(h, C.byref(j0), C.byref(nw)))
    return j0.value, f.record(out)


def device_count() -> int:
    c = C.c_int(0)
    try:
        check(lib.qsr_device_count(C.byref(c)))
    except CudaError:
        return 0
    return c.value


def launch_count() -> int:
    return int(lib.qsr_launch_count())
