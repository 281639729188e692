"""TEST INFRASTRUCTURE ONLY — ctypes binding of the CPU oracles (orc.h).

Two backends share one interface:
  Oracle("port")      -> oracle/liboracle.so           (plain-C restatement, qsr_oracle.c)
  Oracle("reference") -> oracle/_ref/libquasar_ref.so  (reference headers compiled unmodified)
Importable only from tests/, __graft_entry__.smoke() and bench.py's CPU legs.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path
from typing import Optional

import numpy as np

HERE = Path(__file__).resolve().parent
PATHS = {"port": HERE / "liboracle.so", "reference": HERE / "_ref" / "libquasar_ref.so"}

GATE_DTYPE = np.dtype({"names": ["kind", "q0", "q1"], "formats": ["u1", "<u4", "<u4"],
                       "offsets": [0, 4, 8], "itemsize": 12})
ENTRY_DTYPE = np.dtype({"names": ["qubit", "outcome", "deterministic"], "formats": ["<u4", "u1", "u1"],
                        "offsets": [0, 4, 5], "itemsize": 8})


class Report(C.Structure):
    _fields_ = [("to_s", C.c_double), ("t_s", C.c_double), ("cmp_s", C.c_double), ("ge_s", C.c_double),
                ("gate_count", C.c_uint64), ("measure_count", C.c_uint64),
                ("probabilistic_count", C.c_uint64), ("window_count", C.c_uint64),
                ("total_s", C.c_double)]


class OracleError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"[{status}] {msg}")
        self.status = status


class QasmFailure(Exception):
    def __init__(self, msg, line, column):
        super().__init__(msg)
        self.msg, self.line, self.column = msg, line, column


STATUS_NAMES = {1: "invalid_argument", 2: "out_of_range", 3: "logic_error", 7: "other"}


def available(kind: str) -> bool:
    return PATHS[kind].exists()


def _p(a):
    if a is None:
        return None
    if a.dtype.names == GATE_DTYPE.names and a.dtype.itemsize != 12:
        # numpy repacks structured arrays (np.concatenate drops padding): restore the ABI layout
        b = np.zeros(len(a), dtype=GATE_DTYPE)
        for f in GATE_DTYPE.names:
            b[f] = a[f]
        a = b
        _KEEP.append(b)
        del _KEEP[:-64]
    assert a.flags.c_contiguous
    return C.c_void_p(a.ctypes.data)


_KEEP: list = []


class Oracle:
    def __init__(self, kind: str = "port"):
        path = PATHS[kind]
        if not path.exists():
            raise FileNotFoundError(f"oracle library {path} not built (make -C oracle)")
        self.kind = kind
        self.lib = C.CDLL(str(path))
        self.lib.orc_last_error.restype = C.c_char_p
        self.lib.orc_name.restype = C.c_char_p
        self.lib.orc_philox_word.restype = C.c_uint64
        self.lib.orc_philox_word.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint64]
        self.lib.orc_set_threads.argtypes = [C.c_uint]
        self.lib.orc_generate_random.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, C.c_double,
                                                 C.c_void_p, C.c_uint64, C.c_void_p]

    # -- helpers
    def _chk(self, st):
        if st != 0:
            raise OracleError(STATUS_NAMES.get(st, st), (self.lib.orc_last_error() or b"").decode())

    def set_threads(self, n: int) -> None:
        self.lib.orc_set_threads(n)

    @staticmethod
    def geometry(n: int):
        k = (n + 63) // 64
        return k, 64 * k, 64 * k * 2 * k

    # -- rng
    def philox_block(self, ctr, key):
        c = (C.c_uint32 * 4)(*ctr)
        k = (C.c_uint32 * 2)(*key)
        o = (C.c_uint32 * 4)()
        self.lib.orc_philox_block(c, k, o)
        return tuple(o)

    def philox_word(self, seed, stream, ctx, index):
        return int(self.lib.orc_philox_word(seed, stream, ctx, index))

    # -- circuits
    def generate_random(self, n, depth, seed, p) -> np.ndarray:
        cnt = C.c_uint64()
        self._chk(self.lib.orc_generate_random(n, depth, seed, float(p), None, 0, C.byref(cnt)))
        out = np.zeros(cnt.value, dtype=GATE_DTYPE)
        self._chk(self.lib.orc_generate_random(n, depth, seed, float(p), _p(out), cnt.value, C.byref(cnt)))
        return out

    def schedule(self, n, gates: np.ndarray, mode=0):
        ng = len(gates)
        out = np.zeros(ng, dtype=GATE_DTYPE)
        off = np.zeros(ng + 1, dtype=np.uint64)
        fl = np.zeros(max(ng, 1), dtype=np.uint8)
        nw = C.c_uint64()
        self._chk(self.lib.orc_schedule(C.c_uint32(n), _p(gates), C.c_uint64(ng), C.c_int(mode), _p(out),
                                        _p(off), _p(fl), C.byref(nw)))
        return out, off[:nw.value + 1].copy(), fl[:nw.value].copy()

    # -- tableau
    def basis_state(self, n, bits=None):
        _, _, pw = self.geometry(n)
        x = np.zeros(pw, dtype=np.uint64)
        z = np.zeros(pw, dtype=np.uint64)
        s = np.zeros(2 * self.geometry(n)[0], dtype=np.uint64)
        b = None if bits is None else np.asarray(bits, dtype=np.uint8)
        self._chk(self.lib.orc_basis_state(C.c_uint64(n), _p(b), _p(x), _p(z), _p(s)))
        return x, z, s

    def apply_window(self, n, layout, x, z, s, gates):
        self._chk(self.lib.orc_apply_window(C.c_uint64(n), C.c_int(layout), _p(x), _p(z), _p(s),
                                            _p(gates), C.c_uint64(len(gates))))

    def transpose(self, n, layout, x, z) -> int:
        lay = C.c_int(layout)
        self._chk(self.lib.orc_transpose(C.c_uint64(n), C.byref(lay), _p(x), _p(z)))
        return lay.value

    def find_probabilistic(self, n, layout, x, z, gates):
        out = np.zeros(len(gates), dtype=np.int64)
        self._chk(self.lib.orc_find_probabilistic(C.c_uint64(n), C.c_int(layout), _p(x), _p(z), _p(gates),
                                                  C.c_uint64(len(gates)), _p(out)))
        return out

    def find_and_compact_pivots(self, n, layout, x, z, q):
        e = np.zeros(n, dtype=np.int64)
        cnt = C.c_uint64()
        self._chk(self.lib.orc_find_and_compact_pivots(C.c_uint64(n), C.c_int(layout), _p(x), _p(z),
                                                       C.c_uint64(q), _p(e), C.byref(cnt)))
        return e, cnt.value

    def parallel_ge(self, n, layout, x, z, s, entries, count, block=256):
        e = np.ascontiguousarray(entries, dtype=np.int64)
        self._chk(self.lib.orc_parallel_ge(C.c_uint64(n), C.c_int(layout), _p(x), _p(z), _p(s), _p(e),
                                           C.c_uint64(count), C.c_uint64(block)))

    def swap_anti_commuting(self, n, layout, x, z, s, p, q):
        self._chk(self.lib.orc_swap_anti_commuting(C.c_uint64(n), C.c_int(layout), _p(x), _p(z), _p(s),
                                                   C.c_uint64(p), C.c_uint64(q)))

    def inject_x(self, n, s, p):
        self._chk(self.lib.orc_inject_x(C.c_uint64(n), _p(s), C.c_uint64(p)))

    def deterministic_outcome(self, n, layout, x, z, s, q) -> bool:
        o = C.c_uint8()
        self._chk(self.lib.orc_deterministic_outcome(C.c_uint64(n), C.c_int(layout), _p(x), _p(z), _p(s),
                                                     C.c_uint64(q), C.byref(o)))
        return bool(o.value)

    def measure_window(self, n, layout, x, z, s, gates, seed, coin_index):
        out = np.zeros(len(gates), dtype=ENTRY_DTYPE)
        ci = C.c_uint64(coin_index)
        self._chk(self.lib.orc_measure_window(C.c_uint64(n), C.c_int(layout), _p(x), _p(z), _p(s), _p(gates),
                                              C.c_uint64(len(gates)), C.c_uint64(seed), C.byref(ci), _p(out)))
        return out, ci.value

    def run_single_shot(self, n, gates, seed, schedule=None):
        """Returns (x, z, s, record, report); schedule = (gates, offsets, is_meas) or None."""
        _, _, pw = self.geometry(n)
        k = self.geometry(n)[0]
        x = np.zeros(pw, dtype=np.uint64)
        z = np.zeros(pw, dtype=np.uint64)
        s = np.zeros(2 * k, dtype=np.uint64)
        nm = int(np.count_nonzero(gates["kind"] == 11))
        rec = np.zeros(max(nm, 1), dtype=ENTRY_DTYPE)
        nrec = C.c_uint64()
        rep = Report()
        if schedule is None:
            self._chk(self.lib.orc_run_single_shot(C.c_uint64(n), _p(gates), C.c_uint64(len(gates)),
                                                   C.c_uint64(seed), _p(x), _p(z), _p(s), _p(rec),
                                                   C.byref(nrec), C.byref(rep)))
        else:
            sg, off, fl = schedule
            self._chk(self.lib.orc_run_schedule(C.c_uint64(n), _p(sg), _p(off), _p(fl),
                                                C.c_uint64(len(fl)), C.c_uint64(seed), _p(x), _p(z),
                                                _p(s), _p(rec), C.byref(nrec), C.byref(rep)))
        return x, z, s, rec[:nrec.value], rep

    # -- frames
    def init_frames(self, n, shots, seed):
        kf = (shots + 63) // 64
        xf = np.zeros(n * kf, dtype=np.uint64)
        zf = np.zeros(n * kf, dtype=np.uint64)
        self._chk(self.lib.orc_init_frames(C.c_uint64(n), C.c_uint64(shots), C.c_uint64(seed), _p(xf), _p(zf)))
        return xf, zf

    def apply_window_frames(self, n, shots, xf, zf, gates):
        self._chk(self.lib.orc_apply_window_frames(C.c_uint64(n), C.c_uint64(shots), _p(xf), _p(zf),
                                                   _p(gates), C.c_uint64(len(gates))))

    def measure_sample(self, n, shots, xf, zf, gates, seed, epoch, measured, nrows, words):
        nr = C.c_uint64(nrows)
        self._chk(self.lib.orc_measure_sample(C.c_uint64(n), C.c_uint64(shots), _p(xf), _p(zf), _p(gates),
                                              C.c_uint64(len(gates)), C.c_uint64(seed), C.c_uint32(epoch),
                                              _p(measured), C.byref(nr), _p(words)))
        return nr.value

    def sample(self, n, gates, shots, seed):
        kf = (shots + 63) // 64
        measured = np.zeros(max(n, 1), dtype=np.uint32)
        words = np.zeros(max(n, 1) * kf, dtype=np.uint64)
        nr = C.c_uint64()
        rep = Report()
        self._chk(self.lib.orc_sample(C.c_uint64(n), _p(gates), C.c_uint64(len(gates)), C.c_uint64(shots),
                                      C.c_uint64(seed), _p(measured), C.byref(nr), _p(words), C.byref(rep)))
        return measured[:nr.value].copy(), words[:nr.value * kf].copy(), rep

    # -- reference-only: formats either side of the path (oracle/_ref only)
    def _need_ref(self):
        if self.kind != "reference":
            raise NotImplementedError("reference-only oracle entry point")

    def _text(self, fn, *args) -> str:
        n = C.c_uint64()
        self._chk(fn(*args, None, C.c_uint64(0), C.byref(n)))
        buf = C.create_string_buffer(max(n.value, 1))
        self._chk(fn(*args, buf, C.c_uint64(n.value), C.byref(n)))
        return buf.raw[:n.value].decode()

    def parse_qasm(self, text: str):
        """-> (num_qubits, num_clbits, gates) or raises QasmFailure(msg, line, col)."""
        self._need_ref()
        data = text.encode()
        n, ncl, cnt, line, col = C.c_uint32(), C.c_uint32(), C.c_uint64(), C.c_int(), C.c_int()
        f = self.lib.orc_ref_parse_qasm
        f.argtypes = [C.c_char_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p,
                      C.c_void_p, C.c_void_p]
        args = (data, len(data), C.byref(n), C.byref(ncl))
        st = f(*args, None, 0, C.byref(cnt), C.byref(line), C.byref(col))
        if st == 8:
            raise QasmFailure((self.lib.orc_last_error() or b"").decode(), line.value, col.value)
        self._chk(st)
        out = np.zeros(cnt.value, dtype=GATE_DTYPE)
        self._chk(f(*args, _p(out), cnt.value, C.byref(cnt), C.byref(line), C.byref(col)))
        return n.value, ncl.value, out

    def emit_qasm(self, n, gates) -> str:
        self._need_ref()
        return self._text(self.lib.orc_ref_emit_qasm, C.c_uint32(n), _p(gates), C.c_uint64(len(gates)))

    def schedule_text(self, n, gates, mode=0) -> str:
        self._need_ref()
        return self._text(self.lib.orc_ref_schedule_text, C.c_uint32(n), _p(gates), C.c_uint64(len(gates)),
                          C.c_int(mode))

    def validate_schedule(self, n, gates, sgates, offsets, is_meas) -> str:
        self._need_ref()
        off = np.ascontiguousarray(offsets, dtype=np.uint64)
        fl = np.ascontiguousarray(is_meas, dtype=np.uint8)
        return self._text(self.lib.orc_ref_validate_schedule, C.c_uint32(n), _p(gates), C.c_uint64(len(gates)),
                          _p(sgates), _p(off), _p(fl), C.c_uint64(len(fl)))

    def sample_w(self, n, gates, shots, seed, wbits):
        """sample<W>: (measured, kf, row bytes [nrows, kf*W/8]) for W in {8, 16, 32, 64}."""
        self._need_ref()
        kf64 = (shots + 63) // 64
        measured = np.zeros(max(n, 1), dtype=np.uint32)
        data = np.zeros(max(n, 1) * kf64 * 8 + 8, dtype=np.uint8)
        nr, kf = C.c_uint64(), C.c_uint64()
        self._chk(self.lib.orc_ref_sample_w(C.c_uint64(n), _p(gates), C.c_uint64(len(gates)), C.c_uint64(shots),
                                            C.c_uint64(seed), C.c_uint(wbits), _p(measured), C.byref(nr),
                                            C.byref(kf), _p(data)))
        rb = kf.value * wbits // 8
        return measured[:nr.value].copy(), kf.value, data[:nr.value * rb].reshape(nr.value, rb).copy()

    def check_validity(self, n, layout, x, z) -> str:
        self._need_ref()
        return self._text(self.lib.orc_ref_check_validity, C.c_uint64(n), C.c_int(layout), _p(x), _p(z))



def best_available() -> Optional[Oracle]:
    for kind in ("reference", "port"):
        if available(kind):
            return Oracle(kind)
    return None
