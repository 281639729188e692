"""ctypes binding of libqsr.so (include/qsr.h). Fails loudly when the library is missing:
there is no CPU fallback anywhere in the product path."""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

LIB_PATH = Path(os.environ.get("QSR_LIB", Path(__file__).resolve().parent / "libqsr.so"))

# Status codes (qsr.h)
OK, INVALID_ARGUMENT, OUT_OF_RANGE, LOGIC_ERROR, CUDA_ERROR, OUT_OF_MEMORY, NCCL_ERROR, INTERNAL, PARSE_ERROR = range(9)


class QuasarError(RuntimeError):
    status = INTERNAL


class InvalidArgument(QuasarError, ValueError):
    """std::invalid_argument in the reference."""
    status = INVALID_ARGUMENT


class OutOfRange(QuasarError, IndexError):
    """std::out_of_range in the reference."""
    status = OUT_OF_RANGE


class LogicError(QuasarError):
    """std::logic_error in the reference (odd phase = corrupted tableau)."""
    status = LOGIC_ERROR


class CudaError(QuasarError):
    status = CUDA_ERROR


class OutOfMemory(QuasarError, MemoryError):
    status = OUT_OF_MEMORY


class QasmError(QuasarError):
    """quasar::QasmError (qasm.hpp:33-40): what() = "qasm:L:C: reason", plus .line / .column."""
    status = PARSE_ERROR

    def __init__(self, msg: str, line: int = 0, column: int = 0):
        super().__init__(msg)
        self.line, self.column = line, column


class QasmError_t(C.Structure):
    _fields_ = [("line", C.c_int), ("column", C.c_int)]


_ERRORS = {PARSE_ERROR: QasmError, INVALID_ARGUMENT: InvalidArgument, OUT_OF_RANGE: OutOfRange, LOGIC_ERROR: LogicError,
           CUDA_ERROR: CudaError, OUT_OF_MEMORY: OutOfMemory}


class Gate_t(C.Structure):
    _fields_ = [("kind", C.c_uint8), ("q0", C.c_uint32), ("q1", C.c_uint32)]


class Entry_t(C.Structure):
    _fields_ = [("qubit", C.c_uint32), ("outcome", C.c_uint8), ("deterministic", C.c_uint8)]


class Timers_t(C.Structure):
    _fields_ = [("to_seconds", C.c_double), ("t_seconds", C.c_double),
                ("cmp_seconds", C.c_double), ("ge_seconds", C.c_double)]


class Report_t(C.Structure):
    _fields_ = [("timers", Timers_t), ("gate_count", C.c_uint64), ("measure_count", C.c_uint64),
                ("probabilistic_count", C.c_uint64), ("window_count", C.c_uint64),
                ("total_seconds", C.c_double)]


class KernelProfile_t(C.Structure):  # qsr_kernel_profile
    _fields_ = [("absorb_ms", C.c_double), ("absorb_launches", C.c_uint64), ("absorb_rows", C.c_uint64),
                ("absorb_slices", C.c_uint64), ("row_words", C.c_uint64), ("total_ms", C.c_double)]


class ShardConfig_t(C.Structure):
    _fields_ = [("world", C.c_int), ("rank", C.c_int), ("device", C.c_int), ("exchange", C.c_int),
                ("nccl_id", C.POINTER(C.c_uint8))]


EXCHANGE_LOCAL, EXCHANGE_NCCL = 0, 1

GATE_DTYPE = np.dtype({"names": ["kind", "q0", "q1"], "formats": ["u1", "<u4", "<u4"],
                       "offsets": [0, 4, 8], "itemsize": 12})
ENTRY_DTYPE = np.dtype({"names": ["qubit", "outcome", "deterministic"], "formats": ["<u4", "u1", "u1"],
                        "offsets": [0, 4, 5], "itemsize": 8})
assert C.sizeof(Gate_t) == 12 and C.sizeof(Entry_t) == 8

P = C.c_void_p
u64, u32, i32, u8 = C.c_uint64, C.c_uint32, C.c_int, C.c_uint8
pu64, pi64, pu32, pu8 = C.POINTER(u64), C.POINTER(C.c_int64), C.POINTER(u32), C.POINTER(u8)
pi32, pd = C.POINTER(i32), C.POINTER(C.c_double)

# name: (restype, argtypes)
SIGNATURES = {
    "qsr_last_error": (C.c_char_p, []),
    "qsr_abi_version": (i32, []),
    "qsr_device_count": (i32, [pi32]),
    "qsr_launch_count": (u64, []),
    "qsr_release_cached_memory": (None, []),
    "qsr_host_alloc": (i32, [u64, C.POINTER(P)]),
    "qsr_host_free": (None, [P]),
    "qsr_philox_block": (None, [pu32, pu32, pu32]),
    "qsr_philox_word": (u64, [u64, u32, u32, u64]),
    "qsr_circuit_create": (i32, [u32, P, u64, C.POINTER(P)]),
    "qsr_generate_random": (i32, [u32, u32, u64, C.c_double, C.POINTER(P)]),
    "qsr_circuit_info": (i32, [P, pu32, pu64, pu64]),
    "qsr_circuit_gates": (P, [P]),
    "qsr_circuit_destroy": (None, [P]),
    "qsr_circuit_clbits": (i32, [P, pu32]),
    "qsr_circuit_set_clbits": (i32, [P, u32]),
    "qsr_set_num_threads": (None, [C.c_uint]),
    "qsr_get_num_threads": (C.c_uint, []),
    "qsr_parse_qasm": (i32, [C.c_char_p, u64, C.POINTER(P), C.POINTER(QasmError_t)]),
    "qsr_emit_qasm": (i32, [P, P, u64, pu64]),
    "qsr_schedule_text": (i32, [P, P, u64, pu64]),
    "qsr_validate_schedule": (i32, [P, P, P, u64, pu64]),
    "qsr_schedule_windows": (i32, [P, i32, C.POINTER(P)]),
    "qsr_schedule_create": (i32, [P, pu64, pu8, u64, i32, C.POINTER(P)]),
    "qsr_schedule_info": (i32, [P, pu64, pu64, pi32]),
    "qsr_schedule_gates": (P, [P]),
    "qsr_schedule_offsets": (P, [P]),
    "qsr_schedule_is_measurement": (P, [P]),
    "qsr_schedule_destroy": (None, [P]),
    "qsr_tableau_create": (i32, [u64, i32, C.POINTER(P)]),
    "qsr_tableau_basis_state": (i32, [P, pu8]),
    "qsr_tableau_info": (i32, [P, pu64, pu64, pu64, pi32]),
    "qsr_tableau_upload": (i32, [P, pu64, pu64, pu64, i32]),
    "qsr_tableau_download": (i32, [P, pu64, pu64, pu64]),
    "qsr_tableau_clone": (i32, [P, C.POINTER(P)]),
    "qsr_tableau_destroy": (None, [P]),
    "qsr_transpose_in_place": (i32, [P]),
    "qsr_tableau_check_validity": (i32, [P, P, u64, pu64]),
    "qsr_apply_window": (i32, [P, P, u64]),
    "qsr_find_probabilistic": (i32, [P, P, u64, pi64]),
    "qsr_find_and_compact_pivots": (i32, [P, u64, pi64, pu64]),
    "qsr_parallel_ge": (i32, [P, pi64, u64, u64]),
    "qsr_swap_anti_commuting": (i32, [P, u64, u64]),
    "qsr_inject_x": (i32, [P, u64]),
    "qsr_deterministic_outcome": (i32, [P, u64, pu8]),
    "qsr_measure_window": (i32, [P, P, u64, u64, pu64, P, C.POINTER(Timers_t)]),
    "qsr_measure_window_coins": (i32, [P, P, u64, pu8, u64, pu64, P, C.POINTER(Timers_t)]),
    "qsr_run_single_shot": (i32, [P, P, u64, i32, C.POINTER(P), P, C.POINTER(Report_t)]),
    "qsr_engine_create": (i32, [P, P, i32, C.POINTER(P)]),
    "qsr_engine_run": (i32, [P, u64, pd]),
    "qsr_engine_stats": (i32, [P, pd, pu64, pd, pd, pu64]),
    "qsr_engine_record": (i32, [P, P]),
    "qsr_engine_gate_bytes": (i32, [P, pd]),
    "qsr_sharded_gate_bytes": (i32, [P, pd]),
    "qsr_engine_tableau": (i32, [P, pu64, pu64, pu64]),
    "qsr_engine_profile": (i32, [P, u64, C.POINTER(KernelProfile_t)]),
    "qsr_engine_sample": (i32, [P, u64, u64, i32, i32, C.POINTER(P), pd]),
    "qsr_engine_frames_bytes": (i32, [P, pd, pd]),
    "qsr_engine_destroy": (None, [P]),
    "qsr_init_frames": (i32, [u64, u64, u64, i32, C.POINTER(P)]),
    "qsr_frames_info": (i32, [P, pu64, pu64, pu64]),
    "qsr_frames_download": (i32, [P, pu64, pu64]),
    "qsr_frames_upload": (i32, [P, pu64, pu64]),
    "qsr_apply_window_frames": (i32, [P, P, u64, i32]),
    "qsr_measure_sample": (i32, [P, P, u64, i32, u64, u32]),
    "qsr_frames_record": (i32, [P, pu64, pu32, pu64]),
    "qsr_frames_destroy": (None, [P]),
    "qsr_sample": (i32, [P, u64, u64, i32, C.POINTER(P), C.POINTER(Report_t)]),
    "qsr_sample_shard": (i32, [P, u64, u64, i32, i32, i32, C.POINTER(P), C.POINTER(Report_t)]),
    "qsr_frames_shot_words": (i32, [P, pu64, pu64]),
    "qsr_init_frames_word": (i32, [u64, u64, u64, C.c_uint, i32, C.POINTER(P)]),
    "qsr_sample_word": (i32, [P, u64, u64, C.c_uint, i32, C.POINTER(P), C.POINTER(Report_t)]),
    "qsr_frames_word_bits": (i32, [P, C.POINTER(C.c_uint)]),
    "qsr_shard_range": (i32, [u64, i32, i32, pu64, pu64]),
    "qsr_nccl_unique_id": (i32, [pu8]),
    "qsr_sharded_create": (i32, [P, P, C.POINTER(ShardConfig_t), C.POINTER(P)]),
    "qsr_sharded_run": (i32, [P, u64, pd]),
    "qsr_sharded_run_circuit": (i32, [P, C.POINTER(ShardConfig_t), u64, P, C.POINTER(P), pd]),
    "qsr_sharded_stats": (i32, [P, pd, pu64, pd, pd, pu64]),
    "qsr_sharded_record": (i32, [P, P]),
    "qsr_sharded_tableau": (i32, [P, pu64, pu64, pu64]),
    "qsr_sharded_tableau_local": (i32, [P, pu64, pu64, pu64]),
    "qsr_sharded_destroy": (None, [P]),
}


def _load() -> C.CDLL:
    if not LIB_PATH.exists():
        raise ImportError(
            f"libqsr.so not found at {LIB_PATH}: build it with `python paper_2603_14641_b200/build.py` "
            "(there is no CPU fallback)")
    lib = C.CDLL(str(LIB_PATH))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def check(status: int) -> None:
    if status != OK:
        msg = (lib.qsr_last_error() or b"").decode(errors="replace")
        raise _ERRORS.get(status, QuasarError)(msg)


def text(fn, *args) -> bytes:
    """Two-call text output convention of qsr.h (size query, then fill)."""
    n = u64()
    check(fn(*args, None, 0, C.byref(n)))
    buf = C.create_string_buffer(max(n.value, 1))
    check(fn(*args, buf, n.value, C.byref(n)))
    return buf.raw[:n.value]


def ptr(a: np.ndarray, ctype=None):
    if ctype is None:
        return C.c_void_p(a.ctypes.data)
    return a.ctypes.data_as(C.POINTER(ctype))
