"""ctypes binding of libnucsim_b200.so (the C ABI in include/nucsim_b200.h).

The library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_2310_17739_b200/csrc``).  There is no fallback: if the
shared object is missing, importing the engine raises immediately, and any
device entry point fails loudly when no CUDA device is present.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

from .errors import FilterAssertionError, ProjectionError, QasmError, ResourceLimitError

LIB_PATH = Path(__file__).resolve().parent / "libnucsim_b200.so"
if os.environ.get("NSB_LIB_VARIANT"):  # tuning experiments: an in-tree build variant
    LIB_PATH = LIB_PATH.with_name(f"libnucsim_b200_{os.environ['NSB_LIB_VARIANT']}.so")

NSB_OK, NSB_EINVAL, NSB_EASSERT, NSB_EPROJECT, NSB_ERESOURCE, NSB_EDEVICE, NSB_EQASM = range(7)
OP_GATE, OP_MEASURE, OP_RESET, OP_BARRIER = range(4)
PLAN_EXACT = 1  # nsb_plan_create_ex flag: execute every gate
BLAS_CHAIN2, BLAS_FOUR = 1, 2
PASS_ALL = 15

OP_DTYPE = np.dtype([
    ("kind", "<i4"), ("tag", "<i4"), ("nq", "<i4"), ("cbit", "<i4"),
    ("q", "<i4", (5,)), ("src", "<i4"), ("param", "<i8"), ("payload", "<i8"),
    ("mask", "<u8"),
], align=True)
assert OP_DTYPE.itemsize == 64


class Status(ctypes.Structure):
    _fields_ = [("code", ctypes.c_int32), ("step", ctypes.c_int32),
                ("prob", ctypes.c_double), ("msg", ctypes.c_char * 256)]


class Fused(ctypes.Structure):
    _fields_ = [("ops", ctypes.c_void_p), ("n_ops", ctypes.c_int64),
                ("payloads", ctypes.POINTER(ctypes.c_double)), ("n_payload", ctypes.c_int64),
                ("gates_before", ctypes.c_int64),
                ("pass_before", ctypes.c_int64 * 4), ("pass_after", ctypes.c_int64 * 4)]


class Qasm(ctypes.Structure):
    _fields_ = [("n_qubits", ctypes.c_int32), ("n_cregs", ctypes.c_int32),
                ("ops", ctypes.c_void_p), ("n_ops", ctypes.c_int64),
                ("params", ctypes.POINTER(ctypes.c_double)), ("n_params", ctypes.c_int64),
                ("barrier_qubits", ctypes.POINTER(ctypes.c_int32)),
                ("n_barrier_qubits", ctypes.c_int64),
                ("creg_names", ctypes.c_void_p), ("creg_sizes", ctypes.POINTER(ctypes.c_int64))]


class PlanInfo(ctypes.Structure):
    _fields_ = [("n_gates", ctypes.c_int64), ("n_measures", ctypes.c_int64),
                ("n_resets", ctypes.c_int64), ("n_passes", ctypes.c_int64),
                ("n_segments", ctypes.c_int64), ("flops", ctypes.c_int64),
                ("tile_qubits", ctypes.c_int64), ("n_items", ctypes.c_int64),
                ("n_frame_gates", ctypes.c_int64), ("n_flush_gates", ctypes.c_int64),
                ("n_device_gates", ctypes.c_int64), ("n_sweeps", ctypes.c_int64),
                ("n_fused_group_ops", ctypes.c_int64), ("n_identity_gates", ctypes.c_int64),
                ("identity_error", ctypes.c_double)]


class PlanView(ctypes.Structure):
    _fields_ = [("n_qubits", ctypes.c_int32), ("tile_qubits", ctypes.c_int32),
                ("mma_ok", ctypes.c_int32), ("n_measures", ctypes.c_int32),
                ("pass_desc_bytes", ctypes.c_int32), ("group_desc_bytes", ctypes.c_int32),
                ("gate_op_bytes", ctypes.c_int32), ("tma_edges", ctypes.c_int32),
                ("n_passes", ctypes.c_int64), ("n_mma_passes", ctypes.c_int64),
                ("n_groups", ctypes.c_int64), ("n_gate_ops", ctypes.c_int64),
                ("n_matrices", ctypes.c_int64), ("n_items", ctypes.c_int64),
                ("passes", ctypes.c_void_p), ("mma_passes", ctypes.c_void_p),
                ("groups", ctypes.c_void_p), ("gate_ops", ctypes.c_void_p),
                ("matrices", ctypes.c_void_p), ("items", ctypes.c_void_p),
                ("octets", ctypes.c_int32), ("thread_bits", ctypes.c_int32)]


_P = ctypes.c_void_p
_I32, _I64, _D = ctypes.c_int32, ctypes.c_int64, ctypes.c_double
_ST = ctypes.POINTER(Status)

_SIGNATURES = {
    "nsb_gate_matrix": (ctypes.c_int, [_I32, _P, _I32, _P]),
    "nsb_fuse": (ctypes.c_int, [_P, _I64, _P, _P, _I32, _I32, ctypes.POINTER(Fused), _ST]),
    "nsb_fused_free": (None, [ctypes.POINTER(Fused)]),
    "nsb_generate_filter": (ctypes.c_int, [_I32, _P, _P, _I64, _P, _I32, _I64, _P,
                                           ctypes.POINTER(Fused),
                                           ctypes.POINTER(ctypes.POINTER(ctypes.c_double)),
                                           ctypes.POINTER(_I64), _ST]),
    "nsb_free": (None, [_P]),
    "nsb_qasm_parse": (ctypes.c_int, [ctypes.c_char_p, _I64, ctypes.POINTER(Qasm), _ST]),
    "nsb_qasm_free": (None, [ctypes.POINTER(Qasm)]),
    "nsb_device_count": (ctypes.c_int, [ctypes.POINTER(_I32)]),
    "nsb_ctx_create": (ctypes.c_int, [_I32, ctypes.POINTER(_P), _ST]),
    "nsb_ctx_destroy": (None, [_P]),
    "nsb_state_init": (ctypes.c_int, [_P, _I32, _ST]),
    "nsb_state_reset": (ctypes.c_int, [_P, _ST]),
    "nsb_state_upload": (ctypes.c_int, [_P, _P, _ST]),
    "nsb_state_download": (ctypes.c_int, [_P, _P, _ST]),
    "nsb_state_norm2": (ctypes.c_int, [_P, ctypes.POINTER(_D), _ST]),
    "nsb_apply_matrix": (ctypes.c_int, [_P, _P, _P, _I32, _ST]),
    "nsb_branch_probability": (ctypes.c_int, [_P, _I32, _I32, ctypes.POINTER(_D), _ST]),
    "nsb_project": (ctypes.c_int, [_P, _I32, _I32, _D, _ST]),
    "nsb_probabilities": (ctypes.c_int, [_P, _P, _ST]),
    "nsb_prob_chunk_sums": (ctypes.c_int, [_P, _I32, _P, _ST]),
    "nsb_probabilities_range": (ctypes.c_int, [_P, ctypes.c_uint64, ctypes.c_uint64, _P, _ST]),
    "nsb_expectation_pauli": (ctypes.c_int, [_P, _P, _P, _P, _I64, ctypes.POINTER(_D),
                                             ctypes.POINTER(_D), _ST]),
    "nsb_plan_create": (ctypes.c_int, [_P, _P, _I64, _P, _P, ctypes.POINTER(_P), _ST]),
    "nsb_plan_create_ex": (ctypes.c_int, [_P, _P, _I64, _P, _P, ctypes.c_int32,
                                          ctypes.POINTER(_P), _ST]),
    "nsb_plan_destroy": (None, [_P]),
    "nsb_plan_info_get": (ctypes.c_int, [_P, ctypes.POINTER(PlanInfo)]),
    "nsb_plan_analyze": (ctypes.c_int, [_P, _I64, _P, _P, _I32, ctypes.POINTER(PlanInfo), _P,
                                        _ST]),
    "nsb_host_plan_build": (ctypes.c_int, [_P, _I64, _P, _P, _I32, _I32, ctypes.POINTER(_P),
                                           _ST]),
    "nsb_host_plan_view": (ctypes.c_int, [_P, ctypes.POINTER(PlanView)]),
    "nsb_host_plan_free": (None, [_P]),
    "nsb_host_plan_chunk_prefix": (ctypes.c_int, [_P, _I64, _I32, _I32, ctypes.POINTER(_I32),
                                                  ctypes.POINTER(ctypes.c_uint64)]),
    "nsb_plan_run_mma": (ctypes.c_int, [_P, _P, _D, _P, _ST]),
    "nsb_plan_run_segment": (ctypes.c_int, [_P, _P, _I64, _ST]),
    "nsb_plan_run_segment_chunked": (ctypes.c_int, [_P, _P, _I64, _I32, ctypes.POINTER(_I32),
                                                    _ST]),
    "nsb_plan_segment_marker": (ctypes.c_int, [_P, _I64, ctypes.POINTER(_I32),
                                               ctypes.POINTER(_I32), ctypes.POINTER(_I32)]),
    "nsb_plan_last_timing": (ctypes.c_int, [_P, ctypes.POINTER(_D), ctypes.POINTER(_I64)]),
    "nsb_plan_p0_scale": (ctypes.c_int, [_P, ctypes.c_int32, _P]),
    "nsb_run_mma_streamed": (ctypes.c_int, [_P, _P, _I64, _P, _P, _D, _P, _P, _P, _ST]),
    "nsb_plan_run_rejection": (ctypes.c_int, [_P, _P, _P, _I64, _I64, ctypes.c_int32, _P, _P,
                                              _P, _P, _P, _ST]),
    "nsb_timer_start": (ctypes.c_int, [_P, _ST]),
    "nsb_timer_stop": (ctypes.c_int, [_P, ctypes.POINTER(_D), _ST]),
    "nsb_comm_unique_id": (ctypes.c_int, [_P, _ST]),
    "nsb_comm_init": (ctypes.c_int, [_P, _P, _I32, _I32, _ST]),
    "nsb_shard_swap": (ctypes.c_int, [_P, _I32, _I32, _I64, _ST]),
    "nsb_shard_reset": (ctypes.c_int, [_P, _ST]),
    "nsb_shard_allgather": (ctypes.c_int, [_P, _P, _I32, _P, _ST]),
    "nsb_shard_ipc_handle": (ctypes.c_int, [_P, _P, _ST]),
    "nsb_shard_open_peers": (ctypes.c_int, [_P, _P, _ST]),
    "nsb_shard_close_peers": (ctypes.c_int, [_P, _ST]),
    "nsb_shard_swap_p2p": (ctypes.c_int, [_P, _I32, _I32, _ST]),
    "nsb_shard_swap_overlap": (ctypes.c_int, [_P, _I32, _I32, _P, _I64, _I32, _I32,
                                              ctypes.POINTER(_I32), _ST]),
    "nsb_shard_swap_overlap_ce": (ctypes.c_int, [_P, _I32, _I32, _P, _I64, _I32, _I64,
                                                 ctypes.POINTER(_I32), _ST]),
}

EXPORTS = tuple(_SIGNATURES)

_lib = None


def lib() -> ctypes.CDLL:
    """The loaded library; raises if it has not been built."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                "g.build()'` (there is no CPU fallback for the gate-application path)")
        handle = ctypes.CDLL(str(LIB_PATH), mode=ctypes.RTLD_LOCAL)
        for name, (res, args) in _SIGNATURES.items():
            if os.environ.get("NSB_LIB_VARIANT") and not hasattr(handle, name):
                continue  # an older build variant (A/B timing only)
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def ptr(a: np.ndarray | None):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


def check(code: int, st: Status) -> None:
    """Map a status code onto the reference's exception types (errors.py)."""
    if code == NSB_OK:
        return
    msg = st.msg.decode(errors="replace")
    if code == NSB_EINVAL:
        raise ValueError(msg)
    if code == NSB_EASSERT:
        raise FilterAssertionError(int(st.step), float(st.prob))
    if code == NSB_EPROJECT:
        raise ProjectionError(msg)
    if code == NSB_ERESOURCE:
        raise ResourceLimitError(msg)
    if code == NSB_EQASM:
        raise QasmError(msg, int(st.step), int(st.prob))
    raise RuntimeError(f"device error: {msg}")


def device_count() -> int:
    n = _I32(0)
    lib().nsb_device_count(ctypes.byref(n))
    return int(n.value)


class Device:
    """One CUDA context + resident state (the C ABI's nsb_ctx)."""

    def __init__(self, index: int = 0):
        st = Status()
        h = _P()
        check(lib().nsb_ctx_create(index, ctypes.byref(h), ctypes.byref(st)), st)
        self.handle = h
        self.index = index

    def close(self) -> None:
        if self.handle:
            lib().nsb_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def call(self, name: str, *args) -> None:
        st = Status()
        check(getattr(lib(), name)(self.handle, *args, ctypes.byref(st)), st)


_default: dict[int, Device] = {}


def default_device() -> Device:
    """Process-wide context on the device named by NUCSIM_DEVICE (default 0)."""
    idx = int(os.environ.get("NUCSIM_DEVICE", os.environ.get("LOCAL_RANK", "0")))
    dev = _default.get(idx)
    if dev is None:
        dev = Device(idx)
        _default[idx] = dev
    return dev
