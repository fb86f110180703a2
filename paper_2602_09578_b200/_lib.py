"""ctypes binding of the C ABI declared in ``include/flexmarl/cabi.h``.

The shared library is built in-tree (``python -m paper_2602_09578_b200.build``)
into ``paper_2602_09578_b200/_native/libflexmarl_b200.so``.  There is no
fallback: if the library is missing, importing the compute API raises.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "_native" / (
    "libflexmarl_b200_debug.so" if os.environ.get("FLEXMARL_DEBUG_LIB") == "1" else "libflexmarl_b200.so")
if os.environ.get("FLEXMARL_LIB"):  # A/B measurement of a variant build (tools/variant_libs.sh)
    LIB_PATH = Path(os.environ["FLEXMARL_LIB"]).resolve()

# fm_status (cabi.h) — 1..28 are marlsim::ErrorCode + 1 (errors.hpp:10-39)
ERROR_NAMES = [
    "OK", "SchedulingInPast", "DeviceOom", "HostOom", "EmptyPool", "DuplicateKey", "KeyNotFound",
    "GetTimeout", "LayoutOutOfBounds", "EmptyList", "TableExists", "ReservedColumnName",
    "DuplicateSample", "UnknownColumn", "RecordNotFound", "CellAlreadySet", "UnknownTable",
    "NotProcessing", "BadSampleId", "UnknownWorkflow", "NoInstance", "InsufficientResources",
    "BusyGroup", "VersionMismatch", "InactiveGroup", "IncompleteBatch", "ConfigError",
    "StallDetected", "SyncTimeout",
]
FM_ERR_CUDA, FM_ERR_NCCL, FM_ERR_NO_DEVICE, FM_ERR_INVALID_ARG = 100, 101, 102, 103

PRECISION_BF16_TC = 0
PRECISION_PARITY_F64 = 1
TIER_HOST, TIER_DEVICE, TIER_PEER = 0, 1, 2


class fm_sample(C.Structure):
    _fields_ = [("prompt_off", C.c_uint64), ("response_off", C.c_uint64), ("advantage", C.c_double)]


class fm_host_sample(C.Structure):
    _fields_ = [("prompt", C.c_void_p), ("response", C.c_void_p), ("advantage", C.c_double)]


class fm_report(C.Structure):
    _fields_ = [("ticket", C.c_int64), ("tokens", C.c_int64), ("batch_size", C.c_int64),
                ("grad_norm", C.c_double), ("loss", C.c_double)]


class fm_sample_key(C.Structure):
    """GradKey of one trained sample (training.hpp:87-91)."""
    _fields_ = [("input_id", C.c_char_p), ("turns", C.c_int32), ("traj", C.c_int32), ("version", C.c_int64)]


P = C.c_void_p
I, I64, U64, D, F = C.c_int, C.c_int64, C.c_uint64, C.c_double, C.c_float
PI64, PU64, PD = C.POINTER(C.c_int64), C.POINTER(C.c_uint64), C.POINTER(C.c_double)
S = C.c_char_p

_PROTOS = {
    "fm_last_error": (S, []),
    "fm_status_name": (S, [I]),
    "fm_abi_version": (I, []),
    "fm_launch_count": (U64, []),
    "fm_agent_seed": (U64, [U64, S]),
    "fm_seeded_weights": (I, [U64, U64, U64, P, I]),
    "fm_encode_tokens": (U64, [P, U64, P]),
    "fm_ctx_create": (I, [I, C.POINTER(P)]),
    "fm_ctx_destroy": (I, [P]),
    "fm_ctx_device": (I, [P]),
    "fm_ctx_num_sms": (I, [P]),
    "fm_ctx_synchronize": (I, [P]),
    "fm_ctx_reserve": (I, [P, U64, I64, U64, U64]),
    "fm_ctx_timer_start": (I, [P]),
    "fm_ctx_timer_stop": (I, [P, PD]),
    "fm_ctx_set_kernel_timing": (I, [P, I]),
    "fm_ctx_kernel_times": (I, [P, P, P, I]),
    "fm_arena_put": (I, [P, P, U64, PU64]),
    "fm_arena_reset": (I, [P]),
    "fm_arena_used": (U64, [P]),
    "fm_agent_create": (I, [P, S, U64, U64, I, C.POINTER(P)]),
    "fm_agent_destroy": (I, [P]),
    "fm_agent_set_weights": (I, [P, P]),
    "fm_agent_read_weights": (I, [P, P]),
    "fm_agent_read_moments": (I, [P, P, P, PI64]),
    "fm_agent_read_grad": (I, [P, P]),
    "fm_agent_read_grad_f32": (I, [P, P]),
    "fm_agent_read_grad_cols": (I, [P, P, I64, P]),
    "fm_debug_gemm": (I, [P, P, P, I, I, I, I, I, P]),
    "fm_ctx_gemm2_rows": (I, [P, PI64, I]),
    "fm_agent_version": (I64, [P]),
    "fm_agent_samples_accumulated": (I64, [P]),
    "fm_agent_is_active": (I, [P]),
    "fm_train_micro_batch": (I, [P, P, I, I64, PI64]),
    "fm_train_micro_batch_host": (I, [P, P, I, I64, PI64]),
    "fm_agent_set_clip": (I, [P, F, P, I64]),
    "fm_agent_set_shard": (I, [P, I, I]),
    "fm_agent_read_logp": (I, [P, P, I64]),
    "fm_debug_read_rows": (I, [P, I64, P, P, P, P, P]),
    "fm_debug_read_positions": (I, [P, I64, P, I64, P, P]),
    "fm_agent_add_grad_keys": (I, [P, P, I]),
    "fm_agent_sync": (I, [P]),
    "fm_agent_poll_report": (I, [P, I64, C.POINTER(fm_report)]),
    "fm_apply_update": (I, [P, I64, D, D, D, D, PD, PI64]),
    "fm_apply_update_park": (I, [P, I64, D, D, D, D, PD, PI64]),
    "fm_agent_suspend": (I, [P, I, I]),
    "fm_agent_activate": (I, [P, P]),
    "fm_agent_state_checksum": (I, [P, PU64]),
    "fm_agent_migrate_export": (I, [P, P, U64, PU64]),
    "fm_agent_migrate_import": (I, [P, P, P, U64]),
    "fm_agent_migrate_import_rows": (I, [P, P, P, U64, U64, U64]),
    "fm_agent_migrate_release": (I, [P]),
    "fm_agent_share_export": (I, [P, P, U64, PU64]),
    "fm_gang_gather_state": (I, [P]),
    "fm_group_advantages": (I, [P, P, P, I, D, P]),
    "fm_comm_unique_id": (I, [P]),
    "fm_comm_create": (I, [P, P, I, I, C.POINTER(P)]),
    "fm_comm_destroy": (I, [P]),
    "fm_agent_allreduce_grad": (I, [P, P]),
    "fm_agent_set_dp_norms": (I, [P, P]),
    "fm_gang_attach": (I, [P, P, P, U64, PU64]),
    "fm_gang_attach_mode": (I, [P, P, I, P, U64, PU64]),
    "fm_gang_connect": (I, [P, P, U64]),
    "fm_gang_detach": (I, [P]),
    "fm_publish_weights": (I, [P, I, C.POINTER(P)]),
    "fm_publish_into": (I, [P, P]),
    "fm_weights_alloc": (I, [P, U64, U64, I, C.POINTER(P)]),
    "fm_weights_info": (I, [P, PI64, PU64, PU64, C.POINTER(C.c_int), PU64, C.POINTER(C.c_int)]),
    "fm_weights_get": (I, [P, P, I]),
    "fm_weights_broadcast": (I, [P, P, I]),
    "fm_weights_destroy": (I, [P]),
    "fm_generate": (I, [P, P, P, P, I, I, P, P, P, P]),
    "fm_agent_serialize": (I, [P, I64, P, U64, PU64]),
    "fm_agent_deserialize": (I, [P, I64, P, U64]),
    "fm_store_create": (I, [C.POINTER(P)]),
    "fm_store_destroy": (I, [P]),
    "fm_store_create_table": (I, [P, S, P, P, I]),
    "fm_store_insert": (I, [P, S, I64, S, I, I]),
    "fm_store_set_float": (I, [P, S, S, I, I, I64, S, D]),
    "fm_store_set_payload": (I, [P, P, S, S, I, I, I64, S, P, U64]),
    "fm_store_ready_count": (I, [P, S, I64, PU64]),
    "fm_store_record_count": (I, [P, S, PU64]),
    "fm_store_poll": (I, [P, S, I64, I64, S, S, S, P, P, PI64]),
    "fm_store_record_id": (I, [P, S, I64, S, C.c_size_t, C.POINTER(C.c_int), C.POINTER(C.c_int), PI64]),
    "fm_store_complete": (I, [P, S, P, I64]),
    "fm_store_purge_stale": (I, [P, S, I64, PU64]),
    # on-device experience table
    "fm_dtable_create": (I, [P, S, P, P, I, I64, C.POINTER(P)]),
    "fm_dtable_destroy": (I, [P]),
    "fm_dtable_insert": (I, [P, I64, I, P, P, P, P]),
    "fm_dtable_find": (I, [P, S, I, I, I64, PI64]),
    "fm_dtable_set_float": (I, [P, S, I, P, P]),
    "fm_dtable_set_payload": (I, [P, S, I64, P, U64]),
    "fm_dtable_generate": (I, [P, P, S, S, I, P, P, P, I, P]),
    "fm_dtable_release_groups": (I, [P, I, S, S, S, I, P, P, P, P, P, P, P, I, D, P, P]),
    "fm_dtable_poll": (I, [P, I64, I64, S, S, S, P, PI64, PI64, PI64]),
    "fm_train_polled": (I, [P, P, I64, I64, PI64]),
    "fm_dtable_complete": (I, [P, P, I]),
    "fm_dtable_purge_stale": (I, [P, I64, PU64]),
    "fm_dtable_purge_inputs": (I, [P, P, I, PU64]),
    "fm_dtable_drop_record": (I, [P, S, I, I, I64, C.POINTER(C.c_int)]),
    "fm_dtable_ready_count": (I, [P, I64, PU64]),
    "fm_dtable_record_count": (I, [P, PU64]),
    "fm_dtable_record": (I, [P, I64, S, C.c_size_t, C.POINTER(C.c_int), C.POINTER(C.c_int), PI64,
                             C.POINTER(C.c_int), C.POINTER(C.c_uint32)]),
    "fm_dtable_records": (I, [P, I, P, P, C.c_size_t, P, P, P]),
    "fm_dtable_read_cells": (I, [P, S, I, P, P]),
}

# every symbol the header declares (checked by tests/test_abi.py)
EXPORTED = tuple(_PROTOS)

_lib = None


class FlexMarlError(RuntimeError):
    """A non-OK fm_status; ``code`` is the status, ``name`` the marlsim ErrorCode name."""

    def __init__(self, code: int, msg: str):
        self.code = code
        self.name = ERROR_NAMES[code] if 0 <= code < len(ERROR_NAMES) else {
            FM_ERR_CUDA: "CudaError", FM_ERR_NCCL: "NcclError", FM_ERR_NO_DEVICE: "NoDevice",
            FM_ERR_INVALID_ARG: "InvalidArgument"}.get(code, f"status{code}")
        super().__init__(f"{self.name}: {msg}")


def lib() -> C.CDLL:
    """Loads the native library (raises if it was not built — no CPU fallback)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"native library missing: {LIB_PATH} (build with `python -m paper_2602_09578_b200.build`)")
        L = C.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | C.RTLD_GLOBAL)
        for name, (res, args) in _PROTOS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(status: int) -> None:
    if status != 0:
        msg = lib().fm_last_error()
        raise FlexMarlError(status, msg.decode() if msg else "")


def ptr(a) -> int:
    """Data pointer of a C-contiguous numpy array."""
    assert a.flags["C_CONTIGUOUS"], "array must be C-contiguous"
    return a.ctypes.data
