"""ctypes binding of include/gockpt.h (argument marshalling only).

Every step of the hot path runs in libgockpt.so (sm_100a kernels + the C++
runtime). This module only declares the C structs and function signatures and
loads the in-tree library; it never computes anything of the method and never
falls back to another implementation: if the library is missing, ``lib()``
raises.
"""

from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# GCK_LIB_PATH selects another build of the same library (e.g. the ASan/UBSan build of
# scripts/build_asan.sh); the default is the in-tree sm_100a build.
LIB_PATH = os.environ.get("GCK_LIB_PATH") or os.path.join(_HERE, "libgockpt.so")

ABI_VERSION = 2
PLAN_EQUAL, PLAN_BALANCED = 0, 1
K_LIMIT = 64

(OK, E_INVALID, E_PROTOCOL, E_STALE, E_NOMEM, E_CUDA, E_INCOMPLETE, E_ABORTED, E_BUSY, E_NODEVICE, E_IO,
 E_CORRUPT) = range(12)
STATUS_NAMES = ["GCK_OK", "GCK_E_INVALID", "GCK_E_PROTOCOL", "GCK_E_STALE", "GCK_E_NOMEM", "GCK_E_CUDA",
                "GCK_E_INCOMPLETE", "GCK_E_ABORTED", "GCK_E_BUSY", "GCK_E_NODEVICE", "GCK_E_IO", "GCK_E_CORRUPT"]
COPY_ENGINE, COPY_ZEROCOPY = 0, 1
REPLAY_HOST, REPLAY_GPU, REPLAY_DEFERRED, REPLAY_STREAM = 0, 1, 2, 3
STAGE_RING, STAGE_DIRECT, STAGE_BLOCKING = 0, 1, 2


class Hparams(C.Structure):
    _fields_ = [("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double), ("weight_decay", C.c_double)]


class Config(C.Structure):
    _fields_ = [("abi_version", C.c_uint32), ("device", C.c_int32), ("n", C.c_uint64),
                ("k_min", C.c_uint32), ("k_max", C.c_uint32), ("part_align", C.c_uint32),
                ("ring_slots", C.c_uint32), ("copy_mode", C.c_int32), ("chunk_bytes", C.c_uint64),
                ("zc_ctas", C.c_uint32), ("replay_mode", C.c_int32), ("replay_threads", C.c_int32),
                ("timing", C.c_int32), ("eager_replay", C.c_int32), ("staging", C.c_int32),
                ("numa_node", C.c_int32), ("stream_buffers", C.c_uint32), ("verify_drain", C.c_int32),
                ("plan", C.c_int32)]


class Tensors(C.Structure):
    _fields_ = [("master", C.c_void_p), ("exp_avg", C.c_void_p), ("exp_avg_sq", C.c_void_p),
                ("param_bf16", C.c_void_p), ("ring", C.c_void_p), ("ring_bytes", C.c_uint64)]


class StepArgs(C.Structure):
    _fields_ = [("step", C.c_uint64), ("adam_t", C.c_uint64), ("lr", C.c_double), ("grad_scale", C.c_double),
                ("skip", C.c_int32), ("grad_bf16", C.c_void_p)]


class StepRecord(C.Structure):
    _fields_ = [("b1", C.c_float), ("c1", C.c_float), ("b2", C.c_float), ("c2", C.c_float),
                ("bc1", C.c_float), ("bc2", C.c_float), ("lr", C.c_float), ("eps", C.c_float),
                ("wd", C.c_float), ("gs", C.c_float), ("skip", C.c_int32), ("_pad", C.c_uint32),
                ("t", C.c_uint64)]


class Checkpoint(C.Structure):
    _fields_ = [("step", C.c_uint64), ("n", C.c_uint64), ("master", C.c_void_p), ("exp_avg", C.c_void_p),
                ("exp_avg_sq", C.c_void_p), ("K", C.c_uint32), ("replay_pending", C.c_uint32)]


class Staged(C.Structure):
    _fields_ = [("t0", C.c_uint64), ("n", C.c_uint64), ("K", C.c_uint32), ("_pad", C.c_uint32),
                ("lo", C.c_uint64 * K_LIMIT), ("hi", C.c_uint64 * K_LIMIT),
                ("master", C.c_void_p), ("exp_avg", C.c_void_p), ("exp_avg_sq", C.c_void_p),
                ("glog", C.c_void_p * K_LIMIT)]


class Stats(C.Structure):
    _fields_ = [("sessions", C.c_uint64), ("steps", C.c_uint64), ("session_steps", C.c_uint64),
                ("d2h_bytes", C.c_uint64), ("stall_ms_total", C.c_double), ("stall_ms_max", C.c_double),
                ("kernel_ms_total", C.c_double), ("kernel_launches_timed", C.c_uint64),
                ("d2h_ms_total", C.c_double), ("last_session_stall_ms", C.c_double),
                ("last_session_d2h_ms", C.c_double), ("last_replay_ms", C.c_double), ("last_worker_ms", C.c_double),
                ("last_finalize_wait_ms", C.c_double), ("last_session_d2h_bytes", C.c_uint64),
                ("gpu_launches", C.c_uint64), ("replay_threads", C.c_int32), ("numa_node", C.c_int32),
                ("last_session_k", C.c_uint32), ("_pad2", C.c_uint32), ("auto_step_ms", C.c_double),
                ("auto_link_gbs", C.c_double), ("last_stream_wait_ms", C.c_double), ("last_verify_ms", C.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_ if not k.startswith("_")}


class SessionStep(C.Structure):
    _fields_ = [("part", C.c_uint32), ("slot", C.c_uint32), ("wait_ms", C.c_float), ("kernel_ms", C.c_float),
                ("d2h_ms", C.c_float), ("_pad", C.c_uint32), ("d2h_bytes", C.c_uint64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_ if not k.startswith("_")}


class FileHeader(C.Structure):
    _fields_ = [("magic", C.c_char * 8), ("version", C.c_uint32), ("header_bytes", C.c_uint32),
                ("step", C.c_uint64), ("adam_t", C.c_uint64), ("n", C.c_uint64), ("rank", C.c_uint32),
                ("world", C.c_uint32), ("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double),
                ("weight_decay", C.c_double), ("block_bytes", C.c_uint64), ("nblocks", C.c_uint64),
                ("table_offset", C.c_uint64), ("section_offset", C.c_uint64 * 3), ("section_bytes", C.c_uint64 * 3),
                ("table_crc", C.c_uint32), ("header_crc", C.c_uint32)]


class LogHeader(C.Structure):
    _fields_ = [("magic", C.c_char * 8), ("K", C.c_uint32), ("_pad", C.c_uint32), ("t0", C.c_uint64),
                ("lo", C.c_uint64 * K_LIMIT), ("hi", C.c_uint64 * K_LIMIT), ("rec", StepRecord * K_LIMIT),
                ("glog_offset", C.c_uint64 * K_LIMIT), ("glog_table_offset", C.c_uint64),
                ("glog_nblocks", C.c_uint64), ("glog_table_crc", C.c_uint32), ("log_crc", C.c_uint32)]


class PersistStats(C.Structure):
    _fields_ = [("bytes", C.c_uint64), ("seconds", C.c_double), ("data_seconds", C.c_double), ("gbs", C.c_double),
                ("threads", C.c_int32), ("_pad", C.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_ if not k.startswith("_")}


P = C.c_void_p
U64P = C.POINTER(C.c_uint64)

# name -> (restype, argtypes); exactly the functions include/gockpt.h declares
SIGNATURES = {
    "gck_create": (C.c_int, [C.POINTER(Config), C.POINTER(Hparams), C.POINTER(Tensors), C.POINTER(P)]),
    "gck_destroy": (C.c_int, [P]),
    "gck_begin_checkpoint": (C.c_int, [P, C.c_uint64, C.c_uint32]),
    "gck_submit": (C.c_int, [P, C.c_uint32, C.POINTER(StepArgs), P]),
    "gck_wait_drained": (C.c_int, [P]),
    "gck_grad_fence": (C.c_int, [P, P]),
    "gck_get_staged": (C.c_int, [P, C.POINTER(Staged)]),
    "gck_finalize": (C.c_int, [P, C.POINTER(Checkpoint)]),
    "gck_finalize_poll": (C.c_int, [P, C.POINTER(Checkpoint)]),
    "gck_release": (C.c_int, [P]),
    "gck_sync_snapshot": (C.c_int, [P, P, P, P, P]),
    "gck_replay_gpu": (C.c_int, [P, P, P, P, P, P]),
    "gck_get_stats": (C.c_int, [P, C.POINTER(Stats)]),
    "gck_get_session_steps": (C.c_int, [P, C.POINTER(SessionStep), C.c_uint32, C.POINTER(C.c_uint32)]),
    "gck_last_error": (C.c_char_p, [P]),
    "gck_make_step_record": (C.c_int, [C.POINTER(Hparams), C.c_uint64, C.c_double, C.c_double, C.c_int32,
                                       C.POINTER(StepRecord)]),
    "gck_plan_parts": (C.c_int, [C.c_uint64, C.c_uint32, C.c_uint32, U64P]),
    "gck_plan_parts_mode": (C.c_int, [C.c_uint64, C.c_uint32, C.c_uint32, C.c_int32, U64P]),
    "gck_replay_host": (C.c_int, [C.POINTER(StepRecord), C.c_uint32, U64P, C.c_uint64, P, P, P,
                                  C.POINTER(P), C.c_int32]),
    "gck_replay_device": (C.c_int, [C.POINTER(StepRecord), C.c_uint32, U64P, C.c_uint64, P, P, P,
                                    C.POINTER(P), P]),
    "gck_adamw_step": (C.c_int, [C.POINTER(StepRecord), C.c_uint64, P, P, P, P, P, P]),
    "gck_h_generate": (C.c_int, [C.c_int32, C.c_int32, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64,
                                 C.c_uint32, P, P]),
    "gck_d2h_copy": (C.c_int, [P, P, C.c_uint64, C.c_int32, C.c_uint64, C.c_uint32, P]),
    "gck_checksum": (C.c_int, [P, C.c_uint64, C.c_int32, U64P]),
    "gck_write_checkpoint": (C.c_int, [C.c_char_p, C.POINTER(FileHeader), P, P, P, C.c_int32, C.c_char_p,
                                       C.POINTER(PersistStats)]),
    "gck_read_header": (C.c_int, [C.c_char_p, C.POINTER(FileHeader)]),
    "gck_write_checkpoint_log": (C.c_int, [C.c_char_p, C.POINTER(FileHeader), P, P, P, C.c_uint32, C.c_uint64,
                                           U64P, C.POINTER(StepRecord), C.POINTER(P), C.c_int32, C.c_char_p,
                                           C.POINTER(PersistStats)]),
    "gck_read_log_header": (C.c_int, [C.c_char_p, C.POINTER(LogHeader)]),
    "gck_load_checkpoint": (C.c_int, [C.c_char_p, C.c_uint64, P, P, P, C.c_int32, C.POINTER(FileHeader),
                                      C.POINTER(PersistStats)]),
    "gck_load_checkpoint_range": (C.c_int, [C.c_char_p, C.c_uint64, C.c_uint64, P, P, P, C.c_int32,
                                            C.POINTER(FileHeader)]),
    "gck_persist_begin": (C.c_int, [P, C.c_char_p, C.c_uint32, C.c_uint32, C.c_char_p]),
    "gck_persist_wait": (C.c_int, [P, C.POINTER(PersistStats)]),
    "gck_restore": (C.c_int, [P, C.c_char_p, P, C.POINTER(FileHeader)]),
    "gck_model_waste_fraction": (C.c_double, [C.c_double] * 5),
    "gck_model_optimal_interval": (C.c_double, [C.c_double] * 3),
    "gck_model_optimal_waste": (C.c_double, [C.c_double] * 3),
    "gck_model_stall_async_o": (C.c_double, [C.c_uint32, C.c_double]),
    "gck_model_stall_gockpt": (C.c_double, [C.c_uint32, C.c_double, C.c_double]),
    "gck_recommend_k": (C.c_int, [C.c_uint64, C.c_uint32, C.c_int32, C.c_double, C.c_double, C.c_double, C.c_uint32,
                                  C.POINTER(C.c_uint32), C.POINTER(C.c_double)]),
    "gck_ring_bytes_required": (C.c_uint64, [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                             C.c_int32]),
    "gck_device_count": (C.c_int32, []),
}

_LIB = None


class GckError(RuntimeError):
    def __init__(self, status, msg):
        self.status = status
        name = STATUS_NAMES[status] if 0 <= status < len(STATUS_NAMES) else str(status)
        super().__init__(f"{name}: {msg}")


def lib() -> C.CDLL:
    """Load the in-tree libgockpt.so (build it first with __graft_entry__.build())."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python __graft_entry__.py` / build() "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = L
    return _LIB


def check(status: int, ctx=None):
    if status != OK:
        msg = lib().gck_last_error(ctx)
        raise GckError(status, msg.decode() if msg else "")
    return status
