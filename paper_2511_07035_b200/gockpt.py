"""Python face of libgockpt (same names as include/gockpt.h; marshalling only).

PyTorch supplies device memory and streams; every step of the hot path runs
in the library. Host results are returned as numpy views of library-owned
pinned memory (no copy), valid until ``release()``.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib as L
from ._lib import check, lib


def _stream_ptr(stream) -> int | None:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _dptr(t) -> int | None:
    if t is None:
        return None
    if not t.is_cuda or not t.is_contiguous():
        raise ValueError("expected a contiguous CUDA tensor")
    return t.data_ptr()


def _np_view(ptr: int, n: int, dtype) -> np.ndarray:
    if n == 0:
        return np.zeros(0, dtype=dtype)
    ctype = {np.float32: C.c_float, np.uint16: C.c_uint16}[dtype]
    return np.ctypeslib.as_array((ctype * n).from_address(ptr))


def _host_ptr(a: np.ndarray, dtype) -> int:
    if a.dtype != dtype or not a.flags["C_CONTIGUOUS"]:
        raise ValueError(f"expected a contiguous {np.dtype(dtype).name} array")
    return a.ctypes.data


# ----------------------------------------------------------------------------- stateless
def make_step_record(beta1, beta2, eps, weight_decay, adam_t, lr, grad_scale=1.0, skip=False) -> L.StepRecord:
    """a0 (gck_make_step_record)."""
    hp = L.Hparams(beta1, beta2, eps, weight_decay)
    rec = L.StepRecord()
    check(lib().gck_make_step_record(C.byref(hp), adam_t, lr, grad_scale, int(skip), C.byref(rec)))
    return rec


PLANS = {"equal": L.PLAN_EQUAL, "balanced": L.PLAN_BALANCED}


def plan_parts(n: int, K: int, A: int = 1024, plan: str = "equal"):
    """a1 (gck_plan_parts_mode) -> [(lo, hi), ...]; plan "equal" or "balanced" (R17)."""
    buf = (C.c_uint64 * (2 * K))()
    check(lib().gck_plan_parts_mode(n, K, A, PLANS[plan], buf))
    return [(buf[2 * i], buf[2 * i + 1]) for i in range(K)]


def _recs_array(recs):
    arr = (L.StepRecord * len(recs))()
    for i, r in enumerate(recs):
        arr[i] = r
    return arr


def _parts_array(parts):
    buf = (C.c_uint64 * (2 * len(parts)))()
    for i, (lo, hi) in enumerate(parts):
        buf[2 * i], buf[2 * i + 1] = lo, hi
    return buf


def replay_host(recs, parts, master: np.ndarray, m: np.ndarray, v: np.ndarray, glog, threads: int = 0):
    """a5 host (gck_replay_host), in place on numpy float32 arrays; glog[i-1] uint16 arrays."""
    K = len(parts)
    gl = (C.c_void_p * max(1, K))()
    for i, g in enumerate(glog):
        gl[i] = _host_ptr(g, np.uint16)
    check(lib().gck_replay_host(_recs_array(recs), K, _parts_array(parts), len(master),
                                _host_ptr(master, np.float32), _host_ptr(m, np.float32),
                                _host_ptr(v, np.float32), gl, threads))


def replay_device(recs, parts, d_master, d_m, d_v, d_glog, stream=None):
    """a5 GPU (gck_replay_device), in place on CUDA tensors; d_glog[i-1] uint16/int16 CUDA tensors."""
    K = len(parts)
    gl = (C.c_void_p * max(1, K))()
    for i, g in enumerate(d_glog):
        gl[i] = _dptr(g)
    check(lib().gck_replay_device(_recs_array(recs), K, _parts_array(parts), d_master.numel(), _dptr(d_master),
                                  _dptr(d_m), _dptr(d_v), gl, _stream_ptr(stream)))


def adamw_step(rec, d_master, d_m, d_v, d_grad, d_param_bf16=None, stream=None):
    """a2 without a session (gck_adamw_step)."""
    check(lib().gck_adamw_step(C.byref(rec), d_master.numel(), _dptr(d_master), _dptr(d_m), _dptr(d_v),
                               _dptr(d_grad), _dptr(d_param_bf16), _stream_ptr(stream)))


def d2h_copy(dst_host, src_dev, nbytes=None, mode="ce", chunk_bytes=0, zc_ctas=0, stream=None):
    """a3 without a session (gck_d2h_copy): device tensor -> pinned host tensor, async on stream."""
    nb = nbytes if nbytes is not None else src_dev.numel() * src_dev.element_size()
    check(lib().gck_d2h_copy(dst_host.data_ptr(), _dptr(src_dev), nb,
                             {"ce": L.COPY_ENGINE, "zerocopy": L.COPY_ZEROCOPY}[mode], chunk_bytes, zc_ctas,
                             _stream_ptr(stream)))


def checksum(buf: np.ndarray, threads: int = 0) -> tuple[int, int]:
    """gck_checksum over the bytes of a contiguous host array: (A, B) of the drain verification."""
    buf = np.ascontiguousarray(buf)
    out = (C.c_uint64 * 2)()
    check(lib().gck_checksum(buf.ctypes.data if buf.nbytes else None, buf.nbytes, threads, out))
    return int(out[0]), int(out[1])


def _hdr_dict(h: L.FileHeader) -> dict:
    return {"step": h.step, "adam_t": h.adam_t, "n": h.n, "rank": h.rank, "world": h.world, "beta1": h.beta1,
            "beta2": h.beta2, "eps": h.eps, "weight_decay": h.weight_decay, "nblocks": h.nblocks,
            "block_bytes": h.block_bytes}


def write_checkpoint(path: str, master: np.ndarray, m: np.ndarray, v: np.ndarray, *, step: int, adam_t: int,
                     rank: int = 0, world: int = 1, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01,
                     threads: int = 0, meta_json: str | None = None) -> dict:
    """NEXT-1 (gck_write_checkpoint): multithreaded, CRC-protected, atomically published file."""
    h = L.FileHeader()
    h.step, h.adam_t, h.n, h.rank, h.world = step, adam_t, len(master), rank, world
    h.beta1, h.beta2, h.eps, h.weight_decay = beta1, beta2, eps, weight_decay
    st = L.PersistStats()
    check(lib().gck_write_checkpoint(path.encode(), C.byref(h), _host_ptr(master, np.float32), _host_ptr(m, np.float32),
                                     _host_ptr(v, np.float32), threads, meta_json.encode() if meta_json else None,
                                     C.byref(st)))
    return st.as_dict()


def write_checkpoint_log(path: str, master: np.ndarray, m: np.ndarray, v: np.ndarray, *, t0: int, parts, recs,
                         glog, adam_t: int, rank: int = 0, world: int = 1, beta1=0.9, beta2=0.999, eps=1e-8,
                         weight_decay=0.01, threads: int = 0, meta_json: str | None = None) -> dict:
    """NEXT-2 replay-on-restore (gck_write_checkpoint_log): a version-2 file of the captured parts
    (part i at S(t0+i-1)), the K StepRecords and the gradient slices glog[i-1] (hi_i uint16 each)."""
    K = len(parts)
    h = L.FileHeader()
    h.step, h.adam_t, h.n, h.rank, h.world = t0 + K - 1, adam_t, len(master), rank, world
    h.beta1, h.beta2, h.eps, h.weight_decay = beta1, beta2, eps, weight_decay
    gl = (C.c_void_p * max(1, K))()
    for i, g in enumerate(glog):
        gl[i] = _host_ptr(g, np.uint16)
    st = L.PersistStats()
    check(lib().gck_write_checkpoint_log(path.encode(), C.byref(h), _host_ptr(master, np.float32),
                                         _host_ptr(m, np.float32), _host_ptr(v, np.float32), K, t0,
                                         _parts_array(parts), _recs_array(recs), gl, threads,
                                         meta_json.encode() if meta_json else None, C.byref(st)))
    return st.as_dict()


def read_header(path: str) -> dict:
    h = L.FileHeader()
    check(lib().gck_read_header(path.encode(), C.byref(h)))
    d = _hdr_dict(h)
    d["version"] = h.version
    return d


def read_log_header(path: str) -> dict:
    """The replay log of a version-2 file: t0, K, parts, StepRecords, slice offsets."""
    lh = L.LogHeader()
    check(lib().gck_read_log_header(path.encode(), C.byref(lh)))
    K = lh.K
    return dict(t0=lh.t0, K=K, parts=[(lh.lo[i], lh.hi[i]) for i in range(K)], recs=[lh.rec[i] for i in range(K)],
                glog_offset=[lh.glog_offset[i] for i in range(K - 1)], glog_nblocks=lh.glog_nblocks)


def load_checkpoint(path: str, n: int, threads: int = 0):
    """NEXT-1 (gck_load_checkpoint) -> (master, m, v, header dict, stats dict); every block CRC verified."""
    out = [np.empty(n, np.float32) for _ in range(3)]
    h, st = L.FileHeader(), L.PersistStats()
    check(lib().gck_load_checkpoint(path.encode(), n, *[o.ctypes.data for o in out], threads, C.byref(h),
                                    C.byref(st)))
    return out[0], out[1], out[2], _hdr_dict(h), st.as_dict()


def load_checkpoint_range(path: str, offset: int, count: int, out=None, threads: int = 0):
    """gck_load_checkpoint_range -> (master, m, v) numpy views of `out` (3 x count float32) + header."""
    if out is None:
        out = [np.empty(count, np.float32) for _ in range(3)]
    h = L.FileHeader()
    check(lib().gck_load_checkpoint_range(path.encode(), offset, count, *[o.ctypes.data for o in out], threads,
                                          C.byref(h)))
    return out[0], out[1], out[2], _hdr_dict(h)


def recommend_k(n: int, link_gbs: float, t_step_s: float, budget: float = 1.0, k_max: int = 16, A: int = 1024,
                plan: str = "equal"):
    """NEXT-4 (gck_recommend_k) -> (K, V_max bytes); K = 0 if none fits."""
    k, vmax = C.c_uint32(0), C.c_double(0)
    st = lib().gck_recommend_k(n, A, PLANS[plan], link_gbs, t_step_s, budget, k_max, C.byref(k), C.byref(vmax))
    if st not in (L.OK, L.E_INVALID):
        check(st)
    return k.value, vmax.value


GEN_MASTER, GEN_EXP_AVG, GEN_EXP_AVG_SQ, GEN_GRAD = 1, 2, 3, 4


def h_generate(kind, out, seed, step=0, offset=0, mode=0, zero_per_256=4, stream=None):
    """Harness only: fill a CUDA tensor with the gockpt_inputs.py generator (gck_h_generate)."""
    check(lib().gck_h_generate(kind, mode, seed, step, offset, out.numel(), zero_per_256, _dptr(out),
                               _stream_ptr(stream)))


def ring_bytes_required(n: int, k_min: int, k_max: int, part_align: int = 1024, ring_slots: int = 2,
                        plan: str = "equal") -> int:
    return int(lib().gck_ring_bytes_required(n, k_min, k_max, part_align, ring_slots, PLANS[plan]))


def device_count() -> int:
    return int(lib().gck_device_count())


# ----------------------------------------------------------------------------- context
@dataclass
class HostCheckpoint:
    step: int
    master: np.ndarray
    exp_avg: np.ndarray
    exp_avg_sq: np.ndarray
    K: int = 0
    replay_pending: bool = False  # replay_mode="deferred": parts still as captured; S(T) at load


class GoCkpt:
    """One GoCkpt context over a caller-owned fp32 optimizer shard (gck_create ... gck_destroy)."""

    def __init__(self, master, exp_avg, exp_avg_sq, param_bf16=None, *, beta1=0.9, beta2=0.999, eps=1e-8,
                 weight_decay=0.01, k_min=1, k_max=8, part_align=1024, ring_slots=2, copy_mode="ce",
                 chunk_bytes=0, zc_ctas=0, replay_threads=0, timing=True, eager_replay=True, staging="ring",
                 numa_node=-1, replay_mode="host", ring=None, stream_buffers=0, verify_drain=True,
                 plan="equal"):
        n = master.numel()
        if exp_avg.numel() != n or exp_avg_sq.numel() != n or (param_bf16 is not None and param_bf16.numel() != n):
            raise ValueError("state tensors must have the same number of elements")
        self.n = n
        self._keep = (master, exp_avg, exp_avg_sq, param_bf16)
        cfg = L.Config(L.ABI_VERSION, master.device.index or 0, n, k_min, k_max, part_align, ring_slots,
                       {"ce": L.COPY_ENGINE, "zerocopy": L.COPY_ZEROCOPY}[copy_mode], chunk_bytes, zc_ctas,
                       {"host": L.REPLAY_HOST, "gpu": L.REPLAY_GPU, "deferred": L.REPLAY_DEFERRED,
                        "stream": L.REPLAY_STREAM}[replay_mode],
                       replay_threads, int(timing),
                       int(eager_replay),
                       {"ring": L.STAGE_RING, "direct": L.STAGE_DIRECT, "blocking": L.STAGE_BLOCKING}[staging],
                       numa_node, stream_buffers, int(verify_drain), PLANS[plan])
        hp = L.Hparams(beta1, beta2, eps, weight_decay)
        self.hparams = dict(beta1=beta1, beta2=beta2, eps=eps, weight_decay=weight_decay)
        # ring: an optional caller-owned uint8 CUDA tensor of >= ring_bytes_required(...) bytes
        t = L.Tensors(_dptr(master), _dptr(exp_avg), _dptr(exp_avg_sq), _dptr(param_bf16), _dptr(ring),
                      ring.numel() * ring.element_size() if ring is not None else 0)
        self._ring = ring
        ctx = C.c_void_p()
        check(lib().gck_create(C.byref(cfg), C.byref(hp), C.byref(t), C.byref(ctx)))
        self._ctx = ctx

    # -- session
    def begin_checkpoint(self, t0: int, K: int):
        check(lib().gck_begin_checkpoint(self._ctx, t0, K), self._ctx)

    def submit(self, part: int, step: int, adam_t: int, lr: float, grad, grad_scale: float = 1.0,
               skip: bool = False, stream=None) -> int:
        a = L.StepArgs(step, adam_t, lr, grad_scale, int(skip), _dptr(grad))
        st = lib().gck_submit(self._ctx, part, C.byref(a), _stream_ptr(stream))
        if st not in (L.OK,):
            check(st, self._ctx)
        return st

    def grad_fence(self, stream=None):
        """Direct staging: order `stream` after the copy-out of the last gradient slice."""
        check(lib().gck_grad_fence(self._ctx, _stream_ptr(stream)), self._ctx)

    def wait_drained(self):
        check(lib().gck_wait_drained(self._ctx), self._ctx)

    def staged(self):
        s = L.Staged()
        check(lib().gck_get_staged(self._ctx, C.byref(s)), self._ctx)
        K, n = s.K, s.n
        parts = [(s.lo[i], s.hi[i]) for i in range(K)]
        glog = [_np_view(s.glog[i], parts[i][1], np.uint16) for i in range(K - 1)]
        return dict(t0=s.t0, K=K, parts=parts, master=_np_view(s.master, n, np.float32),
                    exp_avg=_np_view(s.exp_avg, n, np.float32), exp_avg_sq=_np_view(s.exp_avg_sq, n, np.float32),
                    glog=glog)

    def finalize(self, block: bool = True) -> HostCheckpoint | None:
        ck = L.Checkpoint()
        fn = lib().gck_finalize if block else lib().gck_finalize_poll
        st = fn(self._ctx, C.byref(ck))
        if st == L.E_BUSY:
            return None
        check(st, self._ctx)
        return HostCheckpoint(ck.step, _np_view(ck.master, ck.n, np.float32),
                              _np_view(ck.exp_avg, ck.n, np.float32), _np_view(ck.exp_avg_sq, ck.n, np.float32),
                              ck.K, bool(ck.replay_pending))

    def release(self):
        check(lib().gck_release(self._ctx), self._ctx)

    # -- references / variants
    def sync_snapshot(self, stream=None):
        out = [np.empty(self.n, np.float32) for _ in range(3)]
        check(lib().gck_sync_snapshot(self._ctx, _stream_ptr(stream), *[o.ctypes.data for o in out]), self._ctx)
        return tuple(out)

    def replay_gpu(self, d_master, d_m, d_v, d_glog, stream=None):
        check(lib().gck_replay_gpu(self._ctx, _stream_ptr(stream), _dptr(d_master), _dptr(d_m), _dptr(d_v),
                                   _dptr(d_glog)), self._ctx)

    # -- NEXT-1 persistence / restore
    def persist_begin(self, path: str, rank: int = 0, world: int = 1, meta_json: str | None = None):
        check(lib().gck_persist_begin(self._ctx, path.encode(), rank, world,
                                      meta_json.encode() if meta_json else None), self._ctx)

    def persist_wait(self) -> dict:
        st = L.PersistStats()
        check(lib().gck_persist_wait(self._ctx, C.byref(st)), self._ctx)
        return st.as_dict()

    def restore(self, path: str, stream=None) -> dict:
        h = L.FileHeader()
        check(lib().gck_restore(self._ctx, path.encode(), _stream_ptr(stream), C.byref(h)), self._ctx)
        return _hdr_dict(h)

    def session_steps(self) -> list[dict]:
        """Per-step log of the last finalized session (part, slot, wait/kernel/D2H ms, D2H bytes)."""
        arr = (L.SessionStep * L.K_LIMIT)()
        cnt = C.c_uint32(0)
        check(lib().gck_get_session_steps(self._ctx, arr, L.K_LIMIT, C.byref(cnt)), self._ctx)
        return [arr[i].as_dict() for i in range(cnt.value)]

    def stats(self) -> dict:
        s = L.Stats()
        check(lib().gck_get_stats(self._ctx, C.byref(s)))
        return s.as_dict()

    def close(self):
        if getattr(self, "_ctx", None):
            lib().gck_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
