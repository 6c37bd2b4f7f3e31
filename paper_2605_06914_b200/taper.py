"""Thin ctypes binding of libtaper.so (include/taper.h).

Argument marshalling only: every step of the hot path runs in the CUDA kernels of
``csrc/``.  There is no CPU or PyTorch fallback -- if the library is missing the
import of this module raises.  Function names mirror the C ABI.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TAPER_LIB", os.path.join(_HERE, "libtaper.so"))  # TAPER_LIB: dev builds

TAPER_OK = 0
TAPER_POLICY_OFF, TAPER_POLICY_CAP, TAPER_POLICY_EAGER, TAPER_POLICY_GREEDY = 0, 1, 2, 3
POLICY = {"off": 0, "cap": 1, "eager": 2, "taper": 3, "greedy": 3}
TAPER_STATUS_EMPTY_REQUEST, TAPER_STATUS_BAD_LENGTH = 1, 2
TAPER_STATUS_PRECISION, TAPER_STATUS_WORK_OVERFLOW = 4, 8
TAPER_STATUS_WORK_MISMATCH, TAPER_STATUS_EMPTY_CONTEXT = 16, 32
TAPER_MAX_SLOTS = 4096
TAPER_CHUNK_TOKENS = 4096
EXPORTS = ("taper_workspace_size", "taper_max_chunk_slots", "taper_admit", "taper_build_work", "taper_decode_attention",
           "taper_append_kv",
           "taper_status_string", "taper_last_error", "taper_last_launch_count",
           "taper_set_profile_events", "taper_set_trace_buffer",
           "taper_decode_attention_gather", "taper_gather_wait", "taper_ipc_handle",
           "taper_ipc_open", "taper_ipc_close", "taper_latency_observe", "taper_latency_refit")
TAPER_MAX_RANKS = 8
TAPER_LATENCY_WINDOW = 200

_vp = ctypes.c_void_p


class _Model(ctypes.Structure):
    _fields_ = [("a", ctypes.c_double), ("b", ctypes.c_double), ("c", ctypes.c_double)]


class _Policy(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("cap", ctypes.c_int32), ("rho", ctypes.c_double),
                ("utility", _vp), ("ctx_counting", ctypes.c_int32),
                ("utility_stride", ctypes.c_int32)]


CTX_COUNTING = {"per_sequence": 0, "per_request": 1}


class _Batch(ctypes.Structure):
    _fields_ = [("n_req", ctypes.c_int32), ("n_slot", ctypes.c_int32),
                ("req_shared_len", _vp), ("req_slot_off", _vp), ("req_slack_ms", _vp),
                ("slot_local_len", _vp), ("slot_seg_off", _vp), ("seg_len", _vp)]


class _Admission(ctypes.Structure):
    _fields_ = [("req_width", _vp), ("slot_admitted", _vp), ("adm_list", _vp), ("n_adm", _vp),
                ("diag", _vp), ("status", _vp)]


class _KV(ctypes.Structure):
    _fields_ = [("k_pages", _vp), ("v_pages", _vp), ("num_pages", ctypes.c_int32),
                ("page_size", ctypes.c_int32), ("h_local", ctypes.c_int32),
                ("req_page_off", _vp), ("req_pages", _vp), ("slot_page_off", _vp),
                ("slot_pages", _vp), ("seg_page_off", _vp)]


class _Gather(ctypes.Structure):
    _fields_ = [("world", ctypes.c_int32), ("rank", ctypes.c_int32),
                ("out", _vp * TAPER_MAX_RANKS), ("flags", _vp * TAPER_MAX_RANKS)]


class _Window(ctypes.Structure):
    _fields_ = [("count", ctypes.c_int32), ("head", ctypes.c_int32),
                ("n", ctypes.c_double * TAPER_LATENCY_WINDOW),
                ("L", ctypes.c_double * TAPER_LATENCY_WINDOW),
                ("t_ms", ctypes.c_double * TAPER_LATENCY_WINDOW)]


def load_library() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; "
                           "g.build()'` (nvcc, sm_100a).  There is no fallback path.")
    lib = ctypes.CDLL(LIB_PATH)
    P = ctypes.POINTER
    lib.taper_workspace_size.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                         ctypes.c_int64, P(ctypes.c_size_t)]
    lib.taper_max_chunk_slots.argtypes = [ctypes.c_int32, ctypes.c_int32, _vp, _vp, _vp, _vp, _vp,
                                          ctypes.c_int32, P(ctypes.c_int64)]
    lib.taper_max_chunk_slots.restype = ctypes.c_int
    lib.taper_admit.argtypes = [P(_Batch), P(_Model), P(_Policy), P(_Admission), ctypes.c_int32,
                                _vp, ctypes.c_size_t, _vp]
    lib.taper_build_work.argtypes = [P(_Batch), P(_Admission), ctypes.c_int32, _vp,
                                     ctypes.c_size_t, _vp]
    lib.taper_decode_attention.argtypes = [P(_Batch), P(_Admission), P(_KV), _vp, _vp, _vp,
                                           ctypes.c_float, _vp, ctypes.c_size_t, _vp]
    lib.taper_decode_attention_gather.argtypes = [P(_Batch), P(_Admission), P(_KV), _vp, P(_Gather),
                                                  _vp, ctypes.c_float, _vp, ctypes.c_size_t, _vp]
    lib.taper_gather_wait.argtypes = [P(_Gather), _vp]
    lib.taper_ipc_handle.argtypes = [_vp, _vp, P(ctypes.c_size_t)]
    lib.taper_ipc_open.argtypes = [_vp, ctypes.c_size_t, P(_vp)]
    lib.taper_ipc_close.argtypes = [_vp, ctypes.c_size_t]
    lib.taper_latency_observe.argtypes = [P(_Window), ctypes.c_double, ctypes.c_double, ctypes.c_double]
    lib.taper_latency_refit.argtypes = [P(_Window), P(_Model), P(ctypes.c_double)]
    lib.taper_append_kv.argtypes = [P(_Batch), P(_Admission), P(_KV), _vp, _vp, _vp]
    lib.taper_append_kv.restype = ctypes.c_int
    lib.taper_status_string.restype = ctypes.c_char_p
    lib.taper_status_string.argtypes = [ctypes.c_int]
    lib.taper_last_error.restype = ctypes.c_char_p
    lib.taper_last_launch_count.restype = ctypes.c_int
    lib.taper_set_trace_buffer.restype = ctypes.c_int
    lib.taper_set_trace_buffer.argtypes = [_vp, ctypes.c_int]
    lib.taper_set_profile_events.restype = ctypes.c_int
    lib.taper_set_profile_events.argtypes = [_vp, ctypes.c_int]
    for name in ("taper_workspace_size", "taper_admit", "taper_build_work",
                 "taper_decode_attention", "taper_decode_attention_gather", "taper_gather_wait",
                 "taper_ipc_handle", "taper_ipc_open", "taper_ipc_close", "taper_latency_observe",
                 "taper_latency_refit"):
        getattr(lib, name).restype = ctypes.c_int
    return lib


_lib = load_library()


class TaperError(RuntimeError):
    pass


def _check(code: int, what: str):
    if code != TAPER_OK:
        raise TaperError(f"{what}: {_lib.taper_status_string(code).decode()} "
                         f"({_lib.taper_last_error().decode()})")


def _ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def _stream(stream) -> int | None:
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream


def taper_status_string(code: int) -> str:
    return _lib.taper_status_string(code).decode()


def taper_last_launch_count() -> int:
    return _lib.taper_last_launch_count()


def taper_set_profile_events(events) -> None:
    """events: three torch.cuda.Event (created with enable_timing) or None."""
    if events is None:
        _check(_lib.taper_set_profile_events(None, 0), "taper_set_profile_events")
        return
    arr = (_vp * 3)(*[e.cuda_event for e in events])
    _check(_lib.taper_set_profile_events(arr, 3), "taper_set_profile_events")


def taper_set_trace_buffer(buf, capacity_tiles: int = 0) -> None:
    """Debug: int64 device tensor [capacity_tiles * 16] receiving CTA 0's pipeline events."""
    _check(_lib.taper_set_trace_buffer(None if buf is None else buf.data_ptr(),
                                       capacity_tiles), "taper_set_trace_buffer")


# ------------------------------------------------------------------ device-side containers
@dataclass
class DeviceBatch:
    """taper_batch: device copies of the SoA batch state."""
    req_shared_len: torch.Tensor  # int32 [R]
    req_slot_off: torch.Tensor    # int32 [R+1]
    req_slack_ms: torch.Tensor    # float64 [R]
    slot_local_len: torch.Tensor  # int32 [S]
    slot_seg_off: torch.Tensor | None = None  # int32 [S+1] local segments (reduce steps)
    seg_len: torch.Tensor | None = None       # int32 [n_seg]

    @property
    def n_req(self):
        return self.req_shared_len.numel()

    @property
    def n_slot(self):
        return self.slot_local_len.numel()

    @classmethod
    def from_host(cls, b, device="cuda") -> "DeviceBatch":
        t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a)).to(device=device, dtype=dt)
        seg_off = getattr(b, "slot_seg_off", None)
        seg = None if seg_off is None else (t(seg_off, torch.int32),
                                            t(b.seg_len if len(b.seg_len) else [0], torch.int32))
        return cls(t(b.req_shared_len, torch.int32), t(b.req_slot_off, torch.int32),
                   t(b.req_slack_ms, torch.float64), t(b.slot_local_len, torch.int32),
                   *(seg or ()))

    def c(self) -> _Batch:
        return _Batch(self.n_req, self.n_slot, _ptr(self.req_shared_len), _ptr(self.req_slot_off),
                      _ptr(self.req_slack_ms), _ptr(self.slot_local_len), _ptr(self.slot_seg_off),
                      _ptr(self.seg_len))


@dataclass
class DeviceAdmission:
    """taper_admission: caller-allocated admission outputs."""
    req_width: torch.Tensor
    slot_admitted: torch.Tensor
    adm_list: torch.Tensor
    n_adm: torch.Tensor
    diag: torch.Tensor
    status: torch.Tensor

    @classmethod
    def empty(cls, n_req, n_slot, device="cuda") -> "DeviceAdmission":
        z = lambda n, dt: torch.zeros(max(n, 1), dtype=dt, device=device)
        return cls(z(n_req, torch.int32), z(n_slot, torch.uint8), z(n_slot, torch.int32),
                   z(1, torch.int32), z(5, torch.float64), z(1, torch.int32))

    def c(self) -> _Admission:
        return _Admission(_ptr(self.req_width), _ptr(self.slot_admitted), _ptr(self.adm_list),
                          _ptr(self.n_adm), _ptr(self.diag), _ptr(self.status))


@dataclass
class DeviceKV:
    """taper_kv: one layer's K/V page pools plus the page tables."""
    k_pages: torch.Tensor  # bf16 [num_pages, h_local, page, 128]
    v_pages: torch.Tensor
    req_page_off: torch.Tensor
    req_pages: torch.Tensor
    slot_page_off: torch.Tensor
    slot_pages: torch.Tensor
    seg_page_off: torch.Tensor | None = None  # int32 [n_seg] with DeviceBatch.slot_seg_off

    def c(self) -> _KV:
        n, h, ps, d = self.k_pages.shape
        return _KV(_ptr(self.k_pages), _ptr(self.v_pages), n, ps, h, _ptr(self.req_page_off),
                   _ptr(self.req_pages), _ptr(self.slot_page_off), _ptr(self.slot_pages),
                   _ptr(self.seg_page_off))


def page_tables_to_device(layout, device="cuda"):
    t = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.int32)).to(device)
    pad = lambda a: a if len(a) else np.zeros(1, np.int32)
    return (t(layout.req_page_off), t(pad(layout.req_pages)), t(layout.slot_page_off),
            t(pad(layout.slot_pages)))


def max_chunk_slots(req_shared_len, req_slot_off, slot_local_len, seg_len=None,
                    h_local: int = 1, slot_seg_off=None) -> int:
    """taper_max_chunk_slots (include/taper.h): the Eager bound of the partial rows for
    taper_workspace_size, from host arrays.  ``seg_len`` without ``slot_seg_off``: the
    segments are counted flat (the bound only needs their lengths)."""
    a = lambda x: np.ascontiguousarray(np.asarray(x, np.int32))
    lsh, off, lloc = a(req_shared_len), a(req_slot_off), a(slot_local_len)
    R, S = len(lsh), len(lloc)
    so = sl = None
    if seg_len is not None:
        sl = a(seg_len) if len(seg_len) else np.zeros(1, np.int32)
        so = a(slot_seg_off) if slot_seg_off is not None else None
        if so is None:  # lengths only: one pseudo-slot per segment, zero-length slots
            so = np.zeros(S + 1, np.int32)
            so[S] = len(seg_len)
    out = ctypes.c_int64(0)
    ptr = lambda x: None if x is None else x.ctypes.data_as(ctypes.c_void_p)
    _check(_lib.taper_max_chunk_slots(R, S, ptr(lsh), ptr(off), ptr(lloc if so is None else np.zeros(max(S, 1), np.int32)),
                                      ptr(so), ptr(sl), h_local, ctypes.byref(out)),
           "taper_max_chunk_slots")
    return out.value


# ------------------------------------------------------------------ C-ABI calls
def taper_workspace_size(n_req: int, n_slot: int, h_local: int, max_chunk_slots: int) -> int:
    out = ctypes.c_size_t(0)
    _check(_lib.taper_workspace_size(n_req, n_slot, h_local, max_chunk_slots, ctypes.byref(out)),
           "taper_workspace_size")
    return out.value


def taper_admit(batch: DeviceBatch, model, policy: str = "taper", rho: float = 0.8,
                adm: DeviceAdmission = None, h_local: int = 8, workspace: torch.Tensor = None,
                cap: int = 2, stream=None, ctx: str = "per_sequence",
                utility: torch.Tensor | None = None) -> DeviceAdmission:
    """utility: None (linear u_r(k) = k) or a float64 device tensor [R, K] with
    utility[r, k] = u_r(k), flat past column K-1 (include/taper.h taper_policy)."""
    a, b, c = (float(x) for x in model)
    ustride = 0
    if utility is not None:
        assert utility.dtype == torch.float64 and utility.is_cuda and utility.is_contiguous()
        assert utility.dim() == 2 and utility.shape[0] >= batch.n_req
        ustride = utility.shape[1]
    kind = POLICY[policy] if isinstance(policy, str) else int(policy)
    bc, ac = batch.c(), adm.c()
    _check(_lib.taper_admit(ctypes.byref(bc), ctypes.byref(_Model(a, b, c)),
                            ctypes.byref(_Policy(kind, cap, rho, _ptr(utility), CTX_COUNTING[ctx],
                                                 ustride)),
                            ctypes.byref(ac),
                            h_local, _ptr(workspace), workspace.numel() * workspace.element_size(),
                            _stream(stream)), "taper_admit")
    return adm


def taper_build_work(batch: DeviceBatch, adm: DeviceAdmission, h_local: int,
                     workspace: torch.Tensor, stream=None):
    bc, ac = batch.c(), adm.c()
    _check(_lib.taper_build_work(ctypes.byref(bc), ctypes.byref(ac), h_local, _ptr(workspace),
                                 workspace.numel() * workspace.element_size(), _stream(stream)),
           "taper_build_work")


def taper_decode_attention(batch: DeviceBatch, adm: DeviceAdmission, kv: DeviceKV,
                           q: torch.Tensor, out: torch.Tensor, lse: torch.Tensor | None,
                           scale: float, workspace: torch.Tensor, stream=None):
    assert q.dtype == torch.bfloat16 and out.dtype == torch.bfloat16
    assert q.is_contiguous() and out.is_contiguous()
    bc, ac, kc = batch.c(), adm.c(), kv.c()
    _check(_lib.taper_decode_attention(ctypes.byref(bc), ctypes.byref(ac), ctypes.byref(kc),
                                       _ptr(q), _ptr(out), _ptr(lse), float(scale),
                                       _ptr(workspace),
                                       workspace.numel() * workspace.element_size(),
                                       _stream(stream)), "taper_decode_attention")


class Gather:
    """taper_gather (include/taper.h): this rank's view of the G ranks' gathered output
    buffers ([S, 64, 128] bf16 device pointers usable in this process) and of the flag
    arrays of one call.  Pointers only; the owner keeps the memory alive."""

    def __init__(self, world: int, rank: int, outs: list[int], flags: list[int]):
        assert len(outs) == world and len(flags) == world
        self.world, self.rank = world, rank
        self._c = _Gather(world, rank, (_vp * TAPER_MAX_RANKS)(*outs),
                          (_vp * TAPER_MAX_RANKS)(*flags))

    def c(self) -> _Gather:
        return self._c


def taper_decode_attention_gather(batch: DeviceBatch, adm: DeviceAdmission, kv: DeviceKV,
                                  q: torch.Tensor, gather: Gather, lse: torch.Tensor | None,
                                  scale: float, workspace: torch.Tensor, stream=None):
    """Attention whose merge epilogue stores every output row into all ranks' gathered
    buffers and then raises this rank's flag in every rank's flag array."""
    assert q.dtype == torch.bfloat16 and q.is_contiguous()
    bc, ac, kc, gc = batch.c(), adm.c(), kv.c(), gather.c()
    _check(_lib.taper_decode_attention_gather(ctypes.byref(bc), ctypes.byref(ac), ctypes.byref(kc),
                                              _ptr(q), ctypes.byref(gc), _ptr(lse), float(scale),
                                              _ptr(workspace),
                                              workspace.numel() * workspace.element_size(),
                                              _stream(stream)), "taper_decode_attention_gather")


def taper_gather_wait(gather: Gather, stream=None):
    gc = gather.c()
    _check(_lib.taper_gather_wait(ctypes.byref(gc), _stream(stream)), "taper_gather_wait")


def taper_ipc_handle(t: torch.Tensor) -> tuple[bytes, int]:
    """(64-byte CUDA IPC handle of the allocation holding t, t's offset in it)."""
    buf = ctypes.create_string_buffer(64)
    off = ctypes.c_size_t(0)
    _check(_lib.taper_ipc_handle(_ptr(t), buf, ctypes.byref(off)), "taper_ipc_handle")
    return buf.raw, int(off.value)


def taper_ipc_open(handle: bytes, offset: int) -> int:
    ptr = _vp()
    _check(_lib.taper_ipc_open(ctypes.create_string_buffer(handle, 64), offset, ctypes.byref(ptr)),
           "taper_ipc_open")
    return int(ptr.value)


def taper_ipc_close(ptr: int, offset: int):
    _check(_lib.taper_ipc_close(ptr, offset), "taper_ipc_close")


class LatencyWindow:
    """taper_latency_window (include/taper.h): the rolling window of the last 200 observed
    steps (App. C.1 "Fitting", L337) and its OLS refit of T(S) = a + b n + c L."""

    def __init__(self):
        self._w = _Window()

    def observe(self, n: float, L: float, t_ms: float):
        _check(_lib.taper_latency_observe(ctypes.byref(self._w), float(n), float(L), float(t_ms)),
               "taper_latency_observe")

    @property
    def count(self) -> int:
        return int(self._w.count)

    def refit(self, model) -> tuple[tuple[float, float, float], dict]:
        """(new model, {r2, mape, rmse_ms}); raises TaperError (the model unchanged) when the
        fit would not be monotone or the window is degenerate."""
        m = _Model(*model)
        fit = (ctypes.c_double * 3)()
        _check(_lib.taper_latency_refit(ctypes.byref(self._w), ctypes.byref(m), fit),
               "taper_latency_refit")
        return (m.a, m.b, m.c), {"r2": fit[0], "mape": fit[1], "rmse_ms": fit[2]}


def taper_append_kv(batch: DeviceBatch, adm: DeviceAdmission, kv: DeviceKV,
                    k_new: torch.Tensor, v_new: torch.Tensor, stream=None):
    """Write each admitted slot's new token K/V ([S, h_local, 128] bf16) into the pages."""
    assert k_new.dtype == torch.bfloat16 and v_new.dtype == torch.bfloat16
    assert k_new.is_contiguous() and v_new.is_contiguous()
    bc, ac, kc = batch.c(), adm.c(), kv.c()
    _check(_lib.taper_append_kv(ctypes.byref(bc), ctypes.byref(ac), ctypes.byref(kc),
                                _ptr(k_new), _ptr(v_new), _stream(stream)), "taper_append_kv")
