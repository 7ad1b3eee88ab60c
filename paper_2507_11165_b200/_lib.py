"""ctypes binding of libhibound_b200.so (include/hibound_b200.h).

This is the whole host/device boundary: every hot-path call below goes
through the C ABI into hand-written sm_100a kernels.  There is no CPU
fallback -- if the shared library or a CUDA device is missing, calls raise.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from .errors import ArchiveError, DegenerateBoundError, FieldError, HiboundError, StageError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libhibound_b200.so")

HB_OK, HB_EARG, HB_EFIELD, HB_EBOUND, HB_EARCHIVE, HB_ESTAGE, HB_ECUDA, HB_EUNSUPPORTED = 0, 2, 3, 4, 5, 7, 8, 9

_lib = None
_lock = threading.Lock()
_tls = threading.local()


class Info(C.Structure):
    _fields_ = [("mode", C.c_int), ("precision", C.c_int), ("ndim", C.c_int), ("stride", C.c_int),
                ("escape", C.c_int), ("cfg", C.c_uint8 * 4), ("dims", C.c_uint64 * 3), ("eb", C.c_double),
                ("anchor_count", C.c_uint64), ("outlier_count", C.c_uint64), ("stream_len", C.c_uint64),
                ("anchor_off", C.c_uint64), ("outlier_off", C.c_uint64), ("stream_off", C.c_uint64)]


def lib():
    """Load the shared library (building it first if this is a source tree)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            from . import _build
            _build.build()
        L = C.CDLL(LIB_PATH)
        P, U64, SZ, I, D = C.c_void_p, C.c_uint64, C.c_size_t, C.c_int, C.c_double
        PU64 = C.POINTER(C.c_uint64)
        L.hb_ctx_create.argtypes = [I, P, C.POINTER(P)]
        L.hb_ctx_destroy.argtypes = [P]
        L.hb_last_error.argtypes = [P]
        L.hb_last_error.restype = C.c_char_p
        L.hb_last_launch_count.argtypes = [P]
        L.hb_last_launch_count.restype = U64
        L.hb_profile.argtypes = [P, I]
        L.hb_last_phases.argtypes = [P, C.POINTER(C.c_char_p), C.POINTER(C.c_float), I]
        L.hb_last_phases.restype = I
        L.hb_compress_bound.argtypes = [PU64, I, C.POINTER(SZ)]
        L.hb_compress.argtypes = [P, P, I, PU64, I, I, D, I, P, SZ, C.POINTER(SZ), C.POINTER(D), P]
        L.hb_archive_info.argtypes = [P, SZ, C.POINTER(Info)]
        L.hb_value_range.argtypes = [P, P, I, U64, C.POINTER(D), C.POINTER(D)]
        L.hb_quality.argtypes = [P, P, P, I, U64, C.POINTER(D)]
        L.hb_decompress.argtypes = [P, P, SZ, P, SZ, C.POINTER(Info)]
        L.hb_tune.argtypes = [P, P, I, PU64, D, P, P]
        L.hb_decompose.argtypes = [P, P, I, PU64, D, P, P, P, P, PU64, P]
        L.hb_reconstruct.argtypes = [P, P, P, P, U64, P, I, PU64, I, D, P, P]
        L.hb_reorder.argtypes = [P, P, PU64, I, P]
        L.hb_inverse_reorder.argtypes = [P, P, PU64, I, P]
        L.hb_stage_encode.argtypes = [P, I, I, P, SZ, P, SZ, C.POINTER(SZ)]
        L.hb_stage_decode.argtypes = [P, I, P, SZ, P, SZ, C.POINTER(SZ)]
        _lib = L
    return _lib


def _torch():
    try:
        import torch
        return torch
    except Exception:  # pragma: no cover - torch is in the image
        return None


def current_device_and_stream():
    t = _torch()
    if t is not None and t.cuda.is_available():
        dev = t.cuda.current_device()
        return dev, t.cuda.current_stream(dev).cuda_stream
    return 0, 0


class _Contexts(dict):
    """This thread's contexts, keyed by (device, stream).  Lives in a
    threading.local, so when the thread exits (or release_contexts() runs)
    every context is destroyed and its device arena, pinned staging, second
    stream and recorded graphs are returned."""

    def release(self):
        L = _lib
        while self:
            _, c = self.popitem()
            if L is not None:
                L.hb_ctx_destroy(c)

    def __del__(self):
        try:
            self.release()
        except Exception:  # interpreter shutdown
            pass


def _thread_contexts() -> _Contexts:
    cs = getattr(_tls, "ctxs", None)
    if cs is None:
        cs = _tls.ctxs = _Contexts()
    return cs


def ctx():
    """Context bound to torch's current device and stream (created on demand,
    one per thread: a context is single-stream and never shared)."""
    dev, stream = current_device_and_stream()
    cs = _thread_contexts()
    c = cs.get((dev, stream))
    if c is None:
        L = lib()
        p = C.c_void_p()
        rc = L.hb_ctx_create(dev, C.c_void_p(stream) if stream else None, C.byref(p))
        if rc != HB_OK:
            raise RuntimeError(f"hb_ctx_create failed (code {rc}): no usable CUDA device for the B200 path")
        c = p
        cs[(dev, stream)] = c
    return c


def release_contexts():
    """Destroy the calling thread's contexts now (device memory back to the
    driver); the next call creates a fresh one."""
    _thread_contexts().release()


def raise_for(rc: int, c=None, what: str = ""):
    if rc == HB_OK:
        return
    msg = lib().hb_last_error(c).decode() if c is not None else what
    if rc == HB_EFIELD:
        raise FieldError(msg)
    if rc == HB_EBOUND:
        raise DegenerateBoundError(msg)
    if rc == HB_ESTAGE:
        raise StageError(msg)
    if rc == HB_EARCHIVE:
        raise ArchiveError(msg)
    if rc == HB_EARG:
        raise ValueError(msg)
    if rc == HB_EUNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(f"CUDA failure in libhibound_b200: {msg}")


def last_launch_count() -> int:
    return int(lib().hb_last_launch_count(ctx()))


def dims3(dims):
    d = tuple(int(x) for x in dims)
    return (C.c_uint64 * 3)(*d)


def ptr(buf) -> C.c_void_p:
    """Raw pointer of a numpy array, torch tensor (host or CUDA) or bytes."""
    if isinstance(buf, np.ndarray):
        return C.c_void_p(buf.ctypes.data)
    t = _torch()
    if t is not None and isinstance(buf, t.Tensor):
        return C.c_void_p(buf.data_ptr())
    if isinstance(buf, (bytes, bytearray, memoryview)):
        arr = np.frombuffer(buf, np.uint8)
        return C.c_void_p(arr.ctypes.data)
    raise TypeError(f"unsupported buffer type {type(buf)!r}")


def is_cuda(x) -> bool:
    t = _torch()
    return t is not None and isinstance(x, t.Tensor) and x.is_cuda


def set_profile(enable):
    """True/1: CUDA-event marks at every phase; 2: only the level-pass marks
    (the cheap form used inside bench.py's timed region); False/0: off."""
    lib().hb_profile(ctx(), 2 if enable == 2 else (1 if enable else 0))


def last_phases() -> list:
    names = (C.c_char_p * 64)()
    ms = (C.c_float * 64)()
    n = lib().hb_last_phases(ctx(), names, ms, 64)
    return [(names[i].decode(), float(ms[i])) for i in range(n)]
