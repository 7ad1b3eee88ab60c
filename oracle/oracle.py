"""ctypes front end of the CPU oracle (oracle/liboracle.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py, always as the checker or the
CPU baseline, never as the product path.  Builds itself with `make` on first
use if the shared object is missing (gcc is in the image).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

CODES = {0: "ok", 2: "ValueError", 3: "FieldError", 4: "DegenerateBoundError", 5: "ArchiveError",
         7: "StageError", 8: "MemoryError"}
STAGE = {"huffman": 1, "rre": 2, "rze": 3, "tcms": 4, "bit": 5, "cr": 10, "tp": 11}


class OracleError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{CODES.get(code, code)}: {msg}")
        self.code = code
        self.kind = CODES.get(code, str(code))


def build(force: bool = False) -> str:
    so = os.path.join(HERE, "liboracle.so")
    src = os.path.join(HERE, "hb_oracle.c")
    if force or not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    return so


def lib():
    global _LIB
    if _LIB is None:
        L = C.CDLL(build())
        P, U64, SZ, I, D = C.c_void_p, C.c_uint64, C.c_size_t, C.c_int, C.c_double
        PU64 = C.POINTER(C.c_uint64)
        L.hbo_last_error.restype = C.c_char_p
        L.hbo_free.argtypes = [P]
        L.hbo_set_threads.argtypes = [I]
        L.hbo_resolve_eb.argtypes = [P, I, U64, I, D, C.POINTER(D)]
        L.hbo_anchor_stride.argtypes = [PU64]
        L.hbo_plan_blocks.argtypes = [PU64, PU64, I, PU64]
        L.hbo_tune.argtypes = [P, I, PU64, D, P, P]
        L.hbo_decompose.argtypes = [P, I, PU64, D, P, P, P, P, PU64, P]
        L.hbo_reconstruct.argtypes = [P, P, P, U64, P, I, PU64, D, P, P]
        L.hbo_index_of.argtypes = [PU64, I, U64, U64, U64]
        L.hbo_index_of.restype = U64
        L.hbo_reorder.argtypes = [P, PU64, I, P]
        L.hbo_inverse_reorder.argtypes = [P, PU64, I, P]
        L.hbo_stage_encode.argtypes = [I, I, P, SZ, C.POINTER(P), C.POINTER(SZ)]
        L.hbo_stage_decode.argtypes = [I, P, SZ, C.POINTER(P), C.POINTER(SZ)]
        L.hbo_compress.argtypes = [P, I, PU64, I, I, D, I, C.POINTER(P), C.POINTER(SZ)]
        L.hbo_decompress.argtypes = [P, SZ, P, SZ, P]
        _LIB = L
    return _LIB


def _check(rc):
    if rc:
        raise OracleError(rc, lib().hbo_last_error().decode())


def _dims(d):
    d = tuple(int(x) for x in d)
    if len(d) == 2:
        d = d + (1,)
    return (C.c_uint64 * 3)(*d)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _prec(a: np.ndarray) -> int:
    if a.dtype == np.float32:
        return 4
    if a.dtype == np.float64:
        return 8
    raise TypeError(a.dtype)


def set_threads(n: int):
    lib().hbo_set_threads(int(n))


def resolve_eb(values: np.ndarray, eb_mode: str, mag: float) -> float:
    v = np.ascontiguousarray(values)
    out = C.c_double()
    _check(lib().hbo_resolve_eb(_ptr(v), _prec(v), v.size, 0 if eb_mode == "abs" else 1, float(mag),
                                C.byref(out)))
    return out.value


def anchor_stride(dims) -> int:
    return lib().hbo_anchor_stride(_dims(dims))


def plan_blocks(dims):
    mx = 1 << 16
    org = (C.c_uint64 * (3 * mx))()
    shp = (C.c_uint64 * 3)()
    n = lib().hbo_plan_blocks(_dims(dims), org, mx, shp)
    return [tuple(org[3 * i:3 * i + 3]) for i in range(n)], tuple(shp)


def tune(values: np.ndarray, eb: float):
    v = np.ascontiguousarray(values)
    cfg = np.zeros(4, np.uint8)
    errs = np.zeros(16, np.float64)
    _check(lib().hbo_tune(_ptr(v), _prec(v), _dims(v.shape), float(eb), _ptr(cfg), _ptr(errs)))
    return cfg, errs.reshape(4, 4)


def decompose(values: np.ndarray, eb: float, cfg):
    v = np.ascontiguousarray(values)
    n = v.size
    a = anchor_stride(v.shape)
    na = int(np.prod([-(-d // a) for d in v.shape]))
    codes = np.empty(v.shape, np.uint8)
    oidx = np.empty(n, np.uint64)
    oval = np.empty(n, v.dtype)
    anc = np.empty(na, v.dtype)
    cnt = C.c_uint64()
    cfgb = np.ascontiguousarray(np.asarray(cfg, np.uint8))
    _check(lib().hbo_decompose(_ptr(v), _prec(v), _dims(v.shape), float(eb), _ptr(cfgb), _ptr(codes), _ptr(oidx),
                               _ptr(oval), C.byref(cnt), _ptr(anc)))
    k = cnt.value
    shape = tuple(-(-d // a) for d in v.shape)
    return codes, oidx[:k].copy(), oval[:k].copy(), anc.reshape(shape)


def reconstruct(codes, oidx, oval, anchors, eb, cfg, dims, dtype):
    codes = np.ascontiguousarray(codes, np.uint8)
    dt = np.dtype(dtype)
    oidx = np.ascontiguousarray(oidx, np.uint64)
    oval = np.ascontiguousarray(oval, dt)
    anchors = np.ascontiguousarray(anchors, dt)
    out = np.empty(tuple(int(d) for d in dims), dt)
    cfgb = np.ascontiguousarray(np.asarray(cfg, np.uint8))
    _check(lib().hbo_reconstruct(_ptr(codes), _ptr(oidx), _ptr(oval), oidx.size, _ptr(anchors), dt.itemsize,
                                 _dims(dims), float(eb), _ptr(cfgb), _ptr(out)))
    return out


def index_of(dims, stride, x, y, z) -> int:
    return int(lib().hbo_index_of(_dims(dims), int(stride), x, y, z))


def reorder(codes: np.ndarray, stride: int) -> np.ndarray:
    c = np.ascontiguousarray(codes, np.uint8)
    seq = np.empty(c.size, np.uint8)
    _check(lib().hbo_reorder(_ptr(c), _dims(c.shape), int(stride), _ptr(seq)))
    return seq


def inverse_reorder(seq: np.ndarray, dims, stride: int) -> np.ndarray:
    s = np.ascontiguousarray(seq, np.uint8)
    out = np.empty(tuple(int(d) for d in dims), np.uint8)
    _check(lib().hbo_inverse_reorder(_ptr(s), _dims(dims), int(stride), _ptr(out)))
    return out


def _call_stage(fn, *args) -> bytes:
    out = C.c_void_p()
    n = C.c_size_t()
    _check(fn(*args, C.byref(out), C.byref(n)))
    try:
        return C.string_at(out, n.value)
    finally:
        lib().hbo_free(out)


def stage_encode(stage: str, data: bytes, width: int = 1) -> bytes:
    buf = np.frombuffer(data, np.uint8) if data else np.zeros(1, np.uint8)
    return _call_stage(lib().hbo_stage_encode, STAGE[stage], int(width), _ptr(buf), len(data))


def stage_decode(stage: str, blob: bytes) -> bytes:
    buf = np.frombuffer(blob, np.uint8) if blob else np.zeros(1, np.uint8)
    return _call_stage(lib().hbo_stage_decode, STAGE[stage], _ptr(buf), len(blob))


def compress(values: np.ndarray, eb_mode: str, mag: float, mode: str = "cr", ndim: int | None = None) -> bytes:
    v = np.ascontiguousarray(values)
    if v.ndim == 2:
        v = v.reshape(v.shape + (1,))
        ndim = 2 if ndim is None else ndim
    if ndim is None:
        ndim = 3
    return _call_stage(lib().hbo_compress, _ptr(v), _prec(v), _dims(v.shape), int(ndim),
                       0 if eb_mode == "abs" else 1, float(mag), 0 if mode == "cr" else 1)


class _Info(C.Structure):
    _fields_ = [("mode", C.c_int), ("precision", C.c_int), ("ndim", C.c_int), ("stride", C.c_int),
                ("escape", C.c_int), ("cfg", C.c_uint8 * 4), ("dims", C.c_uint64 * 3), ("eb", C.c_double),
                ("anchor_count", C.c_uint64), ("outlier_count", C.c_uint64), ("stream_len", C.c_uint64),
                ("anchor_off", C.c_uint64), ("outlier_off", C.c_uint64), ("stream_off", C.c_uint64)]


def decompress(blob: bytes):
    """Returns (values ndarray of shape dims, ndim)."""
    info = _Info()
    buf = np.frombuffer(blob, np.uint8) if blob else np.zeros(1, np.uint8)
    # header first (cap 0 only validates), then the real call
    rc = lib().hbo_decompress(_ptr(buf), len(blob), None, 0, C.byref(info))
    if rc not in (0, 2):
        _check(rc)
    dims = tuple(info.dims)
    dt = np.float32 if info.precision == 4 else np.float64
    out = np.empty(dims, dt)
    _check(lib().hbo_decompress(_ptr(buf), len(blob), _ptr(out), out.nbytes, C.byref(info)))
    return out, info.ndim
