"""Interpolation predictor / quantizer API (reference predictor.py).

`decompose` and `reconstruct` run on the GPU (k_predict.cu level kernels via
hb_decompose / hb_reconstruct); the small scalar helpers (`quantize`,
`interpolate_1d`) and the config objects are host-side conveniences that the
reference also exposes.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import ArchiveError, DegenerateBoundError, FieldError
from .field import Field

ANCHOR_STRIDE = 16
OUTLIER_CODE = 0
CODE_ZERO = 128
MAX_Q = 127

CUBIC, LINEAR = "cubic", "linear"
SEQ1D, MULTIDIM = "seq1d", "multidim"
SPLINES = (CUBIC, LINEAR)
SCHEMES = (MULTIDIM, SEQ1D)


@dataclass(frozen=True)
class InterpConfig:
    """Per-level (spline, scheme); index 0 holds level 1 (predictor.py:56-95).

    Wire form: one byte per level, bit0 = spline (0 cubic, 1 linear),
    bit1 = scheme (0 multidim, 1 seq1d)."""

    levels: tuple

    def __post_init__(self):
        if len(self.levels) != 4:
            raise FieldError("interpolation config must cover 4 levels")
        for spline, scheme in self.levels:
            if spline not in SPLINES or scheme not in SCHEMES:
                raise FieldError(f"bad interpolation config entry ({spline}, {scheme})")

    @classmethod
    def default(cls) -> "InterpConfig":
        return cls(((CUBIC, MULTIDIM),) * 4)

    def level(self, l: int):
        return self.levels[l - 1]

    def replace_level(self, l: int, spline: str, scheme: str) -> "InterpConfig":
        lv = list(self.levels)
        lv[l - 1] = (spline, scheme)
        return InterpConfig(tuple(lv))

    def to_bytes(self) -> bytes:
        return bytes(SPLINES.index(sp) | (SCHEMES.index(sc) << 1) for sp, sc in self.levels)

    @classmethod
    def from_bytes(cls, raw: bytes) -> "InterpConfig":
        if len(raw) != 4:
            raise ArchiveError("interpolation config must be 4 bytes")
        out = []
        for b in raw:
            if b & ~0x03:
                raise ArchiveError(f"invalid interpolation config byte 0x{b:02x}")
            out.append((SPLINES[b & 1], SCHEMES[(b >> 1) & 1]))
        return cls(tuple(out))


@dataclass(frozen=True)
class AnchorGrid:
    stride: int
    values: np.ndarray


@dataclass(frozen=True)
class QuantizedField:
    codes: np.ndarray
    outlier_indices: np.ndarray
    outlier_values: np.ndarray
    anchors: AnchorGrid


def effective_anchor_stride(dims) -> int:
    """Largest power of two <= min(16, smallest non-degenerate dim)."""
    nondeg = [int(d) for d in dims if int(d) > 1]
    limit = min(min(nondeg) if nondeg else 1, ANCHOR_STRIDE)
    a = 1
    while a * 2 <= limit:
        a *= 2
    return a


def extract_anchors(field: Field, stride: int | None = None) -> AnchorGrid:
    a = effective_anchor_stride(field.dims) if stride is None else int(stride)
    v = field.host_values()
    return AnchorGrid(a, np.ascontiguousarray(v[::a, ::a, ::a]))


def quantize(err: float, eb: float):
    """Scalar form of the quantizer (predictor.py:133-149)."""
    if not math.isfinite(err):
        raise ValueError(f"non-finite prediction error {err!r}")
    if not (math.isfinite(eb) and eb > 0):
        raise DegenerateBoundError(f"error bound must be positive and finite, got {eb}")
    q = math.floor(abs(err) / (2.0 * eb) + 0.5)
    q = -q if err < 0 else q
    if abs(q) > MAX_Q or abs(err - 2.0 * eb * q) > eb:
        return OUTLIER_CODE, True
    return q + CODE_ZERO, False


_RULES = (((-3, -1, 1, 3), (-0.0625, 0.5625, 0.5625, -0.0625), 4),
          ((-1, 1, 3), (0.375, 0.75, -0.125), 3),
          ((-3, -1, 1), (-0.125, 0.75, 0.375), 3))


def interpolate_1d(samples, spline: str):
    """Predict offset 0 from (offset, value) samples (predictor.py:152-174)."""
    if spline not in SPLINES:
        raise ValueError(f"unknown spline {spline!r}")
    have = dict(samples)
    if not have:
        raise ValueError("at least one sample is required")
    if spline == CUBIC:
        for offs, wts, order in _RULES:
            if all(o in have for o in offs):
                return sum(w * have[o] for o, w in zip(offs, wts)), order
    near = sorted(have, key=lambda o: (abs(o), o))
    if len(near) >= 2:
        a, b = sorted(near[:2])
        return (b * have[a] - a * have[b]) / (b - a), 2
    return have[near[0]], 1


def _field_buf(field: Field):
    v = field.values
    if isinstance(v, np.ndarray):
        return v, v.dtype.itemsize
    return v, v.element_size()


def decompose(field: Field, eb: float, config: InterpConfig) -> QuantizedField:
    """predictor.py:372 on the GPU: codes (grid order), sorted outliers, anchors."""
    if not (math.isfinite(eb) and eb > 0):
        raise DegenerateBoundError(f"error bound must be positive and finite, got {eb}")
    L, c = _lib.lib(), _lib.ctx()
    buf, prec = _field_buf(field)
    dims = field.dims
    n = field.count
    a = effective_anchor_stride(dims)
    ashape = tuple(-(-d // a) for d in dims)
    dt = np.float32 if prec == 4 else np.float64
    seq = np.empty(n, np.uint8)
    oidx = np.empty(n, np.uint64)
    oval = np.empty(n, dt)
    anc = np.empty(ashape, dt)
    cnt = C.c_uint64()
    cfg = np.frombuffer(config.to_bytes(), np.uint8).copy()
    rc = L.hb_decompose(c, _lib.ptr(buf), prec, _lib.dims3(dims), float(eb), _lib.ptr(cfg), _lib.ptr(seq),
                        _lib.ptr(oidx), _lib.ptr(oval), C.byref(cnt), _lib.ptr(anc))
    _lib.raise_for(rc, c)
    codes = np.empty(dims, np.uint8)
    rc = L.hb_inverse_reorder(c, _lib.ptr(seq), _lib.dims3(dims), a, _lib.ptr(codes))
    _lib.raise_for(rc, c)
    k = cnt.value
    return QuantizedField(codes, oidx[:k].copy(), oval[:k].copy(), AnchorGrid(a, anc))


def reconstruct(quantized: QuantizedField, eb: float, config: InterpConfig, dims=None,
                ndim: int | None = None) -> Field:
    """predictor.py:378-416 on the GPU."""
    if not (math.isfinite(eb) and eb > 0):
        raise DegenerateBoundError(f"error bound must be positive and finite, got {eb}")
    codes = np.ascontiguousarray(quantized.codes, np.uint8)
    if dims is not None and tuple(dims) != codes.shape:
        raise FieldError(f"code array shape {codes.shape} does not match dims {tuple(dims)}")
    dims = codes.shape
    a = quantized.anchors.stride
    anc = np.ascontiguousarray(quantized.anchors.values)
    dt = anc.dtype
    oidx = np.ascontiguousarray(quantized.outlier_indices, np.uint64)
    oval = np.ascontiguousarray(quantized.outlier_values, dt)
    L, c = _lib.lib(), _lib.ctx()
    seq = np.empty(codes.size, np.uint8)
    rc = L.hb_reorder(c, _lib.ptr(codes), _lib.dims3(dims), a, _lib.ptr(seq))
    _lib.raise_for(rc, c)
    out = np.empty(dims, dt)
    cfg = np.frombuffer(config.to_bytes(), np.uint8).copy()
    rc = L.hb_reconstruct(c, _lib.ptr(seq), _lib.ptr(oidx) if oidx.size else None,
                          _lib.ptr(oval) if oval.size else None, oidx.size, _lib.ptr(anc), dt.itemsize,
                          _lib.dims3(dims), a, float(eb), _lib.ptr(cfg), _lib.ptr(out))
    _lib.raise_for(rc, c)
    if ndim is None:
        ndim = 2 if dims[2] == 1 else 3
    return Field(out, ndim=ndim)
