"""Eq. 3 level-grouped order (reference ordering.py).

The closed-form rank is host arithmetic for single points; whole-grid
reorder / inverse_reorder run on the GPU (k_reorder).  Inside compress and
decompress the mapping is fused into the level kernels.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .errors import FieldError


def level_of(x: int, y: int, z: int, stride: int) -> int:
    top = int(stride).bit_length() - 1
    for l in range(top, 0, -1):
        m = (1 << l) - 1
        if not (x & m or y & m or z & m):
            return l
    return 0


class LevelMap:
    """Bijection grid <-> level-grouped sequence (ordering.py:38-118)."""

    def __init__(self, dims, stride: int):
        dims = tuple(int(d) for d in dims)
        if len(dims) != 3 or any(d < 1 for d in dims):
            raise FieldError(f"bad dims {dims}")
        stride = int(stride)
        if stride < 1 or stride & (stride - 1):
            raise FieldError(f"anchor stride must be a power of two, got {stride}")
        self.dims, self.stride = dims, stride
        self.top = stride.bit_length() - 1
        self.count = dims[0] * dims[1] * dims[2]
        self.subdims = [tuple(-(-d // (1 << l)) for d in dims) for l in range(self.top + 1)]
        self.prefixes = [int(np.prod(self.subdims[l + 1])) if l < self.top else 0 for l in range(self.top + 1)]
        self.level_counts = [int(np.prod(self.subdims[l])) - self.prefixes[l] if l < self.top
                             else int(np.prod(self.subdims[l])) for l in range(self.top + 1)]

    def index_of(self, x: int, y: int, z: int) -> int:
        dx, dy, dz = self.dims
        if not (0 <= x < dx and 0 <= y < dy and 0 <= z < dz):
            raise FieldError(f"coordinate ({x},{y},{z}) outside dims {self.dims}")
        l = level_of(x, y, z, self.stride)
        _, gy, gz = self.subdims[l]
        X, Y, Z = x >> l, y >> l, z >> l
        rank = (X * gy + Y) * gz + Z
        if l < self.top:
            ey, ez = (gy + 1) // 2, (gz + 1) // 2
            rank -= ((X + 1) // 2) * ey * ez
            if X % 2 == 0:
                rank -= ((Y + 1) // 2) * ez + (0 if Y % 2 else (Z + 1) // 2)
        return self.prefixes[l] + rank


def reorder(codes: np.ndarray, lmap: LevelMap) -> np.ndarray:
    if tuple(codes.shape) != lmap.dims:
        raise FieldError(f"code array shape {codes.shape} does not match map dims {lmap.dims}")
    c = np.ascontiguousarray(codes, np.uint8)
    out = np.empty(lmap.count, np.uint8)
    L, ctx = _lib.lib(), _lib.ctx()
    _lib.raise_for(L.hb_reorder(ctx, _lib.ptr(c), _lib.dims3(lmap.dims), lmap.stride, _lib.ptr(out)), ctx)
    return out


def inverse_reorder(seq: np.ndarray, lmap: LevelMap) -> np.ndarray:
    if seq.ndim != 1 or seq.size != lmap.count:
        raise FieldError(f"sequence length {seq.size} does not match map point count {lmap.count}")
    s = np.ascontiguousarray(seq, np.uint8)
    out = np.empty(lmap.dims, np.uint8)
    L, ctx = _lib.lib(), _lib.ctx()
    _lib.raise_for(L.hb_inverse_reorder(ctx, _lib.ptr(s), _lib.dims3(lmap.dims), lmap.stride, _lib.ptr(out)), ctx)
    return out
