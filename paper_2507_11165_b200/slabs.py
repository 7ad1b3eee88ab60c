"""Axis-0 slab sharding of large volumes.

A single CSZH archive does not shard (every level needs a +-3s halo of the
level above and the Huffman/bitmap streams need global prefix sums), so a
large volume is cut into independent axis-0 slabs.  Each slab becomes an
ordinary reference-format archive -- `hibound.decompress` reads it -- and a
small container records where each slab sits:

    magic "CSZS" | version u8 | ndim u8 | precision u8 | mode u8 | axis u8 (0)
    | n_slabs u32 | global dims 3 x u64
    | n_slabs x (x0 u64, x1 u64, offset u64, length u64)   offsets from container start
    | concatenated CSZH archives

Relative error bounds keep whole-volume semantics: the slabs share
abs eb = mag * float(max - min) over the whole volume (field.py:135-142), so
`slab_archive_i == hibound.compress(slab_i, ErrorBoundSpec("abs", eb), mode)`.
In the distributed driver the only collectives are one all-reduce of
(max, -min) and one all-gather of the archive sizes; no field data moves
between GPUs.
"""

from __future__ import annotations

import struct

import numpy as np

from .errors import ArchiveError, DegenerateBoundError
from .field import ErrorBoundSpec, Field

MAGIC = b"CSZS"
VERSION = 1
_HEAD = struct.Struct("<4sBBBBBI3Q")
_ENTRY = struct.Struct("<4Q")
_MODES = {"cr": 0, "tp": 1}


def slab_bounds(d0: int, n_slabs: int):
    """Even split of axis 0 into n_slabs contiguous [x0, x1) ranges."""
    if n_slabs < 1 or n_slabs > d0:
        raise ValueError(f"n_slabs must be in [1, {d0}], got {n_slabs}")
    base, extra = divmod(d0, n_slabs)
    out, x = [], 0
    for i in range(n_slabs):
        n = base + (1 if i < extra else 0)
        out.append((x, x + n))
        x += n
    return out


def global_abs_eb(spec: ErrorBoundSpec, vmin, vmax, dtype) -> float:
    """field.py:135-142 from a (min, max) pair; the subtraction in the field dtype."""
    if spec.mode == "abs":
        return float(spec.magnitude)
    rng = float(np.asarray(vmax, dtype) - np.asarray(vmin, dtype))
    if rng == 0.0:
        raise DegenerateBoundError("relative error bound on a constant field (value range 0)")
    return float(spec.magnitude) * rng


def assemble(dims, ndim: int, precision: int, mode: str, bounds, archives) -> bytes:
    """Container bytes from per-slab archives (same order as bounds)."""
    n = len(archives)
    off = _HEAD.size + n * _ENTRY.size
    head = _HEAD.pack(MAGIC, VERSION, ndim, precision, _MODES[mode], 0, n, *[int(d) for d in dims])
    entries = []
    for (x0, x1), a in zip(bounds, archives):
        entries.append(_ENTRY.pack(x0, x1, off, len(a)))
        off += len(a)
    return head + b"".join(entries) + b"".join(bytes(a) for a in archives)


def header_bytes(n_slabs: int) -> int:
    return _HEAD.size + n_slabs * _ENTRY.size


def parse(blob: bytes):
    """-> (dims, ndim, precision, mode, [(x0, x1, offset, length)])"""
    if len(blob) < _HEAD.size:
        raise ArchiveError("slab container truncated in header")
    magic, ver, ndim, prec, mode, axis, n, d0, d1, d2 = _HEAD.unpack_from(blob, 0)
    if magic != MAGIC or ver != VERSION or axis != 0 or mode not in (0, 1):
        raise ArchiveError("not a CSZS slab container")
    if len(blob) < _HEAD.size + n * _ENTRY.size:
        raise ArchiveError("slab container truncated in slab table")
    ents = [_ENTRY.unpack_from(blob, _HEAD.size + i * _ENTRY.size) for i in range(n)]
    x = 0
    for x0, x1, o, ln in ents:
        if x0 != x or x1 <= x0 or o + ln > len(blob):
            raise ArchiveError("corrupt slab table")
        x = x1
    if x != d0:
        raise ArchiveError("slabs do not cover axis 0")
    return (d0, d1, d2), ndim, prec, ("cr" if mode == 0 else "tp"), ents


def compress_slabs(field: Field, spec: ErrorBoundSpec, mode: str = "cr", n_slabs: int = 2,
                   compress_fn=None) -> bytes:
    """Single-process slab container (e.g. one GPU compressing slabs in turn)."""
    from . import archive
    compress_fn = compress_fn or archive.compress
    from .field import min_max
    v = field.values
    vmin, vmax = min_max(field) if spec.mode == "rel" else (0.0, 1.0)
    eb = global_abs_eb(spec, vmin, vmax, field.dtype)
    bounds = slab_bounds(field.dims[0], n_slabs)
    abs_spec = ErrorBoundSpec("abs", eb)
    arcs = [compress_fn(Field(v[x0:x1], ndim=field.ndim), abs_spec, mode) for x0, x1 in bounds]
    return assemble(field.dims, field.ndim, field.dtype.itemsize, mode, bounds, arcs)


def decompress_slabs(blob: bytes, decompress_fn=None) -> Field:
    from . import archive
    decompress_fn = decompress_fn or archive.decompress
    dims, ndim, prec, mode, ents = parse(blob)
    out = np.empty(dims, np.float32 if prec == 4 else np.float64)
    for x0, x1, o, ln in ents:
        f = decompress_fn(blob[o:o + ln])
        out[x0:x1] = f.values if isinstance(f, Field) else f
    return Field._trusted(out, ndim)


def compress_distributed(local_values, x0: int, global_dims, spec: ErrorBoundSpec, mode: str = "cr",
                         group=None, compress_fn=None, device=None):
    """One rank's part of a multi-GPU slab compression.

    local_values: this rank's slab (numpy array or torch tensor), rows
    [x0, x0 + len) of the global volume.  Collectives (torch.distributed, NCCL
    on GPUs / gloo on CPU): all-reduce MAX of (max, -min) for the global eb,
    all-gather of (x0, x1, archive length).  Returns (archive bytes of this
    slab, byte offset of this archive in the container, container header
    bytes).  Rank 0 can write the header and every rank its archive at its
    offset (pwrite / shared buffer) -- see gather_container for a
    single-writer variant.
    """
    import torch
    import torch.distributed as dist
    from . import archive
    compress_fn = compress_fn or archive.compress
    world = dist.get_world_size(group)
    from .field import min_max
    is_t = isinstance(local_values, torch.Tensor)
    dev = device or (local_values.device if is_t else torch.device("cpu"))
    ndim0 = 2 if len(tuple(global_dims)) == 2 else 3
    lo, hi = min_max(Field(local_values, ndim=ndim0))
    vmin, vmax = float(lo), float(hi)
    np_dtype = np.dtype(np.float32) if (local_values.dtype in (np.float32, torch.float32)) else np.dtype(np.float64)
    mm = torch.tensor([vmax, -vmin], dtype=torch.float64, device=dev)
    dist.all_reduce(mm, op=dist.ReduceOp.MAX, group=group)
    gmax, gmin = mm[0].item(), -mm[1].item()
    eb = global_abs_eb(spec, np_dtype.type(gmin), np_dtype.type(gmax), np_dtype)
    ndim = 2 if len(tuple(global_dims)) == 2 else 3
    f = Field(local_values, ndim=ndim)
    arc = compress_fn(f, ErrorBoundSpec("abs", eb), mode)
    mine = torch.tensor([x0, x0 + f.dims[0], len(arc)], dtype=torch.int64, device=dev)
    allv = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(allv, mine, group=group)
    table = sorted(tuple(int(x) for x in t.tolist()) for t in allv)
    bounds = [(a, b) for a, b, _ in table]
    sizes = [n for _, _, n in table]
    dims = tuple(int(d) for d in global_dims)
    if len(dims) == 2:
        dims = dims + (1,)
    hb = header_bytes(world)
    offs, o = [], hb
    for n in sizes:
        offs.append(o)
        o += n
    my = [i for i, (a, b) in enumerate(bounds) if a == x0][0]
    head = assemble(dims, ndim, np_dtype.itemsize, mode, bounds, [b"\0" * n for n in sizes])[:hb]
    return arc, offs[my], head


def gather_container(arc: bytes, x0: int, head: bytes, group=None, dst: int = 0):
    """Collect every rank's archive at `dst`; returns the full container there (None elsewhere)."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    objs = [None] * world if dist.get_rank(group) == dst else None
    dist.gather_object((int(x0), bytes(arc)), objs, dst=dst, group=group)
    if objs is None:
        return None
    by_x0 = dict(objs)
    body = []
    for sx0, sx1, off, ln in parse_table(head):
        a = by_x0[sx0]
        if len(a) != ln:
            raise ArchiveError("archive size changed between all-gather and gather")
        body.append(a)
    return bytes(head) + b"".join(body)


def parse_table(head: bytes):
    n = _HEAD.unpack_from(head, 0)[6]
    return [_ENTRY.unpack_from(head, _HEAD.size + i * _ENTRY.size) for i in range(n)]
