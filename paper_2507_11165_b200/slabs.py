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

import os
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


def _coll_device(group, hint):
    """Collective buffers: CUDA for NCCL, host for gloo."""
    import torch
    import torch.distributed as dist
    if dist.get_backend(group) == "nccl":
        return hint if hint is not None and torch.device(hint).type == "cuda" else torch.device("cuda")
    return torch.device("cpu")


def global_eb_distributed(local_fields, spec: ErrorBoundSpec, dtype, group=None, device=None) -> float:
    """Volume-global abs eb from this rank's slabs: device min/max per slab
    (k_minmax), one all-reduce MAX of (max, -min) -- 2 doubles."""
    import torch
    import torch.distributed as dist
    from .field import min_max
    if spec.mode == "abs":
        return float(spec.magnitude)
    vmax, nmin = -np.inf, -np.inf
    for f in local_fields:
        lo, hi = min_max(f)
        vmax, nmin = max(vmax, float(hi)), max(nmin, -float(lo))
    mm = torch.tensor([vmax, nmin], dtype=torch.float64, device=_coll_device(group, device))
    dist.all_reduce(mm, op=dist.ReduceOp.MAX, group=group)
    dt = np.dtype(dtype)
    return global_abs_eb(spec, dt.type(-mm[1].item()), dt.type(mm[0].item()), dt)


def container_layout(global_dims, ndim: int, precision: int, mode: str, local_ranges, local_sizes, group=None,
                     device=None):
    """All-gather of every slab's (x0, x1, archive length) -- the only exchange
    the container needs -- then the prefix offsets.  Returns (header bytes,
    byte offset of each local archive in the container, total length)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    cdev = _coll_device(group, device)
    k = len(local_ranges)
    counts = torch.tensor([k], dtype=torch.int64, device=cdev)
    allc = [torch.empty_like(counts) for _ in range(world)]
    dist.all_gather(allc, counts, group=group)
    kmax = max(int(c.item()) for c in allc)
    mine = torch.full((kmax, 3), -1, dtype=torch.int64, device=cdev)
    for i, ((x0, x1), n) in enumerate(zip(local_ranges, local_sizes)):
        mine[i] = torch.tensor([x0, x1, n], dtype=torch.int64)
    allv = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(allv, mine, group=group)
    table = sorted(tuple(int(x) for x in row) for t in allv for row in t.tolist() if row[0] >= 0)
    dims = tuple(int(d) for d in global_dims)
    if len(dims) == 2:
        dims = dims + (1,)
    hb = header_bytes(len(table))
    offs, o = {}, hb
    for a, b, n in table:
        offs[a] = o
        o += n
    head = _HEAD.pack(MAGIC, VERSION, ndim, precision, _MODES[mode], 0, len(table), *dims)
    head += b"".join(_ENTRY.pack(a, b, offs[a], n) for a, b, n in table)
    return head, [offs[x0] for x0, _ in local_ranges], o


def compress_distributed_many(local_slabs, global_dims, spec: ErrorBoundSpec, mode: str = "cr", group=None,
                              compress_fn=None, device=None):
    """This rank's slabs [(values, x0), ...] of a multi-GPU slab compression:
    global eb (2-double all-reduce), one archive per slab (no field data
    crosses GPUs), size all-gather.  Returns (archives, offsets, header)."""
    from . import archive
    compress_fn = compress_fn or archive.compress
    ndim = 2 if len(tuple(global_dims)) == 2 else 3
    fields = [Field(v, ndim=ndim) for v, _ in local_slabs]
    dt = fields[0].dtype if fields else np.dtype(np.float32)
    eb = global_eb_distributed(fields, spec, dt, group, device)
    arcs = [compress_fn(f, ErrorBoundSpec("abs", eb), mode) for f in fields]
    ranges = [(x0, x0 + f.dims[0]) for (_, x0), f in zip(local_slabs, fields)]
    head, offs, _ = container_layout(global_dims, ndim, dt.itemsize, mode, ranges, [len(a) for a in arcs], group,
                                     device)
    return arcs, offs, head


def compress_distributed(local_values, x0: int, global_dims, spec: ErrorBoundSpec, mode: str = "cr",
                         group=None, compress_fn=None, device=None):
    """One slab per rank: (archive of this slab, its byte offset in the
    container, container header).  See compress_distributed_many."""
    arcs, offs, head = compress_distributed_many([(local_values, x0)], global_dims, spec, mode, group, compress_fn,
                                                 device)
    return arcs[0], offs[0], head


def _host_bytes(arc) -> bytes:
    if isinstance(arc, (bytes, bytearray, memoryview)):
        return bytes(arc)
    return arc.cpu().numpy().tobytes()  # device archive (compress_device)


def write_container(path: str, head: bytes, archives, offsets, group=None):
    """Offset writes: every rank pwrites its own archives at their prefix
    offsets into one shared file; rank 0 writes the header.  No archive bytes
    cross ranks (the size all-gather already fixed every offset)."""
    import torch.distributed as dist
    rank = dist.get_rank(group)
    if rank == 0:
        with open(path, "wb"):
            pass
    dist.barrier(group=group)
    fd = os.open(path, os.O_WRONLY)
    try:
        if rank == 0:
            os.pwrite(fd, bytes(head), 0)
        for a, o in zip(archives, offsets):
            os.pwrite(fd, _host_bytes(a), o)
    finally:
        os.close(fd)
    dist.barrier(group=group)


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
