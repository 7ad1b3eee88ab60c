"""Host-resident volumes through the GPU with transfers overlapped.

`compress_volume(values, spec, mode, n_slabs)` compresses a host array (numpy,
or a torch CPU tensor -- page-locked for full PCIe speed) into the CSZS slab
container of slabs.py; `decompress_volume(blob)` decodes one back to host
memory.  Both keep the PCIe copy engine busy while the SMs work:

compress
    every slab's host->device copy is queued at once on a copy stream, each
    with an event; slab i's device min/max (k_minmax) runs as soon as its copy
    lands, while the later copies are still in flight.  The volume-global
    rel-eb (field.py:135-142 over the whole volume) is known when the last
    slab's min/max is; then every slab is compressed from HBM and its archive
    (a few MB) queued back to the host.  With an absolute bound slab i
    compresses while slab i+1 is still arriving.  A volume too large for the
    device streams through two slab buffers (a relative bound then costs a
    second host->device pass).
decompress
    slab i is decoded into one of two device slab buffers while slab i-1's
    reconstruction streams back to the host.

Every slab archive equals `hibound.compress(slab, ErrorBoundSpec("abs", eb))`:
the container is byte-identical to slabs.compress_slabs'.  The device checks
every value (FieldError on NaN/Inf from the compress kernels).
"""

from __future__ import annotations

import numpy as np

from . import archive, slabs
from .errors import FieldError
from .field import ErrorBoundSpec, Field, min_max


def _host_tensor(values):
    import torch
    if isinstance(values, torch.Tensor):
        if values.is_cuda:
            raise FieldError("compress_volume takes a host array; use compress_device for CUDA tensors")
        t = values.contiguous()
    else:
        t = torch.from_numpy(np.ascontiguousarray(values))
    if t.dtype not in (torch.float32, torch.float64):
        raise FieldError(f"unsupported precision {t.dtype}; expected float32 or float64")
    return t


def _fits(nbytes: int, frac: float = 0.45) -> bool:
    import torch
    free, _ = torch.cuda.mem_get_info()
    return nbytes <= frac * free


class _Copier:
    """Host->device slab copies on their own stream, each ending in an event;
    the page-locked source stays referenced until the copy is done."""

    def __init__(self, host):
        import torch
        self.torch = torch
        self.host = host
        self.pinned = host.is_pinned()
        self.stream = torch.cuda.Stream()
        self.keep = []

    def issue(self, dst, x0, x1, after=None):
        torch = self.torch
        src = self.host[x0:x1] if self.pinned else self.host[x0:x1].pin_memory()
        self.keep.append(src)
        with torch.cuda.stream(self.stream):
            if after is not None:
                self.stream.wait_event(after)
            dst.copy_(src, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(self.stream)
        return ev


def compress_volume(values, spec: ErrorBoundSpec, mode: str = "cr", n_slabs: int = 8, ndim: int | None = None,
                    resident: bool | None = None) -> bytes:
    """Host volume -> CSZS container, transfers overlapped with compute.
    `resident=None` keeps the whole volume on the device when it fits (one
    host->device pass even for a relative bound)."""
    import torch
    host = _host_tensor(values)
    if host.dim() == 2:
        host = host.reshape(tuple(host.shape) + (1,))
        ndim = 2
    if host.dim() != 3:
        raise FieldError("values must be a 2- or 3-axis array")
    ndim = ndim or 3
    dims = tuple(int(d) for d in host.shape)
    dt = np.dtype(np.float32 if host.dtype == torch.float32 else np.float64)
    bounds = slabs.slab_bounds(dims[0], n_slabs)
    if resident is None:
        resident = _fits(host.numel() * host.element_size())
    comp = torch.cuda.current_stream()
    cp = _Copier(host)
    rel = spec.mode == "rel"

    def gmin_max(views_and_events):
        lo, hi = np.inf, -np.inf
        for view, ev in views_and_events:
            comp.wait_event(ev)
            a, b = min_max(Field(view, ndim=ndim))  # k_minmax on this slab while later copies run
            lo, hi = min(lo, float(a)), max(hi, float(b))
        return slabs.global_abs_eb(spec, dt.type(lo), dt.type(hi), dt)

    archives = []
    if resident:
        dev = torch.empty(dims, dtype=host.dtype, device="cuda")
        evs = [cp.issue(dev[x0:x1], x0, x1) for x0, x1 in bounds]  # all queued at once
        eb = gmin_max([(dev[x0:x1], ev) for (x0, x1), ev in zip(bounds, evs)]) if rel else float(spec.magnitude)
        aspec = ErrorBoundSpec("abs", eb)
        pend = []
        for (x0, x1), ev in zip(bounds, evs):
            comp.wait_event(ev)
            arc = archive.compress_device(Field(dev[x0:x1], ndim=ndim), aspec, mode)
            h = torch.empty(arc.numel(), dtype=torch.uint8, pin_memory=True)
            done = torch.cuda.Event()
            done.record(comp)
            with torch.cuda.stream(cp.stream):
                cp.stream.wait_event(done)
                h.copy_(arc, non_blocking=True)
            pend.append((h, arc))
        cp.stream.synchronize()
        archives = [h.numpy().tobytes() for h, _ in pend]
    else:
        rows = max(x1 - x0 for x0, x1 in bounds)
        bufs = [torch.empty((rows,) + dims[1:], dtype=host.dtype, device="cuda") for _ in range(2)]

        def stream_slabs(work):
            """slab i+1 copies into the other buffer while `work` runs on slab i"""
            free = [None, None]
            pending = cp.issue(bufs[0][: bounds[0][1] - bounds[0][0]], *bounds[0])
            for i, (x0, x1) in enumerate(bounds):
                ev = pending
                if i + 1 < len(bounds):
                    a, b = bounds[i + 1]
                    pending = cp.issue(bufs[(i + 1) % 2][: b - a], a, b, after=free[(i + 1) % 2])
                comp.wait_event(ev)
                work(bufs[i % 2][: x1 - x0])
                free[i % 2] = torch.cuda.Event()
                free[i % 2].record(comp)

        eb = float(spec.magnitude)
        if rel:
            acc = [np.inf, -np.inf]

            def mm(view):
                a, b = min_max(Field(view, ndim=ndim))
                acc[0], acc[1] = min(acc[0], float(a)), max(acc[1], float(b))

            stream_slabs(mm)
            eb = slabs.global_abs_eb(spec, dt.type(acc[0]), dt.type(acc[1]), dt)
        aspec = ErrorBoundSpec("abs", eb)
        stream_slabs(lambda view: archives.append(
            archive.compress_device(Field(view, ndim=ndim), aspec, mode).cpu().numpy().tobytes()))
    return slabs.assemble(dims, ndim, dt.itemsize, mode, bounds, archives)


def decompress_volume(blob: bytes, out=None) -> Field:
    """CSZS container -> host Field; slab i decodes while slab i-1 streams out.
    `out` may be a page-locked torch CPU tensor of the volume's shape."""
    import torch
    data = bytes(blob)
    dims, ndim, prec, mode, ents = slabs.parse(data)
    tdt = torch.float32 if prec == 4 else torch.float64
    npdt = np.float32 if prec == 4 else np.float64
    if out is None:
        out = torch.empty(dims, dtype=tdt, pin_memory=True)
    out = out.reshape(dims)
    comp = torch.cuda.current_stream()
    copy = torch.cuda.Stream()
    rows = max(x1 - x0 for x0, x1, _, _ in ents)
    bufs = [torch.empty((rows,) + tuple(dims[1:]), dtype=tdt, device="cuda") for _ in range(2)]
    freed = [None, None]
    for i, (x0, x1, off, ln) in enumerate(ents):
        b = bufs[i % 2][: x1 - x0]
        if freed[i % 2] is not None:
            comp.wait_event(freed[i % 2])  # the buffer's previous slab has left for the host
        arc = torch.from_numpy(np.frombuffer(data, np.uint8, ln, off).copy()).cuda()
        archive.decompress_device(arc, (x1 - x0,) + tuple(dims[1:]), npdt, out=b)
        ready = torch.cuda.Event()
        ready.record(comp)
        with torch.cuda.stream(copy):
            copy.wait_event(ready)
            out[x0:x1].copy_(b, non_blocking=True)
            e = torch.cuda.Event()
            e.record(copy)
        freed[i % 2] = e
    copy.synchronize()
    vals = out.numpy()
    return Field._trusted(vals, ndim)
