"""Slab container and the distributed slab driver.

CPU tests: the per-slab compressor is injected (the oracle, test-only) so the
host logic -- bounds, global eb all-reduce, size all-gather, offsets,
container layout -- runs on gloo with world_size 2.  The GPU test runs the
real CUDA compressor.
"""
import os
import socket

import numpy as np
import pytest

from conftest import has_cuda

import paper_2507_11165_b200 as hb
from paper_2507_11165_b200 import slabs, synth


def oracle_compress(f, spec, mode):
    from oracle import oracle
    return oracle.compress(np.ascontiguousarray(f.values), spec.mode, spec.magnitude, mode, f.ndim)


def oracle_decompress(blob):
    from oracle import oracle
    out, _ = oracle.decompress(blob)
    return out


def test_slab_bounds():
    assert slabs.slab_bounds(10, 3) == [(0, 4), (4, 7), (7, 10)]
    assert slabs.slab_bounds(8, 8)[-1] == (7, 8)
    with pytest.raises(ValueError):
        slabs.slab_bounds(4, 5)


def test_container_round_trip_single_process(oracle):
    vals = synth.make("grf", (48, 40, 36), seed=3)
    f = hb.Field(vals)
    spec = hb.ErrorBoundSpec("rel", 1e-3)
    blob = slabs.compress_slabs(f, spec, "cr", 3, compress_fn=oracle_compress)
    dims, ndim, prec, mode, ents = slabs.parse(blob)
    assert dims == (48, 40, 36) and ndim == 3 and prec == 4 and mode == "cr" and len(ents) == 3
    eb = oracle.resolve_eb(vals, "rel", 1e-3)
    for (x0, x1, o, n) in ents:  # every slab is a plain reference-format archive
        ref = oracle.compress(np.ascontiguousarray(vals[x0:x1]), "abs", eb, "cr", 3)
        assert blob[o:o + n] == ref
    out = slabs.decompress_slabs(blob, decompress_fn=oracle_decompress)
    assert np.max(np.abs(out.values.astype(np.float64) - vals)) <= eb
    with pytest.raises(hb.ArchiveError):
        slabs.parse(blob[:20])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, vals, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    bounds = slabs.slab_bounds(vals.shape[0], world)
    x0, x1 = bounds[rank]
    spec = hb.ErrorBoundSpec("rel", 1e-3)
    arc, off, head = slabs.compress_distributed(np.ascontiguousarray(vals[x0:x1]), x0, vals.shape, spec, "tp",
                                                compress_fn=oracle_compress)
    full = slabs.gather_container(arc, x0, head)
    q.put((rank, off, len(arc), full))
    dist.destroy_process_group()


def test_distributed_gloo_world2(oracle):
    import multiprocessing as mp
    vals = synth.make("rough", (40, 33, 30), seed=5)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, vals, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in ps:
        p.join(timeout=60)
    res.sort()
    full = res[0][3]
    assert full is not None and res[1][3] is None
    single = slabs.compress_slabs(hb.Field(vals), hb.ErrorBoundSpec("rel", 1e-3), "tp", 2,
                                  compress_fn=oracle_compress)
    assert full == single  # same bytes as the single-process container
    dims, ndim, prec, mode, ents = slabs.parse(full)
    assert [(o, n) for _, _, o, n in ents] == [(res[0][1], res[0][2]), (res[1][1], res[1][2])]


@pytest.mark.gpu
@pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")
def test_gpu_slab_container_matches_oracle(oracle):
    vals = synth.make("grf", (64, 48, 40), seed=9)
    f = hb.Field(vals)
    spec = hb.ErrorBoundSpec("rel", 1e-3)
    gpu = slabs.compress_slabs(f, spec, "cr", 4)
    ref = slabs.compress_slabs(f, spec, "cr", 4, compress_fn=oracle_compress)
    assert gpu == ref
    out = slabs.decompress_slabs(gpu)
    assert np.max(np.abs(out.values.astype(np.float64) - vals)) <= oracle.resolve_eb(vals, "rel", 1e-3)


def _worker_many(rank, world, port, vals, q, path, use_gpu):
    """Two slabs per rank (the config-5 layout at small size): global eb
    all-reduce, size all-gather, offset writes into one shared file."""
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    bounds = slabs.slab_bounds(vals.shape[0], 2 * world)[2 * rank:2 * rank + 2]
    spec = hb.ErrorBoundSpec("rel", 1e-3)
    if use_gpu:
        import torch
        local = [(torch.from_numpy(np.ascontiguousarray(vals[a:b])).cuda(), a) for a, b in bounds]
        fn = hb.compress_device
    else:
        local = [(np.ascontiguousarray(vals[a:b]), a) for a, b in bounds]
        fn = oracle_compress
    arcs, offs, head = slabs.compress_distributed_many(local, vals.shape, spec, "cr", compress_fn=fn)
    slabs.write_container(path, head, arcs, offs)
    q.put((rank, offs, [len(a) for a in arcs]))
    dist.destroy_process_group()


def _run_many(vals, path, use_gpu):
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker_many, args=(r, 2, port, vals, q, path, use_gpu)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(2))
    for p in ps:
        p.join(timeout=60)
    return res


def test_distributed_offset_writes_gloo_world2(oracle, tmp_path):
    vals = synth.make("grf", (44, 30, 26), seed=6)
    path = str(tmp_path / "c.cszs")
    _run_many(vals, path, use_gpu=False)
    blob = open(path, "rb").read()
    single = slabs.compress_slabs(hb.Field(vals), hb.ErrorBoundSpec("rel", 1e-3), "cr", 4,
                                  compress_fn=oracle_compress)
    assert blob == single  # offset-written file == single-process container


@pytest.mark.gpu
@pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")
def test_gpu_distributed_world2_matches_oracle(oracle, tmp_path):
    """Two ranks (gloo; one GPU shared) drive the CUDA compressor on CUDA
    tensors; the offset-written container equals the oracle's, slab by slab."""
    vals = synth.make_modes((64, 96, 80), seed=4, device="cuda").cpu().numpy()
    path = str(tmp_path / "g.cszs")
    _run_many(vals, path, use_gpu=True)
    blob = open(path, "rb").read()
    ref = slabs.compress_slabs(hb.Field(vals), hb.ErrorBoundSpec("rel", 1e-3), "cr", 4, compress_fn=oracle_compress)
    assert blob == ref
    out = slabs.decompress_slabs(blob)
    assert np.max(np.abs(out.values.astype(np.float64) - vals)) <= oracle.resolve_eb(vals, "rel", 1e-3)


@pytest.mark.gpu
@pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")
def test_gpu_config5_slab_matches_oracle(oracle):
    """One full config-5 slab (rows 768..1024 of the 2048^3 field, generated
    on the GPU from global coordinates) byte-identical to the oracle under the
    volume-global eb -- the per-slab parity behind bench.py's config5 line."""
    import torch
    oracle.set_threads(0)
    g = (2048, 2048, 2048)
    v = synth.make_modes((256, 2048, 2048), seed=2048, x0=768, global_dims=g)
    # global eb from all 8 slabs' min/max (as the bench computes it)
    lo, hi = np.inf, -np.inf
    for x0 in range(0, 2048, 256):
        s = v if x0 == 768 else synth.make_modes((256, 2048, 2048), seed=2048, x0=x0, global_dims=g)
        lo, hi = min(lo, float(s.min())), max(hi, float(s.max()))
        del s
    eb = slabs.global_abs_eb(hb.ErrorBoundSpec("rel", 1e-3), np.float32(lo), np.float32(hi), np.float32)
    f = hb.Field(v)
    arch = hb.compress_device(f, hb.ErrorBoundSpec("abs", eb), "cr")
    host = v.cpu().numpy()
    ref = oracle.compress(host, "abs", eb, "cr", 3)
    assert arch.cpu().numpy().tobytes() == ref
    back, _ = oracle.decompress(ref)
    out = hb.decompress_device(arch, f.dims, np.float32)
    assert np.array_equal(out.values.cpu().numpy().reshape(-1), back.reshape(-1))
    del v, f, arch, out
    torch.cuda.empty_cache()


@pytest.mark.gpu
@pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")
@pytest.mark.parametrize("resident", [True, False])
@pytest.mark.parametrize("ebm,mode", [("rel", "cr"), ("abs", "tp")])
def test_gpu_streamed_volume_matches_oracle(oracle, resident, ebm, mode):
    """streaming.compress_volume (host volume, copies overlapped with the
    per-slab min/max and compress) writes the same container as the oracle
    slab by slab; decompress_volume returns the oracle's reconstruction."""
    import torch
    from paper_2507_11165_b200 import streaming
    vals = synth.make("grf", (72, 40, 52), seed=12)
    spec = hb.ErrorBoundSpec(ebm, 1e-3 if ebm == "rel" else 2e-4)
    host = torch.from_numpy(vals).pin_memory() if resident else vals
    blob = streaming.compress_volume(host, spec, mode, n_slabs=5, resident=resident)
    ref = slabs.compress_slabs(hb.Field(vals), spec, mode, 5, compress_fn=oracle_compress)
    assert blob == ref
    out = streaming.decompress_volume(blob)
    assert np.array_equal(out.values, slabs.decompress_slabs(ref, decompress_fn=oracle_decompress).values)


@pytest.mark.gpu
@pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")
def test_gpu_streamed_volume_2d(oracle):
    from paper_2507_11165_b200 import streaming
    vals = synth.make("rough", (300, 410), seed=3)
    spec = hb.ErrorBoundSpec("rel", 1e-3)
    blob = streaming.compress_volume(vals, spec, "cr", n_slabs=3, ndim=2)
    ref = slabs.compress_slabs(hb.Field(vals, ndim=2), spec, "cr", 3, compress_fn=oracle_compress)
    assert blob == ref
    out = streaming.decompress_volume(blob)
    assert out.ndim == 2 and np.array_equal(out.values, slabs.decompress_slabs(ref, decompress_fn=oracle_decompress).values)
