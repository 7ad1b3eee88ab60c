"""GPU vs the pinned CPU oracle on seeded inputs larger than the goldens,
plus size-independent properties at the benchmark size (512^3)."""
import numpy as np
import pytest

from conftest import has_cuda

pytestmark = pytest.mark.gpu

if not has_cuda():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2507_11165_b200 as hb  # noqa: E402
from paper_2507_11165_b200 import synth  # noqa: E402


CASES = [
    ("grf", (96, 80, 112), "rel", 1e-3, "f32"),
    ("grf", (130, 66, 97), "rel", 1e-4, "f32"),
    ("gauss", (128, 128, 128), "rel", 1e-3, "f32"),
    ("rough", (64, 96, 80), "rel", 1e-3, "f32"),
    ("rough", (50, 120, 110), "rel", 1e-2, "f64"),
    ("grf", (600, 900), "rel", 1e-3, "f32"),
    ("rough", (333, 777), "rel", 1e-5, "f32"),
    ("grf", (256, 384, 20), "abs", 2e-3, "f32"),
]


@pytest.mark.parametrize("kind,dims,ebm,mag,dt", CASES)
def test_archive_matches_oracle(oracle, kind, dims, ebm, mag, dt):
    vals = synth.make(kind, dims, seed=11, dtype=dt)
    f = hb.Field(vals, ndim=len(dims))
    spec = hb.ErrorBoundSpec(ebm, mag)
    for mode in ("cr", "tp"):
        blob = hb.compress(f, spec, mode)
        ref = oracle.compress(vals, ebm, mag, mode, len(dims))
        assert len(blob) == len(ref), (kind, dims, mode)
        assert blob == ref, (kind, dims, mode)
        out = hb.decompress(blob)
        back, _ = oracle.decompress(blob)
        assert np.array_equal(out.values, back.reshape(out.values.shape))
        eb = oracle.resolve_eb(vals, ebm, mag)
        assert np.max(np.abs(out.values.astype(np.float64) - f.values.astype(np.float64))) <= eb


def test_512_cubed_properties():
    import torch
    vals = synth.make_device("grf", (512, 512, 512), seed=2025)
    f = hb.Field(vals)
    spec = hb.ErrorBoundSpec("rel", 1e-3)
    a_cr = hb.compress_device(f, spec, "cr").clone()
    a_tp = hb.compress_device(f, spec, "tp").clone()
    assert torch.equal(hb.compress_device(f, spec, "cr"), a_cr)  # deterministic
    info = hb.section_sizes(a_cr.cpu().numpy().tobytes())
    r_cr = hb.decompress_device(a_cr, f.dims, np.float32)
    r_tp = hb.decompress_device(a_tp, f.dims, np.float32)
    assert torch.equal(r_cr.values, r_tp.values)  # CR/TP reconstructions identical
    err = (r_cr.values.double() - vals.double()).abs().max().item()
    assert err <= info["abs_eb"]


@pytest.mark.parametrize("dims", [(12, 70, 65), (16, 48, 40), (9, 33, 200), (5, 300, 310)])
def test_thin_field_whole_block_tuner(oracle, dims):
    """min dim < 17: the tuner's single block is the whole field (tuning.py:74-75)."""
    vals = synth.make("grf", dims, seed=4)
    f = hb.Field(vals)
    eb = oracle.resolve_eb(vals, "rel", 1e-3)
    cfg, errs = oracle.tune(vals, eb)
    rep = hb.tune_report(f, eb)
    assert rep.chosen.to_bytes() == bytes(cfg)
    for level, e in rep.level_errors.items():
        for i, c in enumerate(hb.tuning.CONFIG_CHOICES):
            assert e[c] == errs[level - 1, i]
    for mode in ("cr", "tp"):
        assert hb.compress(f, hb.ErrorBoundSpec("rel", 1e-3), mode) == oracle.compress(vals, "rel", 1e-3, mode, 3)


# every interpolation config per level on shapes with many interior blocks:
# exercises the TMA dependency passes (k_pass.cu) for all four stencil /
# scheme combinations, all seq1d axis orders, even and odd E rows (direct vs
# gathered class-0 lattice), f32 and f64
CFG_SHAPES = [
    ((70, 90, 100), "f32"),   # seq1d order z, y, x; even E rows
    ((100, 66, 97), "f32"),   # order x, z, y; odd E rows -> gathered lattice
    ((48, 120, 40), "f64"),   # order y, x, z
]
CFGS = [bytes([0, 0, 0, 0]), bytes([1, 1, 1, 1]), bytes([2, 2, 2, 2]), bytes([3, 3, 3, 3]), bytes([2, 1, 3, 0])]


@pytest.mark.parametrize("dims,dt", CFG_SHAPES)
def test_forced_configs_match_oracle(oracle, dims, dt):
    vals = synth.make("grf", dims, seed=21, dtype=dt)
    f = hb.Field(vals)
    eb = oracle.resolve_eb(vals, "rel", 1e-3)
    for cb in CFGS:
        cfg = hb.InterpConfig.from_bytes(cb)
        qf = hb.decompose(f, eb, cfg)
        codes, oidx, oval, anchors = oracle.decompose(vals, eb, list(cb))
        assert np.array_equal(qf.codes.reshape(-1), codes.reshape(-1)), (dims, cb)
        assert np.array_equal(qf.outlier_indices, oidx), (dims, cb)
        assert np.array_equal(qf.outlier_values, oval), (dims, cb)
        rec = hb.reconstruct(qf, eb, cfg, dims=f.dims, ndim=f.ndim)
        ref = oracle.reconstruct(codes, oidx, oval, anchors, eb, list(cb), dims, vals.dtype)
        assert np.array_equal(rec.values.reshape(-1), ref.reshape(-1)), (dims, cb)


def test_interleaved_calls_reuse_state_correctly(oracle):
    """Context state carried between calls (resident compress tables, graph
    replays, the shared arena, the in-stream archive copy into a caller's
    device buffer) never changes an archive: interleave two shapes, both
    modes, decompressions and a stage call, compare every archive with the
    oracle's."""
    import torch
    va = synth.make("grf", (40, 56, 72), seed=3)
    vb = synth.make("rough", (33, 48, 21), seed=4)
    ref = {("a", "cr"): oracle.compress(va, "rel", 1e-3, "cr", 3), ("b", "tp"): oracle.compress(vb, "rel", 1e-3, "tp", 3)}
    recon = {km: oracle.decompress(blob)[0] for km, blob in ref.items()}
    fields = {"a": hb.Field(torch.from_numpy(va).cuda()), "b": hb.Field(torch.from_numpy(vb).cuda())}
    spec = hb.ErrorBoundSpec("rel", 1e-3)
    bufs = {k: torch.full((hb.compress_bound(f.dims, 4),), 0xA5, dtype=torch.uint8, device="cuda")
            for k, f in fields.items()}
    for rnd in range(3):
        for (k, mode) in (("a", "cr"), ("a", "cr"), ("b", "tp"), ("a", "cr"), ("b", "tp"), ("b", "tp")):
            out = hb.compress_device(fields[k], spec, mode, out=bufs[k] if rnd % 2 else None)
            assert out.cpu().numpy().tobytes() == ref[(k, mode)], (rnd, k, mode)
            if rnd >= 1:  # rounds 1 and 2 replay the recorded decompress graphs
                back = hb.decompress_device(out, fields[k].dims, np.float32)
                assert np.array_equal(back.values.cpu().numpy(), recon[(k, mode)]), (rnd, k, mode)
        hb.stages.huffman_encode(bytes(range(256)) * 3)
    assert hb.compress(hb.Field(va), spec, "cr") == ref[("a", "cr")]
