"""Generate the golden fixtures that pin the oracle (and through it the CUDA path)
to the reference `hibound` package.

Run ONLY in the build container, where the reference is importable:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/gen_golden.py

Nothing on the GPU box runs this script; the .npz files it writes are committed
and are the only thing the tests read.  Every array stored here is the
reference's own output for the stored input bytes:

  * ``<case>.npz``   -- input field, resolved eb, tune report (chosen config +
    per-level error table), decompose() codes / outliers / anchors, the
    level-grouped sequence, full CR and TP archives, and the decompressed
    values.  Reference entry points: archive.py:41 (compress), :121
    (decompress), tuning.py:105 (tune_report), predictor.py:372 (decompose),
    ordering.py:142 (reorder).
  * ``cfg_<case>.npz`` -- decompose() codes for every uniform InterpConfig and
    a mixed one (predictor parity independent of the tuner).
  * ``stages.npz``   -- byte-exact stage records (stages.py:103-435) for
    adversarial and random inputs, every width.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

import hibound as hb
from hibound import stages
from hibound.ordering import LevelMap, reorder
from hibound.predictor import CUBIC, LINEAR, MULTIDIM, SEQ1D, InterpConfig

HERE = os.path.dirname(os.path.abspath(__file__))


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def field_cases():
    """(name, Field, eb_mode, magnitude) -- mirrors the reference tests'
    fixtures (conftest.py:7-19, test_archive.py, test_acceptance.py) plus the
    SURVEY §8d smoke shapes."""
    g = hb.generate
    out = [
        ("gauss64_rel1e-3", g("gaussian-mix", (64, 64, 64), seed=7, dtype="f32"), "rel", 1e-3),
        ("gauss64_rel1e-5", g("gaussian-mix", (64, 64, 64), seed=7, dtype="f32"), "rel", 1e-5),
        ("affine64_abs1e-3", g("affine", (64, 64, 64), seed=11, dtype="f32"), "abs", 1e-3),
        ("turb64_rel1e-3", g("turbulence-like-spectral", (64, 64, 64), seed=3, dtype="f32"), "rel", 1e-3),
        ("turb48_rel1e-4", g("turbulence-like-spectral", (48, 40, 56), seed=5, dtype="f32"), "rel", 1e-4),
        ("gauss32f64_rel1e-5", g("gaussian-mix", (32, 32, 32), seed=21, dtype="f64"), "rel", 1e-5),
        ("gauss32f64_rel1e-2", g("gaussian-mix", (32, 32, 32), seed=21, dtype="f64"), "rel", 1e-2),
        ("turb2d_96x64_rel1e-4", g("turbulence-like-spectral", (96, 64), seed=2, dtype="f32"), "rel", 1e-4),
        ("gauss2d_180x360_rel1e-3", g("gaussian-mix", (180, 360), seed=1, dtype="f32"), "rel", 1e-3),
        ("turb2d_180x360_rel1e-5", g("turbulence-like-spectral", (180, 360), seed=1, dtype="f32"), "rel", 1e-5),
        ("noise24_abs3e-3", g("uniform-noise", (24, 24, 24), seed=5, dtype="f32"), "abs", 3e-3),
        ("noise24_rel1e-5", g("uniform-noise", (24, 24, 24), seed=5, dtype="f32"), "rel", 1e-5),
        ("noise17f64_rel1e-3", g("uniform-noise", (17, 17, 17), seed=8, dtype="f64"), "rel", 1e-3),
        ("turb33x48x21_rel1e-3", g("turbulence-like-spectral", (33, 48, 21), seed=8, dtype="f32"), "rel", 1e-3),
        ("gauss20x12x9_rel1e-2", g("gaussian-mix", (20, 12, 9), seed=4, dtype="f32"), "rel", 1e-2),
        ("turb33x8x5_rel1e-3", g("turbulence-like-spectral", (33, 8, 5), seed=6, dtype="f64"), "rel", 1e-3),
        ("gauss48x31_rel1e-4", g("gaussian-mix", (48, 31), seed=9, dtype="f32"), "rel", 1e-4),
        ("gauss100x50x50_rel1e-3", g("gaussian-mix", (100, 50, 50), seed=1, dtype="f32"), "rel", 1e-3),
        ("turb40x70x36_rel1e-3", g("turbulence-like-spectral", (40, 70, 36), seed=12, dtype="f32"), "rel", 1e-3),
        ("constant32_abs1e-3", g("constant", (32, 32, 32)), "abs", 1e-3),
    ]
    rng = np.random.default_rng(0)
    out.append(("tiny3x4x2_abs1e-3", hb.Field(np.ascontiguousarray(rng.random((3, 4, 2)))), "abs", 1e-3))
    out.append(("tiny1x1x1_abs1e-1", hb.Field(np.ascontiguousarray(np.array([[[0.25]]], np.float32))), "abs", 1e-1))
    out.append(("line1x9x1_abs1e-2", hb.Field(np.ascontiguousarray(
        np.linspace(0, 1, 9, dtype=np.float32).reshape(1, 9, 1))), "abs", 1e-2))
    # strong variation along x only: pushes the tuner off the default config
    x = np.arange(40, dtype=np.float64)[:, None, None]
    out.append(("sinx40x24x24_abs1e-3", hb.Field(np.ascontiguousarray(
        np.broadcast_to(np.sin(x * 1.3) * 50.0, (40, 24, 24)))), "abs", 1e-3))
    z = np.arange(36, dtype=np.float64)[None, None, :]
    y = np.arange(34, dtype=np.float64)[None, :, None]
    vals = (np.sin(z * 0.9) * 3.0 + np.cos(y * 0.05)) * np.ones((35, 1, 1))
    out.append(("sinz35x34x36_rel1e-3", hb.Field(np.ascontiguousarray(vals.astype(np.float32))), "rel", 1e-3))
    return out


def tune_table(rep):
    errs = np.full((4, 4), np.nan)
    from hibound.tuning import CONFIG_CHOICES
    for level, d in rep.level_errors.items():
        for i, c in enumerate(CONFIG_CHOICES):
            errs[level - 1, i] = d[c]
    return errs


def dump_case(name, f, mode, mag):
    spec = hb.ErrorBoundSpec(mode, mag)
    eb = hb.resolve_error_bound(spec, f)
    rep = hb.tune_report(f, eb)
    qf = hb.decompose(f, eb, rep.chosen)
    lmap = LevelMap(f.dims, qf.anchors.stride)
    seq = reorder(qf.codes, lmap)
    acr = hb.compress(f, spec, "cr")
    atp = hb.compress(f, spec, "tp")
    rec = hb.decompress(acr)
    rec_tp = hb.decompress(atp)
    assert np.array_equal(rec.values, rec_tp.values)
    np.savez_compressed(
        os.path.join(HERE, f"{name}.npz"),
        input=f.values, ndim=np.int64(f.ndim), eb_mode=np.array(mode), mag=np.float64(mag),
        eb=np.float64(eb), cfg=np.frombuffer(rep.chosen.to_bytes(), np.uint8),
        tune_errs=tune_table(rep), n_blocks=np.int64(len(rep.block_origins)),
        oidx=qf.outlier_indices, oval=qf.outlier_values,
        anchors=qf.anchors.values, stride=np.int64(qf.anchors.stride), seq=seq,
        arch_cr=np.frombuffer(acr, np.uint8), arch_tp=np.frombuffer(atp, np.uint8),
        recon_sha256=np.array(sha(rec.values.tobytes())),
    )
    return {
        "dims": list(f.dims), "ndim": f.ndim, "dtype": str(f.dtype), "eb_mode": mode, "mag": mag,
        "eb": eb, "cfg": rep.chosen.to_bytes().hex(), "outliers": int(qf.outlier_indices.size),
        "cr_len": len(acr), "cr_sha256": sha(acr), "tp_len": len(atp), "tp_sha256": sha(atp),
        "input_sha256": sha(f.to_bytes()),
        "cr_escape": hb.section_sizes(acr)["raw_escape"], "tp_escape": hb.section_sizes(atp)["raw_escape"],
    }


ALL_UNIFORM = [InterpConfig(tuple((sp, sc) for _ in range(4)))
               for sp in (CUBIC, LINEAR) for sc in (MULTIDIM, SEQ1D)]
MIXED = InterpConfig(((LINEAR, SEQ1D), (CUBIC, SEQ1D), (LINEAR, MULTIDIM), (CUBIC, MULTIDIM)))


def dump_cfg_case(name, f, mode, mag):
    eb = hb.resolve_error_bound(hb.ErrorBoundSpec(mode, mag), f)
    arrays = {"input": f.values, "eb": np.float64(eb), "ndim": np.int64(f.ndim)}
    for k, cfg in enumerate(ALL_UNIFORM + [MIXED]):
        qf = hb.decompose(f, eb, cfg)
        arrays[f"cfg{k}"] = np.frombuffer(cfg.to_bytes(), np.uint8)
        arrays[f"codes{k}"] = qf.codes
        arrays[f"oidx{k}"] = qf.outlier_indices
        arrays[f"oval{k}"] = qf.outlier_values
        rec = hb.reconstruct(qf, eb, cfg, dims=f.dims, ndim=f.ndim)
        arrays[f"recon_sha256_{k}"] = np.array(sha(rec.values.tobytes()))
    np.savez_compressed(os.path.join(HERE, f"cfg_{name}.npz"), **arrays)


def stage_inputs():
    rng = np.random.default_rng(1234)
    items = [b"", b"\x00", b"\x00" * 4096, b"\xab" * 1000, bytes([0, 1] * 500),
             bytes(range(256)) * 4, b"\x80" * 333, b"\x00" * 65536, b"\x80" * (1 << 16)]
    for n in (1, 2, 3, 7, 8, 9, 17, 63, 64, 65, 100, 255, 511, 513, 1000, 4096, 4097, 20000):
        items.append(rng.integers(0, 256, n, dtype=np.uint8).tobytes())
    # skewed / code-like streams (mostly 128, some neighbours, rare outlier 0)
    for n, p in ((5000, 0.9), (70000, 0.99), (30000, 0.5)):
        a = np.full(n, 128, np.uint8)
        m = rng.random(n) > p
        a[m] = (128 + rng.integers(-6, 7, int(m.sum()))).astype(np.uint8)
        a[rng.random(n) > 0.999] = 0
        items.append(a.tobytes())
    # Fibonacci-like histogram -> long Huffman codes
    fib = [1, 1]
    while len(fib) < 24:
        fib.append(fib[-1] + fib[-2])
    a = np.concatenate([np.full(c, s, np.uint8) for s, c in enumerate(fib)])
    rng.shuffle(a)
    items.append(a.tobytes())
    return items


def dump_stages():
    arrays = {}
    items = stage_inputs()
    arrays["count"] = np.int64(len(items))
    for i, data in enumerate(items):
        arrays[f"in{i}"] = np.frombuffer(data, np.uint8)
        arrays[f"hf{i}"] = np.frombuffer(stages.huffman_encode(data), np.uint8)
        arrays[f"cr{i}"] = np.frombuffer(stages.pipeline_cr_encode(data), np.uint8)
        arrays[f"tp{i}"] = np.frombuffer(stages.pipeline_tp_encode(data), np.uint8)
        for w in stages.WIDTHS:
            arrays[f"tcms{w}_{i}"] = np.frombuffer(stages.tcms_encode(data, w), np.uint8)
            arrays[f"bit{w}_{i}"] = np.frombuffer(stages.bit_shuffle(data, w), np.uint8)
            arrays[f"rre{w}_{i}"] = np.frombuffer(stages.rre_encode(data, w), np.uint8)
            arrays[f"rze{w}_{i}"] = np.frombuffer(stages.rze_encode(data, w), np.uint8)
    np.savez_compressed(os.path.join(HERE, "stages.npz"), **arrays)


def dump_ordering():
    """index_of for every point of a few (dims, stride) pairs (ordering.py:68-84)."""
    arrays = {}
    cases = [((5, 5, 5), 4), ((7, 6, 5), 4), ((9, 9, 9), 8), ((17, 9, 3), 16), ((33, 12, 20), 16),
             ((1, 9, 1), 2), ((13, 6, 5), 8), ((40, 1, 24), 16), ((3, 4, 2), 2), ((1, 1, 1), 1)]
    for k, (dims, a) in enumerate(cases):
        lm = LevelMap(dims, a)
        idx = np.array([[[lm.index_of(x, y, z) for z in range(dims[2])] for y in range(dims[1])]
                        for x in range(dims[0])], np.int64)
        arrays[f"dims{k}"] = np.array(dims, np.int64)
        arrays[f"stride{k}"] = np.int64(a)
        arrays[f"index{k}"] = idx
    arrays["count"] = np.int64(len(cases))
    np.savez_compressed(os.path.join(HERE, "ordering.npz"), **arrays)


def dump_plan_blocks():
    dims_list = [(512, 512, 512), (256, 384, 384), (100, 500, 500), (1800, 3600, 1),
                 (256, 2048, 2048), (64, 64, 64), (17, 17, 17), (32, 32, 32), (9, 40, 12),
                 (128, 96, 1), (100, 300, 40), (200, 90, 64), (48, 48, 48), (321, 123, 77),
                 (2048, 2048, 2048)]
    doc = []
    for d in dims_list:
        origins, shape = hb.plan_blocks(d)
        doc.append({"dims": list(d), "shape": list(shape), "origins": [list(o) for o in origins]})
    with open(os.path.join(HERE, "plan_blocks.json"), "w") as fh:
        json.dump(doc, fh)


def main():
    manifest = {"reference": "/root/reference/pkg (hibound 0.1.0)",
                "python": sys.version.split()[0], "numpy": np.__version__, "cases": {}}
    for name, f, mode, mag in field_cases():
        try:
            manifest["cases"][name] = dump_case(name, f, mode, mag)
        except hb.HiboundError as exc:  # e.g. degenerate bound
            manifest["cases"][name] = {"error": type(exc).__name__}
        print(name, manifest["cases"][name].get("cr_len"), flush=True)
    for name, f, mode, mag in field_cases():
        if name == "gauss64_rel1e-3" or f.count <= 40000:
            dump_cfg_case(name, f, mode, mag)
    dump_stages()
    dump_ordering()
    dump_plan_blocks()
    with open(os.path.join(HERE, "manifest.json"), "w") as fh:
        json.dump(manifest, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
