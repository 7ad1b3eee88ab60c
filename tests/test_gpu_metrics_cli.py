"""Quality metrics on the GPU (k_quality, reference field.py:145-187) and the
command-line front end (reference cli.py:151-240).

The device pass must give numpy's exact numbers: mse = np.mean(d*d) bit for
bit (pairwise summation order), max |d|, and psnr from them; the config-4 RD
sweep (CESM 1800x3600, rel 1e-2 .. 1e-5, CR and TP) must equal the curve the
oracle's archives and numpy metrics give -- CR, bitrate, PSNR, MSE, max error.
"""
import math
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT, has_cuda

pytestmark = pytest.mark.gpu

if not has_cuda():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch  # noqa: E402

import paper_2507_11165_b200 as hb  # noqa: E402
from paper_2507_11165_b200 import cli, synth  # noqa: E402


def np_metrics(o, r):
    d = o.astype(np.float64) - r.astype(np.float64)
    e = float(np.mean(d * d))
    mx = float(np.max(np.abs(d)))
    rng = float(o.max() - o.min())
    p = math.inf if e == 0 else (-math.inf if rng == 0 else 20 * math.log10(rng) - 10 * math.log10(e))
    return e, mx, p


@pytest.mark.parametrize("shape,dt", [((1,), "f32"), ((7,), "f32"), ((100,), "f64"), ((333, 777), "f32"),
                                      ((37, 41, 53), "f64"), ((1800, 3600), "f32"), ((512, 512, 512), "f32"),
                                      ((3, 1 << 20), "f32")])
def test_quality_pass_matches_numpy(shape, dt):
    rng = np.random.default_rng(len(shape) * 7 + shape[-1])
    dtype = np.float32 if dt == "f32" else np.float64
    o = rng.standard_normal(shape).astype(dtype)
    r = (o + rng.uniform(-1e-3, 1e-3, shape)).astype(dtype)
    o3 = o.reshape(shape + (1,) * (3 - len(shape)))
    r3 = r.reshape(o3.shape)
    for fo, fr in ((hb.Field(o3), hb.Field(r3)),
                   (hb.Field(torch.from_numpy(o3).cuda()), hb.Field(torch.from_numpy(r3).cuda()))):
        e, mx, p = np_metrics(o3, r3)
        assert hb.mse(fo, fr) == e
        assert hb.max_abs_error(fo, fr) == mx
        assert hb.psnr(fo, fr) == p
    assert hb.psnr(hb.Field(o3), hb.Field(o3)) == math.inf


def test_quality_report_shape_mismatch():
    a = hb.Field(np.zeros((4, 4, 4), np.float32))
    b = hb.Field(np.zeros((4, 4, 2), np.float32))
    with pytest.raises(hb.FieldError):
        hb.mse(a, b)


def test_config4_rd_curve_identical_to_reference(oracle):
    """BASELINE configs[3]: CESM-shape 1800x3600, rel 1e-2 .. 1e-5, both
    pipelines -- every RD point equal to oracle archive + numpy metrics."""
    oracle.set_threads(0)
    vals = synth.make("grf", (1800, 3600), seed=1)
    f = hb.Field(vals, ndim=2)
    bounds = [1e-2, 1e-3, 1e-4, 1e-5]
    recs = cli.sweep_records(f, "cesm-grf", "rel", bounds, ["cr", "tp"])
    assert len(recs) == 8
    for r in recs:
        ref = oracle.compress(vals, "rel", r.eb_magnitude, r.mode, 2)
        back, _ = oracle.decompress(ref)
        e, mx, p = np_metrics(vals, back.reshape(vals.shape))
        assert r.compressed_bytes == len(ref)
        assert r.cr == vals.nbytes / len(ref)
        assert r.bitrate == 32 / (vals.nbytes / len(ref))
        assert (r.mse, r.max_abs_error, r.psnr_db) == (e, mx, p), (r.eb_magnitude, r.mode)


def run_cli(*argv, cwd=None):
    return subprocess.run([sys.executable, "-m", "paper_2507_11165_b200", *argv], capture_output=True, text=True,
                          cwd=cwd or ROOT, timeout=600)


def test_cli_round_trip_and_analyze(tmp_path, oracle):
    vals = synth.make("grf", (40, 56, 72), seed=3)
    raw = tmp_path / "f.raw"
    raw.write_bytes(vals.astype("<f4").tobytes())
    arc = tmp_path / "f.cszh"
    r = run_cli("compress", "-i", str(raw), "-t", "f32", "-d", "40", "56", "72", "-m", "rel", "-e", "1e-3",
                "-o", str(arc))
    assert r.returncode == 0, r.stderr
    assert arc.read_bytes() == oracle.compress(vals, "rel", 1e-3, "cr", 3)
    out = tmp_path / "f.out"
    r = run_cli("decompress", "-i", str(arc), "-o", str(out))
    assert r.returncode == 0, r.stderr
    back, _ = oracle.decompress(arc.read_bytes())
    assert out.read_bytes() == back.astype("<f4").tobytes()
    r = run_cli("analyze", "-i", str(raw), "-a", str(arc), "--format", "json")
    assert r.returncode == 0, r.stderr
    import json
    rec = json.loads(r.stdout.strip().splitlines()[-1])
    e, mx, p = np_metrics(vals, back.reshape(vals.shape))
    assert (rec["mse"], rec["max_abs_error"], rec["psnr_db"]) == (e, mx, p)
    assert rec["compressed_bytes"] == arc.stat().st_size
    csv_path, svg = tmp_path / "rd.csv", tmp_path / "rd.svg"
    r = run_cli("sweep", "-i", str(raw), "-t", "f32", "-d", "40", "56", "72", "-m", "rel", "-e", "1e-2", "1e-3",
                "--csv", str(csv_path), "--svg", str(svg))
    assert r.returncode == 0, r.stderr
    lines = csv_path.read_text().splitlines()
    assert lines[0].split(",") == cli.RUN_RECORD_COLUMNS and len(lines) == 5
    assert svg.read_text().startswith("<svg")
    r = run_cli("gen", "--kind", "modes", "-d", "16", "24", "32", "-o", str(tmp_path / "g.raw"))
    assert r.returncode == 0 and (tmp_path / "g.raw").stat().st_size == 16 * 24 * 32 * 4


def test_cli_exit_codes(tmp_path):
    raw = tmp_path / "c.raw"
    raw.write_bytes(np.ones(8 * 8 * 8, "<f4").tobytes())
    r = run_cli("compress", "-i", str(raw), "-t", "f32", "-d", "8", "8", "8", "-m", "rel", "-e", "1e-3",
                "-o", str(tmp_path / "c.cszh"))
    assert r.returncode == 4  # rel bound on a constant field
    bad = tmp_path / "bad.cszh"
    bad.write_bytes(b"CSZH" + b"\0" * 10)
    r = run_cli("decompress", "-i", str(bad), "-o", str(tmp_path / "x"))
    assert r.returncode == 5
    r = run_cli("compress", "-i", str(raw), "-t", "f32", "-d", "8", "8", "9", "-m", "abs", "-e", "1e-3",
                "-o", str(tmp_path / "c.cszh"))
    assert r.returncode == 3  # size mismatch
    r = run_cli("decompress", "-i", str(tmp_path / "missing"), "-o", str(tmp_path / "x"))
    assert r.returncode == 6
