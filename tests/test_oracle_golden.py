"""Pins the CPU oracle (oracle/) to the reference's own outputs.

Every fixture under tests/golden/ was produced by the reference package
(tests/golden/gen_golden.py).  The oracle must reproduce them bit for bit:
archives (archive.py:41-74), tune tables (tuning.py:105-150), decompose()
codes/outliers (predictor.py:332-375), reconstruct() (predictor.py:378-416),
the Eq. 3 order (ordering.py:68-84) and every stage record (stages.py).
"""
import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, case_names, cfg_case_names, load_case


def sha(b):
    return hashlib.sha256(b).hexdigest()


@pytest.mark.parametrize("name", case_names())
def test_archives_byte_identical(oracle, name):
    c = load_case(name)
    vals = c["input"]
    ndim = int(c["ndim"])
    mode, mag = str(c["eb_mode"]), float(c["mag"])
    assert oracle.resolve_eb(vals, mode, mag) == float(c["eb"])
    cfg, errs = oracle.tune(vals, float(c["eb"]))
    assert bytes(cfg) == bytes(c["cfg"])
    ge = c["tune_errs"]
    assert np.array_equal(np.isnan(errs), np.isnan(ge))
    assert np.array_equal(errs[~np.isnan(errs)], ge[~np.isnan(ge)])
    for m, key in (("cr", "arch_cr"), ("tp", "arch_tp")):
        blob = oracle.compress(vals, mode, mag, m, ndim)
        assert blob == c[key].tobytes(), (name, m, len(blob), c[key].size)


@pytest.mark.parametrize("name", case_names())
def test_decompress_reference_archives(oracle, name):
    c = load_case(name)
    for key in ("arch_cr", "arch_tp"):
        out, ndim = oracle.decompress(c[key].tobytes())
        assert ndim == int(c["ndim"])
        assert out.dtype == c["input"].dtype
        assert sha(out.tobytes()) == str(c["recon_sha256"])
        assert np.max(np.abs(out.astype(np.float64) - c["input"].astype(np.float64))) <= float(c["eb"])


@pytest.mark.parametrize("name", case_names())
def test_decompose_and_reorder(oracle, name):
    c = load_case(name)
    vals = c["input"]
    codes, oidx, oval, anc = oracle.decompose(vals, float(c["eb"]), c["cfg"])
    assert np.array_equal(oidx, c["oidx"])
    assert np.array_equal(oval, c["oval"])
    assert np.array_equal(anc, c["anchors"])
    seq = oracle.reorder(codes, int(c["stride"]))
    assert np.array_equal(seq, c["seq"])
    back = oracle.inverse_reorder(seq, vals.shape, int(c["stride"]))
    assert np.array_equal(back, codes)


@pytest.mark.parametrize("name", cfg_case_names())
def test_decompose_every_config(oracle, name):
    with np.load(os.path.join(GOLDEN, f"cfg_{name}.npz")) as z:
        c = {k: z[k] for k in z.files}
    vals, eb = c["input"], float(c["eb"])
    for k in range(5):
        codes, oidx, oval, anc = oracle.decompose(vals, eb, c[f"cfg{k}"])
        assert np.array_equal(codes, c[f"codes{k}"]), (name, k)
        assert np.array_equal(oidx, c[f"oidx{k}"])
        assert np.array_equal(oval, c[f"oval{k}"])
        rec = oracle.reconstruct(codes, oidx, oval, anc, eb, c[f"cfg{k}"], vals.shape, vals.dtype)
        assert sha(rec.tobytes()) == str(c[f"recon_sha256_{k}"]), (name, k)


def test_stage_records(oracle):
    with np.load(os.path.join(GOLDEN, "stages.npz")) as z:
        c = {k: z[k] for k in z.files}
    for i in range(int(c["count"])):
        data = c[f"in{i}"].tobytes()
        assert oracle.stage_encode("huffman", data) == c[f"hf{i}"].tobytes(), i
        assert oracle.stage_encode("cr", data) == c[f"cr{i}"].tobytes(), i
        assert oracle.stage_encode("tp", data) == c[f"tp{i}"].tobytes(), i
        assert oracle.stage_decode("cr", c[f"cr{i}"].tobytes()) == data
        assert oracle.stage_decode("tp", c[f"tp{i}"].tobytes()) == data
        assert oracle.stage_decode("huffman", c[f"hf{i}"].tobytes()) == data
        for w in (1, 2, 4, 8):
            for st in ("tcms", "bit", "rre", "rze"):
                rec = c[f"{st}{w}_{i}"].tobytes()
                assert oracle.stage_encode(st, data, w) == rec, (st, w, i)
                assert oracle.stage_decode(st, rec) == data, (st, w, i)


def test_index_of(oracle):
    with np.load(os.path.join(GOLDEN, "ordering.npz")) as z:
        c = {k: z[k] for k in z.files}
    for k in range(int(c["count"])):
        dims = tuple(int(x) for x in c[f"dims{k}"])
        a = int(c[f"stride{k}"])
        idx = c[f"index{k}"]
        for x in range(dims[0]):
            for y in range(dims[1]):
                for z in range(dims[2]):
                    assert oracle.index_of(dims, a, x, y, z) == idx[x, y, z]


def test_plan_blocks(oracle):
    with open(os.path.join(GOLDEN, "plan_blocks.json")) as fh:
        doc = json.load(fh)
    for item in doc:
        origins, shape = oracle.plan_blocks(item["dims"])
        assert list(shape) == item["shape"]
        assert [list(o) for o in origins] == item["origins"]
