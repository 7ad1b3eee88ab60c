"""GPU parity: the CUDA path (through the C ABI) against the reference's own
golden outputs (tests/golden/) and against the pinned CPU oracle on larger
seeded inputs.  Bit-exact for codes, outliers, stage records and archives;
decompressed values bit-identical to the reference's and within eb."""
import hashlib
import os

import numpy as np
import pytest

from conftest import GOLDEN, case_names, cfg_case_names, has_cuda, load_case

pytestmark = pytest.mark.gpu

if not has_cuda():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2507_11165_b200 as hb  # noqa: E402


def sha(b):
    return hashlib.sha256(b).hexdigest()


def field_of(c):
    return hb.Field(np.ascontiguousarray(c["input"]), ndim=int(c["ndim"]))


@pytest.mark.parametrize("name", case_names())
def test_compress_matches_reference_archive(name):
    c = load_case(name)
    f = field_of(c)
    spec = hb.ErrorBoundSpec(str(c["eb_mode"]), float(c["mag"]))
    for mode, key in (("cr", "arch_cr"), ("tp", "arch_tp")):
        blob = hb.compress(f, spec, mode)
        ref = c[key].tobytes()
        assert len(blob) == len(ref), (name, mode)
        assert blob == ref, (name, mode)


@pytest.mark.parametrize("name", case_names())
def test_decompress_reference_archive(name):
    c = load_case(name)
    for key in ("arch_cr", "arch_tp"):
        out = hb.decompress(c[key].tobytes())
        assert out.ndim == int(c["ndim"])
        assert out.dtype == c["input"].dtype
        assert sha(out.values.tobytes()) == str(c["recon_sha256"]), (name, key)
        err = np.max(np.abs(out.values.astype(np.float64) - c["input"].astype(np.float64)))
        assert err <= float(c["eb"])


@pytest.mark.parametrize("name", case_names())
def test_tune_report_matches(name):
    c = load_case(name)
    f = field_of(c)
    rep = hb.tune_report(f, float(c["eb"]))
    assert rep.chosen.to_bytes() == bytes(c["cfg"])
    ge = c["tune_errs"]
    for level, errs in rep.level_errors.items():
        for i, cfg in enumerate(hb.tuning.CONFIG_CHOICES):
            assert errs[cfg] == ge[level - 1, i], (name, level, cfg)


@pytest.mark.parametrize("name", case_names())
def test_decompose_outliers_and_seq(name):
    c = load_case(name)
    f = field_of(c)
    qf = hb.decompose(f, float(c["eb"]), hb.InterpConfig.from_bytes(bytes(c["cfg"])))
    assert np.array_equal(qf.outlier_indices, c["oidx"])
    assert np.array_equal(qf.outlier_values, c["oval"])
    assert np.array_equal(qf.anchors.values, c["anchors"])
    lm = hb.LevelMap(f.dims, qf.anchors.stride)
    assert np.array_equal(hb.reorder(qf.codes, lm), c["seq"])


@pytest.mark.parametrize("name", cfg_case_names())
def test_decompose_reconstruct_every_config(name):
    with np.load(os.path.join(GOLDEN, f"cfg_{name}.npz")) as z:
        c = {k: z[k] for k in z.files}
    f = hb.Field(np.ascontiguousarray(c["input"]), ndim=int(c["ndim"]))
    eb = float(c["eb"])
    for k in range(5):
        cfg = hb.InterpConfig.from_bytes(bytes(c[f"cfg{k}"]))
        qf = hb.decompose(f, eb, cfg)
        assert np.array_equal(qf.codes, c[f"codes{k}"]), (name, k)
        assert np.array_equal(qf.outlier_indices, c[f"oidx{k}"])
        assert np.array_equal(qf.outlier_values, c[f"oval{k}"])
        rec = hb.reconstruct(qf, eb, cfg, dims=f.dims, ndim=f.ndim)
        assert sha(rec.values.tobytes()) == str(c[f"recon_sha256_{k}"]), (name, k)


def test_stage_records():
    with np.load(os.path.join(GOLDEN, "stages.npz")) as z:
        c = {k: z[k] for k in z.files}
    st = hb.stages
    for i in range(int(c["count"])):
        data = c[f"in{i}"].tobytes()
        assert st.huffman_encode(data) == c[f"hf{i}"].tobytes(), i
        assert st.huffman_decode(c[f"hf{i}"].tobytes()) == data, i
        assert st.pipeline_cr_encode(data) == c[f"cr{i}"].tobytes(), i
        assert st.pipeline_tp_encode(data) == c[f"tp{i}"].tobytes(), i
        assert st.pipeline_cr_decode(c[f"cr{i}"].tobytes()) == data, i
        assert st.pipeline_tp_decode(c[f"tp{i}"].tobytes()) == data, i
        for w in (1, 2, 4, 8):
            assert st.tcms_encode(data, w) == c[f"tcms{w}_{i}"].tobytes(), (i, w)
            assert st.tcms_decode(c[f"tcms{w}_{i}"].tobytes()) == data
            assert st.bit_shuffle(data, w) == c[f"bit{w}_{i}"].tobytes(), (i, w)
            assert st.bit_unshuffle(c[f"bit{w}_{i}"].tobytes()) == data
            assert st.rre_encode(data, w) == c[f"rre{w}_{i}"].tobytes(), (i, w)
            assert st.rre_decode(c[f"rre{w}_{i}"].tobytes()) == data
            assert st.rze_encode(data, w) == c[f"rze{w}_{i}"].tobytes(), (i, w)
            assert st.rze_decode(c[f"rze{w}_{i}"].tobytes()) == data


def test_fused_pipeline_decode_entry_points():
    """hb_stage_decode(HB_PIPE_CR / HB_PIPE_TP) in one call: the CR pipeline's
    Huffman workspace is laid out for the capacity-bounded intermediate record,
    which for compressible inputs is far larger than the input record."""
    from paper_2507_11165_b200 import stages as st
    rng = np.random.default_rng(5)
    cases = [bytes(200_000), (bytes([128]) * 90_000 + bytes(range(256)) * 40),
             rng.integers(120, 137, 300_000).astype(np.uint8).tobytes(), b"x"]
    for data in cases:
        cr = st.pipeline_cr_encode(data)
        tp = st.pipeline_tp_encode(data)
        assert st._decode(st._PIPE_CR, cr, len(data) + 64) == data
        assert st._decode(st._PIPE_TP, tp, len(data) + 64) == data


def test_huffman_encode_tile_paths(oracle):
    """Warp-tile encoder paths vs the oracle (stages.py:293-329): tiles denser
    than 8 bits/symbol (global OR path), lanes whose 32 codes exceed 128 bits
    (per-code shared-memory path), ragged tails, a single symbol."""
    from paper_2507_11165_b200 import stages as st
    rng = np.random.default_rng(17)
    # near-uniform over 256 symbols: half the codes get 9 bits; sorting puts
    # whole tiles of 9-bit symbols together
    freq = np.where(np.arange(256) < 128, 1100, 900)
    uni = np.repeat(np.arange(256, dtype=np.uint8), freq)
    long_first = np.concatenate([uni[uni >= 128], uni[uni < 128]])
    # Fibonacci-skewed: codes up to ~24 bits, rare symbols clustered per lane
    fib = [1, 1]
    while len(fib) < 26:
        fib.append(fib[-1] + fib[-2])
    skew = np.repeat(np.arange(26, dtype=np.uint8), fib[::-1])
    cases = [long_first.tobytes(), rng.permutation(uni).tobytes(), skew.tobytes(),
             rng.permutation(skew)[:77_777].tobytes(), bytes([7]) * 5000, b"\x01", b"\x02\x03" * 513,
             rng.integers(0, 256, 1023).astype(np.uint8).tobytes()]
    for i, data in enumerate(cases):
        ref = oracle.stage_encode("huffman", data)
        assert st.huffman_encode(data) == ref, i
        assert st.huffman_decode(ref) == data, i


def test_huffman_codes_longer_than_32_bits(oracle):
    """Fibonacci frequencies over 36 symbols give canonical codes of up to 35
    bits: the encoder's per-code path for tables with codes > 32 bits and the
    decoder's beyond-LUT path, against the oracle (stages.py:246-329)."""
    from paper_2507_11165_b200 import stages as st
    fib = [1, 1]
    while len(fib) < 36:
        fib.append(fib[-1] + fib[-2])
    counts = fib[::-1]  # symbol 0 most frequent
    data = np.repeat(np.arange(36, dtype=np.uint8), counts)
    data = np.random.default_rng(9).permutation(data).tobytes()
    ref = oracle.stage_encode("huffman", data)
    assert max(ref[18:18 + 256]) >= 33  # some code is longer than 32 bits
    assert st.huffman_encode(data) == ref
    assert st.huffman_decode(ref) == data
