"""Error behaviour of the CUDA path mirrors the reference's exceptions
(test_archive.py:79-122, test_stages.py:99-103,180-192)."""
import numpy as np
import pytest

from conftest import has_cuda, load_case

pytestmark = pytest.mark.gpu

if not has_cuda():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2507_11165_b200 as hb  # noqa: E402


@pytest.fixture(scope="module")
def blob32():
    c = load_case("gauss32f64_rel1e-2")
    return c["arch_cr"].tobytes()


def test_constant_field_relative_eb_fails():
    f = hb.Field(np.ones((64, 64, 64), np.float32))
    with pytest.raises(hb.DegenerateBoundError):
        hb.compress(f, hb.ErrorBoundSpec("rel", 1e-3), "cr")


def test_nan_on_device_is_field_error():
    import torch
    v = torch.rand((40, 40, 40), device="cuda")
    v[3, 5, 7] = float("nan")
    with pytest.raises(hb.FieldError):
        hb.compress_device(hb.Field(v), hb.ErrorBoundSpec("abs", 1e-3))
    v[3, 5, 7] = float("inf")
    with pytest.raises(hb.FieldError):
        hb.compress_device(hb.Field(v), hb.ErrorBoundSpec("rel", 1e-3))


def test_bad_mode():
    with pytest.raises(ValueError):
        hb.compress(hb.Field(np.zeros((8, 8, 8), np.float32)), hb.ErrorBoundSpec("abs", 1e-3), "zz")


def test_bad_magic_and_version(blob32):
    b = bytearray(blob32)
    b[0] ^= 0xFF
    with pytest.raises(hb.ArchiveError):
        hb.decompress(bytes(b))
    b = bytearray(blob32)
    b[4] = 99
    with pytest.raises(hb.ArchiveError):
        hb.decompress(bytes(b))


def test_truncations_fail_cleanly(blob32):
    for cut in (0, 3, 10, 45, 46, 100, len(blob32) // 2, len(blob32) - 1):
        with pytest.raises(hb.ArchiveError):
            hb.decompress(blob32[:cut])


def test_trailing_garbage_rejected(blob32):
    with pytest.raises(hb.ArchiveError):
        hb.decompress(blob32 + b"\x00")


def test_stream_corruption_is_detected_or_bounded():
    c = load_case("turb64_rel1e-3")
    blob = c["arch_cr"].tobytes()
    info = hb.section_sizes(blob)
    rng = np.random.default_rng(0)
    start = len(blob) - info["stream_bytes"]
    for _ in range(20):
        b = bytearray(blob)
        pos = start + int(rng.integers(0, info["stream_bytes"]))
        b[pos] ^= 1 << int(rng.integers(0, 8))
        try:
            out = hb.decompress(bytes(b))
        except hb.ArchiveError:
            continue
        assert out.dims == info["dims"]


def test_orphan_outlier_marker():
    c = load_case("gauss64_rel1e-5")
    blob = bytearray(c["arch_cr"].tobytes())
    info = hb.section_sizes(bytes(blob))
    assert info["outlier_count"] > 1
    # drop the last outlier record: count and section shrink, stream unchanged
    off = info["header_bytes"] - 16 + info["anchor_bytes"] + 8
    k = info["outlier_count"]
    rec = 8 + info["precision"]
    cnt_off = 46 + 8 + info["anchor_bytes"]
    new = bytearray(blob[:cnt_off]) + (k - 1).to_bytes(8, "little") + blob[cnt_off + 8:cnt_off + 8 + (k - 1) * rec] \
        + blob[cnt_off + 8 + k * rec:]
    with pytest.raises(hb.ArchiveError):
        hb.decompress(bytes(new))
    del off


def test_stage_errors():
    st = hb.stages
    enc = bytearray(st.rre_encode(b"\x01\x02", 1))
    enc[19] &= 0x7F  # clear the first-symbol bit
    with pytest.raises(hb.StageError):
        st.rre_decode(bytes(enc))
    enc = st.huffman_encode(np.random.default_rng(6).integers(0, 256, 512, dtype=np.uint8).tobytes())
    with pytest.raises(hb.StageError):
        st.huffman_decode(enc[:-3])
    enc = bytearray(st.huffman_encode(bytes(range(16)) * 8))
    table = np.frombuffer(bytes(enc[18:274]), np.uint8).copy()
    table[np.flatnonzero(table)] = 1
    enc[18:274] = table.tobytes()
    with pytest.raises(hb.StageError):
        st.huffman_decode(bytes(enc))
    with pytest.raises(hb.StageError):
        st.pipeline_tp_decode(st.pipeline_cr_encode(b"hello world"))
    with pytest.raises(hb.StageError):
        st.tcms_encode(b"x", 3)


def test_raw_escape_round_trip():
    f = hb.Field(np.random.default_rng(5).random((24, 24, 24)).astype(np.float32))
    for mode in ("cr", "tp"):
        blob = hb.compress(f, hb.ErrorBoundSpec("abs", 3e-3), mode)
        s = hb.section_sizes(blob)
        assert s["raw_escape"] and s["stream_bytes"] == f.count
        out = hb.decompress(blob)
        assert hb.max_abs_error(f, out) <= 3e-3


def test_device_archive_decompress_matches_host():
    import torch
    c = load_case("turb33x48x21_rel1e-3")
    blob = c["arch_tp"].tobytes()
    dev = torch.frombuffer(bytearray(blob), dtype=torch.uint8).cuda()
    out = hb.decompress_device(dev, c["input"].shape, c["input"].dtype)
    host = hb.decompress(blob)
    assert np.array_equal(out.values.cpu().numpy(), host.values)


def test_decompress_device_checks_header():
    """dims / dtype / ndim given by the caller must match the archive header
    (a float64 request for an f32 archive is refused, not reinterpreted)."""
    import torch
    from paper_2507_11165_b200 import synth
    vals = synth.make("grf", (20, 24, 28), seed=2)
    arch = hb.compress_device(hb.Field(torch.from_numpy(vals).cuda()), hb.ErrorBoundSpec("rel", 1e-3))
    r = hb.decompress_device(arch)
    assert r.values.shape == (20, 24, 28) and r.values.dtype == torch.float32 and r.ndim == 3
    with pytest.raises(ValueError):
        hb.decompress_device(arch, (20, 24, 28), np.float64)
    with pytest.raises(ValueError):
        hb.decompress_device(arch, (20, 24, 28), np.float32, ndim=2)


def test_concurrent_compress_threads(oracle):
    """compress() is reentrant: threads compressing different
    fields at once each get their own context and staging buffer."""
    import threading
    from paper_2507_11165_b200 import synth
    fields = [synth.make(k, d, seed=s) for k, d, s in
              (("grf", (40, 50, 60), 1), ("rough", (33, 48, 21), 2), ("gauss", (64, 64, 64), 3),
               ("grf", (300, 400), 4))]
    refs = [oracle.compress(v, "rel", 1e-3, "cr", v.ndim) for v in fields]
    backs = [oracle.decompress(r)[0] for r in refs]
    spec = hb.ErrorBoundSpec("rel", 1e-3)
    errors = []

    def work(i):
        try:
            for _ in range(4):
                blob = hb.compress(hb.Field(fields[i], ndim=fields[i].ndim), spec, "cr")
                if blob != refs[i]:
                    errors.append(i)
                out = hb.decompress(refs[i])  # decompress is reentrant too
                if not np.array_equal(out.values.reshape(-1), backs[i].reshape(-1)):
                    errors.append(f"decompress {i}")
            hb._lib.release_contexts()
        except Exception as e:  # pragma: no cover - reported below
            errors.append(repr(e))

    ts = [threading.Thread(target=work, args=(i,)) for i in range(len(fields))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors
