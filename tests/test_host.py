"""CPU-only checks: the C-ABI library loads and exports every symbol the
header declares (no compute calls), and the host-side mirror of the reference
interface (config bytes, LevelMap closed form, block plan, header parsing)
agrees with the reference's goldens."""
import json
import os
import re

import numpy as np
import pytest

from conftest import GOLDEN, ROOT, case_names, load_case

import paper_2507_11165_b200 as hb
from paper_2507_11165_b200 import _lib


def header_symbols():
    with open(os.path.join(ROOT, "include", "hibound_b200.h")) as fh:
        src = fh.read()
    return sorted(set(re.findall(r"HB_API\s+[\w\s\*]+?\b(hb_\w+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    import ctypes
    L = ctypes.CDLL(_lib.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(L, s), s


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_archive_info_without_gpu():
    import ctypes as C
    for name in case_names()[:6]:
        c = load_case(name)
        blob = c["arch_cr"].tobytes()
        s = hb.section_sizes(blob)
        assert s["total_bytes"] == len(blob)
        assert s["header_bytes"] + s["anchor_bytes"] + s["outlier_bytes"] + s["stream_bytes"] == len(blob)
        assert s["outlier_count"] == c["oidx"].size
        assert s["abs_eb"] == float(c["eb"])
        for cut in (0, 10, 45, 46, len(blob) // 2, len(blob) - 1):
            with pytest.raises(hb.ArchiveError, match="archive truncated in "):
                hb.section_sizes(blob[:cut])
        # like the reference (archive.py:174-200) the walk ignores trailing bytes
        assert hb.section_sizes(blob + b"\0")["total_bytes"] == len(blob) + 1
        bad = bytearray(blob)
        bad[0] ^= 0xFF
        with pytest.raises(hb.ArchiveError, match="bad magic"):
            hb.section_sizes(bytes(bad))


def test_section_sizes_messages_match_reference():
    """Messages observed from hibound.section_sizes on the affine 64^3 golden."""
    blob = load_case("affine64_abs1e-3")["arch_cr"].tobytes()
    expect = {0: "archive truncated in header", 45: "archive truncated in header",
              46: "archive truncated in anchor count", len(blob) // 2: "archive truncated in anchor values"}
    for cut, msg in expect.items():
        with pytest.raises(hb.ArchiveError) as e:
            hb.section_sizes(blob[:cut])
        assert str(e.value) == msg
    bad = bytearray(blob)
    bad[0] ^= 0xFF
    with pytest.raises(hb.ArchiveError) as e:
        hb.section_sizes(bytes(bad))
    assert str(e.value) == "bad magic b'\\xbcSZH'"


def test_interp_config_bytes():
    cfgs = [hb.InterpConfig(((sp, sc),) * 4) for sp in ("cubic", "linear") for sc in ("multidim", "seq1d")]
    assert [c.to_bytes() for c in cfgs] == [b"\0" * 4, b"\2" * 4, b"\1" * 4, b"\3" * 4]
    for c in cfgs:
        assert hb.InterpConfig.from_bytes(c.to_bytes()) == c
    with pytest.raises(hb.ArchiveError):
        hb.InterpConfig.from_bytes(b"\x04\0\0\0")


def test_level_map_against_reference_index():
    with np.load(os.path.join(GOLDEN, "ordering.npz")) as z:
        c = {k: z[k] for k in z.files}
    for k in range(int(c["count"])):
        dims = tuple(int(x) for x in c[f"dims{k}"])
        lm = hb.LevelMap(dims, int(c[f"stride{k}"]))
        idx = c[f"index{k}"]
        for x in range(dims[0]):
            for y in range(dims[1]):
                for z in range(dims[2]):
                    assert lm.index_of(x, y, z) == idx[x, y, z]
    lm = hb.LevelMap((5, 5, 5), 4)
    assert (lm.index_of(0, 0, 0), lm.index_of(2, 0, 0), lm.index_of(1, 0, 0), lm.prefixes[0]) == (0, 13, 43, 27)


def test_plan_blocks_against_reference():
    with open(os.path.join(GOLDEN, "plan_blocks.json")) as fh:
        doc = json.load(fh)
    for item in doc:
        origins, shape = hb.plan_blocks(item["dims"])
        assert list(shape) == item["shape"]
        assert [list(o) for o in origins] == item["origins"]


def test_anchor_stride_and_scalar_helpers():
    assert hb.effective_anchor_stride((64, 64, 64)) == 16
    assert hb.effective_anchor_stride((15, 64, 64)) == 8
    assert hb.effective_anchor_stride((5, 5, 1)) == 4
    assert hb.effective_anchor_stride((1, 1, 1)) == 1
    assert hb.quantize(0.0, 1e-3) == (128, False)
    assert hb.quantize(2e-3, 1e-3) == (129, False)
    assert hb.quantize(300e-3, 1e-3) == (0, True)
    v, o = hb.interpolate_1d([(-3, 1.0), (-1, 1.0), (1, 1.0), (3, 1.0)], "cubic")
    assert v == 1.0 and o == 4


def test_field_validation():
    with pytest.raises(hb.FieldError):
        hb.Field(np.array([[[np.nan]]], np.float32))
    with pytest.raises(hb.FieldError):
        hb.Field(np.zeros((2, 2), np.float32))
    with pytest.raises(hb.DegenerateBoundError):
        hb.ErrorBoundSpec("rel", 0.0)
    f = hb.Field.from_array(np.zeros((4, 5), np.float32))
    assert f.ndim == 2 and f.dims == (4, 5, 1)


def test_gpu_path_fails_loudly_without_cuda():
    from conftest import has_cuda
    if has_cuda():
        pytest.skip("has a GPU")
    with pytest.raises(RuntimeError):
        hb.compress(hb.Field(np.zeros((4, 4, 4), np.float32)), hb.ErrorBoundSpec("abs", 1e-3))


def test_cli_parser_mirrors_reference():
    """Sub-commands, flags and run-record columns of reference cli.py:236-333."""
    from paper_2507_11165_b200 import cli
    p = cli.build_parser()
    a = p.parse_args(["compress", "-i", "x", "-t", "f32", "-d", "4", "5", "6", "-m", "rel", "-e", "1e-3", "-o", "y"])
    assert (a.command, a.mode, tuple(a.dims), a.error_mode, a.error_bound) == ("compress", "cr", (4, 5, 6), "rel",
                                                                               1e-3)
    a = p.parse_args(["sweep", "-i", "x", "--dataset", "cesm-atm", "-m", "rel", "-e", "1e-2", "1e-3", "--csv", "o"])
    assert a.modes == ["cr", "tp"] and a.error_bounds == [1e-2, 1e-3]
    assert set(cli.COMMANDS) == {"compress", "decompress", "analyze", "sweep", "gen"}
    assert len(cli.RUN_RECORD_COLUMNS) == 24 and cli.RUN_RECORD_COLUMNS[14] == "psnr_db"
    with pytest.raises(SystemExit) as e:
        cli.main(["compress", "-i", "x", "-m", "rel", "-e", "1", "-o", "y"])  # no -t / -d
    assert e.value.code == 2
    svg = cli.rd_svg({"cr": [(1.0, 40.0), (2.0, 60.0)], "tp": [(1.5, float("inf"))]})
    assert svg.startswith("<svg") and svg.count("<polyline") == 1


def test_modes_generator_is_per_global_coordinate():
    """synth.make_modes: any axis-0 slab equals the same rows of the whole
    volume (config-5 slabs are generated independently per GPU)."""
    import torch
    from paper_2507_11165_b200 import synth
    full = synth.make_modes((24, 20, 18), seed=5, device="cpu")
    parts = [synth.make_modes((b - a, 20, 18), seed=5, x0=a, global_dims=(24, 20, 18), device="cpu")
             for a, b in ((0, 7), (7, 16), (16, 24))]
    assert torch.equal(torch.cat(parts), full)
