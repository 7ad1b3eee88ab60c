"""Lossless stages and the two pipelines (reference stages.py), on the GPU.

Records are byte-identical to the reference's; each call runs the
corresponding k_stages.cu kernels through hb_stage_encode / hb_stage_decode.
"""

from __future__ import annotations

import ctypes as C
import struct
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import StageError

STAGE_HUFFMAN, STAGE_RRE, STAGE_RZE, STAGE_TCMS, STAGE_BITSHUFFLE = 1, 2, 3, 4, 5
STAGE_NAMES = {1: "huffman", 2: "rre", 3: "rze", 4: "tcms", 5: "bit"}
WIDTHS = (1, 2, 4, 8)
MAX_BITMAP_DEPTH = 3
_PIPE_CR, _PIPE_TP = 10, 11

_COMMON = struct.Struct("<BBQ")
_BM_EXTRA = struct.Struct("<BQ")
_HF_EXTRA = struct.Struct("<Q")


@dataclass(frozen=True)
class StageHeader:
    stage_id: int
    width: int
    orig_len: int
    header_len: int


def peek_header(blob: bytes) -> StageHeader:
    if len(blob) < _COMMON.size:
        raise StageError("truncated stage header")
    stage, width, orig = _COMMON.unpack_from(blob, 0)
    if stage not in STAGE_NAMES:
        raise StageError(f"unknown stage id {stage}")
    hlen = _COMMON.size + (_HF_EXTRA.size + 256 if stage == STAGE_HUFFMAN else
                           _BM_EXTRA.size if stage in (STAGE_RRE, STAGE_RZE) else 0)
    return StageHeader(stage, width, orig, hlen)


def _check_width(width: int):
    if width not in WIDTHS:
        raise StageError(f"symbol width must be one of {WIDTHS}, got {width}")


def _encode(stage: int, width: int, data: bytes) -> bytes:
    data = bytes(data)
    n = len(data)
    inp = np.frombuffer(data, np.uint8) if n else np.zeros(1, np.uint8)
    cap = 2 * n + 4096
    out = np.empty(cap, np.uint8)
    olen = C.c_size_t()
    L, c = _lib.lib(), _lib.ctx()
    rc = L.hb_stage_encode(c, stage, width, _lib.ptr(inp), n, _lib.ptr(out), cap, C.byref(olen))
    _lib.raise_for(rc, c)
    return out[:olen.value].tobytes()


def _decode(stage: int, blob: bytes, cap: int) -> bytes:
    blob = bytes(blob)
    n = len(blob)
    inp = np.frombuffer(blob, np.uint8) if n else np.zeros(1, np.uint8)
    out = np.empty(max(cap, 1), np.uint8)
    olen = C.c_size_t()
    L, c = _lib.lib(), _lib.ctx()
    rc = L.hb_stage_decode(c, stage, _lib.ptr(inp), n, _lib.ptr(out), cap, C.byref(olen))
    _lib.raise_for(rc, c)
    return out[:olen.value].tobytes()


def _orig_len(blob: bytes) -> int:
    if len(blob) < _COMMON.size:
        raise StageError("truncated stage header")
    return _COMMON.unpack_from(blob, 0)[2]


def tcms_encode(data: bytes, width: int) -> bytes:
    _check_width(width)
    return _encode(STAGE_TCMS, width, data)


def tcms_decode(blob: bytes) -> bytes:
    return _decode(STAGE_TCMS, blob, max(len(blob), 16))


def bit_shuffle(data: bytes, width: int) -> bytes:
    _check_width(width)
    return _encode(STAGE_BITSHUFFLE, width, data)


def bit_unshuffle(blob: bytes) -> bytes:
    return _decode(STAGE_BITSHUFFLE, blob, max(len(blob), 16))


def rre_encode(data: bytes, width: int) -> bytes:
    _check_width(width)
    return _encode(STAGE_RRE, width, data)


def _bitmap_cap(blob: bytes) -> int:
    # the decoded size is the record's orig_len; a valid record expands by at
    # most 8x per bitmap level (1 + 3 nested), so larger claims are corrupt
    return int(min(_orig_len(blob), 8 ** 5 * (len(blob) + 64))) + 64


def rre_decode(blob: bytes) -> bytes:
    return _decode(STAGE_RRE, blob, _bitmap_cap(blob))


def rze_encode(data: bytes, width: int) -> bytes:
    _check_width(width)
    return _encode(STAGE_RZE, width, data)


def rze_decode(blob: bytes) -> bytes:
    return _decode(STAGE_RZE, blob, _bitmap_cap(blob))


def huffman_encode(data: bytes) -> bytes:
    return _encode(STAGE_HUFFMAN, 1, data)


def huffman_decode(blob: bytes) -> bytes:
    # every code is >= 1 bit: a valid record never holds more symbols than payload bits
    orig = _orig_len(blob)
    nb = max(0, len(blob) - (_COMMON.size + _HF_EXTRA.size + 256))
    return _decode(STAGE_HUFFMAN, blob, int(min(orig, 8 * nb + 64)))


def pipeline_cr_encode(data: bytes) -> bytes:
    return _encode(_PIPE_CR, 1, data)


def pipeline_cr_decode(blob: bytes) -> bytes:
    # stage by stage so every output buffer is sized from its record header
    return huffman_decode(rre_decode(tcms_decode(rze_decode(blob))))


def pipeline_tp_encode(data: bytes) -> bytes:
    return _encode(_PIPE_TP, 1, data)


def pipeline_tp_decode(blob: bytes) -> bytes:
    return tcms_decode(bit_unshuffle(rre_decode(blob)))
