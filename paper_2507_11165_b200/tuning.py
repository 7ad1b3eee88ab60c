"""Sampling auto-tuner API (reference tuning.py).

Block planning is deterministic host integer logic; the trials, the
pairwise/Neumaier error sums and the argmin run on the GPU (k_tune.cu) via
hb_tune.
"""

from __future__ import annotations

import json
import math
import os
from dataclasses import dataclass

import numpy as np

from . import _lib
from .field import Field
from .predictor import CUBIC, LINEAR, MULTIDIM, SEQ1D, InterpConfig, effective_anchor_stride

BLOCK_EDGE = 17
SAMPLE_FRACTION = 0.002
CONFIG_CHOICES = ((CUBIC, MULTIDIM), (CUBIC, SEQ1D), (LINEAR, MULTIDIM), (LINEAR, SEQ1D))


def worker_count() -> int:
    """HIBOUND_THREADS (tuning.py:32-38); the GPU tuner ignores it, results are identical."""
    try:
        return max(1, int(os.environ.get("HIBOUND_THREADS", "")))
    except ValueError:
        return 1


@dataclass(frozen=True)
class TuneReport:
    anchor_stride: int
    block_origins: tuple
    block_shape: tuple
    level_errors: dict
    chosen: InterpConfig

    def to_json(self) -> str:
        levels = {}
        for level in sorted(self.level_errors, reverse=True):
            errs = self.level_errors[level]
            levels[str(level)] = {"errors": {f"{sp}-{sc}": e for (sp, sc), e in errs.items()},
                                  "chosen": "-".join(self.chosen.level(level))}
        doc = {"anchor_stride": self.anchor_stride, "block_shape": list(self.block_shape),
               "block_origins": [list(o) for o in self.block_origins], "levels": levels}
        return json.dumps(doc, indent=2, sort_keys=True)


def _ceil_blocks(total_points: int, block_points: int) -> int:
    return max(1, -(-(total_points * 2) // (block_points * 1000)))


def plan_blocks(dims):
    """Evenly spaced, non-overlapping 17^3 origins on the 16-lattice (tuning.py:66-97)."""
    dims = tuple(int(d) for d in dims)
    nondeg = [d for d in dims if d > 1]
    if not nondeg or min(nondeg) < BLOCK_EDGE:
        return [(0, 0, 0)], dims
    shape = tuple(BLOCK_EDGE if d > 1 else 1 for d in dims)
    axes = [[0] if d == 1 else list(range(0, d - b + 1, 16)) for d, b in zip(dims, shape)]
    cand = [(x, y, z) for x in axes[0] for y in axes[1] for z in axes[2]]
    m = len(cand)
    want = min(m, _ceil_blocks(dims[0] * dims[1] * dims[2], shape[0] * shape[1] * shape[2]))
    if want == 1:
        picked = [cand[m // 2]]
    else:
        picked = [cand[i] for i in sorted({(i * (m - 1)) // (want - 1) for i in range(want)})]
    kept = []
    for o in picked:
        if all(any(abs(o[a] - p[a]) >= shape[a] for a in range(3)) for p in kept):
            kept.append(o)
    return kept, shape


def tune_report(field: Field, eb: float) -> TuneReport:
    L, c = _lib.lib(), _lib.ctx()
    v = field.values
    prec = field.dtype.itemsize
    cfg = np.zeros(4, np.uint8)
    errs = np.zeros(16, np.float64)
    rc = L.hb_tune(c, _lib.ptr(v), prec, _lib.dims3(field.dims), float(eb), _lib.ptr(cfg), _lib.ptr(errs))
    _lib.raise_for(rc, c)
    origins, shape = plan_blocks(field.dims)
    top = effective_anchor_stride(shape).bit_length() - 1
    level_errors = {}
    for level in range(top, 0, -1):
        level_errors[level] = {cfgc: float(errs[(level - 1) * 4 + i]) for i, cfgc in enumerate(CONFIG_CHOICES)}
    chosen = InterpConfig.from_bytes(bytes(cfg))
    return TuneReport(anchor_stride=effective_anchor_stride(shape), block_origins=tuple(origins),
                      block_shape=shape, level_errors=level_errors, chosen=chosen)


def tune(field: Field, eb: float) -> InterpConfig:
    return tune_report(field, eb).chosen
