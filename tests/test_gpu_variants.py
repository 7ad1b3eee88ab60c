"""Every alternative level-kernel path and scheduling switch stays byte-identical
to the oracle (archive.py:41-74, :121-171).

The production path picks its level kernels by shape (TMA dependency passes,
the axis-0 marching kernel, the 2D tiled kernel); the switches below force the
others so none of them ships untested:
  HB_TILED_LEVELS    column-mapped 3D tile kernel (k_col.cuh) instead of TMA passes
  HB_GENERIC_LEVELS  generic per-phase kernel (k_predict.cu) for every level
  HB_NO_GRAPHS       no CUDA-graph capture/replay of the compress tail / decompress
  HB_NO_FULL_GRAPH   host-driven tuner/level overlap instead of the conditional-node compress graph
  HB_SERIAL_TUNE     tuner and level passes on one stream (no overlap)
  HB_MARCH=1         axis-0 marching level kernel (k_march.cu) for multidim 3D levels
  HB_SWEEP=2 / 1     level 1 as one slab-ordered sweep (persistent / one item per CTA)
                     instead of the seven per-class TMA passes
  HB_SPLIT_TAIL      reducer chain levels 1..3 and the record assembly as four
                     launches instead of the fused k_reduce_tail
  HB_SPLIT_BM_DECODE bitmap decode as header parse + one launch per nested level
                     instead of the fused k_bm_decode_head
"""
import os
import subprocess
import sys

import pytest

from conftest import ROOT, has_cuda

pytestmark = pytest.mark.gpu

if not has_cuda():
    pytest.skip("needs a CUDA device", allow_module_level=True)

VARIANTS = {
    "tiled": {"HB_TILED_LEVELS": "1"},
    "generic": {"HB_GENERIC_LEVELS": "1"},
    "no-graphs": {"HB_NO_GRAPHS": "1"},
    "no-full-graph": {"HB_NO_FULL_GRAPH": "1"},
    "serial-tune": {"HB_SERIAL_TUNE": "1"},
    "march": {"HB_MARCH": "1"},
    "sweep": {"HB_SWEEP": "2"},
    "sweep-one": {"HB_SWEEP": "1"},
    "split-tail": {"HB_SPLIT_TAIL": "1"},
    "split-bm-decode": {"HB_SPLIT_BM_DECODE": "1"},
}


@pytest.mark.parametrize("name", list(VARIANTS))
def test_variant_matches_oracle(name):
    env = dict(os.environ)
    env.update(VARIANTS[name])
    env["HB_VARIANT"] = name
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "_variant_check.py")], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, f"{name}: {r.stdout[-2000:]}\n{r.stderr[-2000:]}"
    assert "variant ok" in r.stdout
