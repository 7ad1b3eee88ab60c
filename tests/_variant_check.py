"""Subprocess body of test_gpu_variants.py: compress/decompress a set of
seeded fields through the CUDA path under whatever HB_* switches the parent
put in the environment, and compare every archive and reconstruction with
the oracle byte for byte.  Exit code 0 = all equal; prints the first
mismatch otherwise.  (The switches are read once per process by the
library, hence the subprocess.)"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2507_11165_b200 as hb  # noqa: E402
from oracle import oracle  # noqa: E402
from paper_2507_11165_b200 import synth  # noqa: E402

CASES = [
    ("grf", (96, 80, 112), 1e-3, "f32"),
    ("rough", (64, 96, 80), 1e-3, "f32"),
    ("grf", (130, 66, 97), 1e-4, "f32"),
    ("gauss", (70, 90, 100), 1e-3, "f32"),
    ("rough", (50, 120, 110), 1e-2, "f64"),
    ("grf", (600, 900), 1e-3, "f32"),
    ("rough", (333, 777), 1e-5, "f32"),
    ("grf", (33, 48, 21), 1e-3, "f32"),
]


def main() -> int:
    oracle.build()
    oracle.set_threads(0)
    spec = hb.ErrorBoundSpec("rel", 1e-3)
    n = 0
    for kind, dims, mag, dt in CASES:
        vals = synth.make(kind, dims, seed=11, dtype=dt)
        spec = hb.ErrorBoundSpec("rel", mag)
        f_dev = hb.Field(torch.from_numpy(vals).cuda(), ndim=len(dims))
        for mode in ("cr", "tp"):
            ref = oracle.compress(vals, "rel", mag, mode, len(dims))
            back, _ = oracle.decompress(ref)
            for rep in range(4):  # later calls: graph capture / replays where enabled
                arch = hb.compress_device(f_dev, spec, mode)
                if arch.cpu().numpy().tobytes() != ref:
                    print(f"archive mismatch {kind} {dims} {dt} {mode} rep {rep}")
                    return 1
                out = hb.decompress_device(arch, f_dev.dims, vals.dtype, ndim=len(dims))
                if not np.array_equal(out.values.cpu().numpy().reshape(-1), back.reshape(-1)):
                    print(f"reconstruction mismatch {kind} {dims} {dt} {mode} rep {rep}")
                    return 1
                n += 1
    print(f"variant ok: {n} compress/decompress pairs byte-identical", os.environ.get("HB_VARIANT", ""))
    return 0


if __name__ == "__main__":
    sys.exit(main())
