"""One compress + decompress step inside a cudaProfilerStart/Stop range, for
the ncu launch lists under profiles/ (after warm-up calls that build the
graphs):

    ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \\
        --csv --log-file launches.csv python profiles/step_probe.py [nx ny nz | nx ny] [rel_eb] [grf|rough|gauss]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2507_11165_b200 as hb  # noqa: E402
from paper_2507_11165_b200 import synth  # noqa: E402

args = sys.argv[1:]
dims = tuple(int(a) for a in args if a.isdigit()) or (512, 512, 512)
kinds = [a for a in args if a in ("grf", "rough", "gauss")]
ebs = [a for a in args if not a.isdigit() and a not in kinds]
spec = hb.ErrorBoundSpec("rel", float(ebs[0]) if ebs else 1e-3)
f = hb.Field(synth.make_device(kinds[0] if kinds else "grf", dims, seed=2025), ndim=len(dims))
for _ in range(4):
    a = hb.compress_device(f, spec, "cr")
    hb.decompress_device(a, f.dims, np.float32)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
a = hb.compress_device(f, spec, "cr")
hb.decompress_device(a, f.dims, np.float32)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
