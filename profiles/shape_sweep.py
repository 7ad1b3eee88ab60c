"""Device-resident compress / decompress throughput at the BASELINE.json shapes
(configs[1..4]), with the per-phase CUDA-event split of one profiled call.

    python profiles/shape_sweep.py [--steps 5] [--out gpurun_out/sweep.jsonl]

One JSON line per (shape, kind, eb, mode): GB/s of each direction (CUDA events
around the library's stream, 3 warm-ups) and the phase table (hb_profile).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2507_11165_b200 as hb  # noqa: E402
from paper_2507_11165_b200 import _lib, synth  # noqa: E402

CASES = [
    ("nyx", "grf", (512, 512, 512), 1e-3, "cr"),
    ("nyx", "grf", (512, 512, 512), 1e-4, "cr"),
    ("nyx", "grf", (512, 512, 512), 1e-3, "tp"),
    ("nyx", "rough", (512, 512, 512), 1e-3, "cr"),
    ("miranda", "grf", (256, 384, 384), 1e-3, "cr"),
    ("hurricane", "grf", (100, 500, 500), 1e-3, "cr"),
    ("cesm", "grf", (1800, 3600), 1e-2, "cr"),
    ("cesm", "grf", (1800, 3600), 1e-3, "cr"),
    ("cesm", "grf", (1800, 3600), 1e-4, "cr"),
    ("cesm", "grf", (1800, 3600), 1e-5, "cr"),
]


def run(name, kind, dims, eb, mode, steps):
    v = synth.make_device(kind, dims, seed=2025)
    f = hb.Field(v, ndim=len(dims))
    spec = hb.ErrorBoundSpec("rel", eb)
    out = torch.empty(hb.compress_bound(f.dims, 4), dtype=torch.uint8, device="cuda")
    rec = torch.empty_like(v)
    s = torch.cuda.current_stream()
    for _ in range(3):
        a = hb.compress_device(f, spec, mode, out=out)
        hb.decompress_device(a, f.dims, np.float32, ndim=len(dims), out=rec)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    tc = td = 0.0
    for _ in range(steps):
        ev[0].record(s)
        a = hb.compress_device(f, spec, mode, out=out)
        ev[1].record(s)
        hb.decompress_device(a, f.dims, np.float32, ndim=len(dims), out=rec)
        ev[2].record(s)
        torch.cuda.synchronize()
        tc += ev[0].elapsed_time(ev[1])
        td += ev[1].elapsed_time(ev[2])
    nbytes = v.numel() * 4
    _lib.set_profile(True)
    phases = {}
    a = hb.compress_device(f, spec, mode, out=out)
    phases.update({k: round(t, 4) for k, t in _lib.last_phases()})
    hb.decompress_device(a, f.dims, np.float32, ndim=len(dims), out=rec)
    phases.update({k: round(t, 4) for k, t in _lib.last_phases()})
    _lib.set_profile(False)
    return {"case": name, "kind": kind, "dims": list(dims), "eb": eb, "mode": mode,
            "cr": round(nbytes / a.numel(), 3),
            "compress_gbs": round(nbytes * steps / (tc / 1e3) / 1e9, 1),
            "decompress_gbs": round(nbytes * steps / (td / 1e3) / 1e9, 1),
            "compress_ms": round(tc / steps, 4), "decompress_ms": round(td / steps, 4), "phases_ms": phases}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "sweep.jsonl"))
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as fh:
        for c in CASES:
            if a.only and a.only not in c[0]:
                continue
            r = run(*c, a.steps)
            line = json.dumps(r)
            print(line, flush=True)
            fh.write(line + "\n")
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
