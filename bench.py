#!/usr/bin/env python
"""Benchmark: cuSZ-Hi compress + decompress round trip on B200.

Workload (BASELINE.json configs[1]): Nyx-shape 512^3 f32 synthetic Gaussian
random field (SURVEY §8d "GRF-k"), rel-eb 1e-3, CR pipeline.  One step = one
compress (resolve eb -> tune -> predict/quantize/reorder -> Huffman/RRE4/
TCMS8/RZE1 -> archive, incl. the size read-back) plus one decompress of that
archive.  `value` = input bytes of all ranks / (compress + decompress time),
device-resident buffers; compress_gbs / decompress_gbs are the two halves.

N > 1 (torchrun): weak scaling over independent axis-0 slabs -- every rank
compresses its own 512^3 slab of a (512N)x512x512 volume; the only exchange is
an all-gather of the per-slab archive sizes (NCCL) that assembles the slab
container offsets.  Timing: CUDA events on the stream the library
launches on, barrier + synchronize on both sides, max over ranks.

--impl reference: the CPU oracle (C restatement of the reference path,
oracle/; `kind: port`) on the same workload with all host threads, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", default="cr", choices=["cr", "tp"])
    ap.add_argument("--kind", default="grf", choices=["grf", "gauss", "rough"])
    ap.add_argument("--size", type=int, default=512)
    ap.add_argument("--eb", type=float, default=1e-3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-config5", action="store_true", help="skip the 2048^3 slab-sharded secondary measurement")
    ap.add_argument("--no-traffic", action="store_true", help="skip the ncu DRAM-traffic probe of the dominant kernel")
    ap.add_argument("--probe", action="store_true", help=argparse.SUPPRESS)  # one compress, for the ncu probe
    return ap.parse_args()


METRIC = "compress+decompress round-trip GB/s (input bytes / (t_compress + t_decompress)), rel-eb 1e-3"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """Clock / throttle sampler during the timed region (B200_PROFILING.md
    clocks line): NVML polled every 5 ms (nvidia-smi -lms cannot resolve a
    ~100 ms region); falls back to nvidia-smi."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.h = None
        self.stop = threading.Event()
        self.max_mhz = None

    def _poll(self):
        import pynvml
        h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
        self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        self.h = h
        while not self.stop.is_set():
            self._sample()
            self.ready.set()
            time.sleep(0.002)

    def _sample(self):
        import pynvml
        try:
            sm = pynvml.nvmlDeviceGetClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            self.samples.append((sm, rs))
        except Exception:
            pass

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.ready = threading.Event()
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            self.ready.wait(2.0)  # the poller is sampling before the timed region starts
            self.samples.clear()
        except Exception:
            self.t = None
        return self

    def __exit__(self, *a):
        if self.t and not self.samples and getattr(self, "h", None) is not None:
            self._sample()  # a region shorter than one poll: sample at its end
        self.stop.set()
        if self.t:
            self.t.join(timeout=2)

    def summary(self):
        sm = [x for x, _ in self.samples]
        reasons = set()
        for _, rs in self.samples:
            for nm, bit in self.REASONS.items():
                if rs & bit:
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(reasons), "samples": len(sm)}


# algorithmic bytes per launch for the kernels we attribute a roofline to
def algo_bytes(phase: str, n: int, prec: int, archive: int) -> float:
    if phase == "level1":  # 7/8 targets: read orig, read f64 2-lattice, write code bytes
        return n * (7 / 8 * prec + 1 / 8 * 8 + 7 / 8)
    if phase == "rlevel1":  # read codes + f64 2-lattice, write all outputs
        return n * (7 / 8 + 1 / 8 * 8 + prec)
    if phase == "eb_range":
        return n * prec
    if phase in ("huff_encode",):
        return n
    if phase in ("decode_stream",):
        return n + archive
    return 0.0


def run_reference(args):
    from oracle import oracle
    from paper_2507_11165_b200 import synth
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    oracle.set_threads(cores)
    S = args.size
    # the same input bytes as the GPU arm (generated with torch on the GPU when
    # one is present; generation is not part of the timed path)
    try:
        import torch
        if torch.cuda.is_available():
            vals = synth.make_device(args.kind, (S, S, S), seed=2025).cpu().numpy()
        else:
            raise RuntimeError
    except Exception:
        vals = synth.make(args.kind, (S, S, S), seed=2025)
    n = vals.size
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        blob = oracle.compress(vals, "rel", args.eb, args.mode, 3)
        out, _ = oracle.decompress(blob)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
    t = sum(times)
    v = n * 4 * args.steps / t / 1e9
    line = {
        "metric": METRIC, "value": round(v, 4), "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(1e3 * t / args.steps, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32->u8 codes (f64 predictor)", "data": "synthetic",
        "config": {"workload": f"{args.kind} {S}^3 f32 rel-eb {args.eb} {args.mode.upper()}",
                   "l2": "input 537 MB > 126 MB L2"},
        "impl": "reference",
        "cpu_baseline": {"value": round(v, 4), "unit": "GB/s", "cores": cores, "kind": "port",
                         "sample": f"full {S}^3 workload, oracle/hb_oracle.c (OpenMP, {cores} threads)"},
        "e2e": {"value": round(v, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "cr": round(n * 4 / len(blob), 3),
    }
    print(json.dumps(line), flush=True)


def run_probe(args):
    """Child of measure_traffic(): one warm compress, then one compress with
    the level-1 launches inside a cudaProfilerStart/Stop range (HB_NCU_RANGE)."""
    import torch

    import paper_2507_11165_b200 as hb
    from paper_2507_11165_b200 import synth
    S = args.size
    f = hb.Field(synth.make_device(args.kind, (S, S, S), seed=2025))
    spec = hb.ErrorBoundSpec("rel", args.eb)
    out = torch.empty(hb.compress_bound(f.dims, 4), dtype=torch.uint8, device="cuda")
    hb.compress_device(f, spec, args.mode, out=out)
    torch.cuda.synchronize()
    # HB_PROBE_RANGE=0: no profiler range (a launch list of the whole step;
    # cudaProfilerStop would end an ncu session that profiles from the start)
    if os.environ.get("HB_PROBE_RANGE", "1") != "0":
        os.environ["HB_NCU_RANGE"] = "level1"
    a = hb.compress_device(f, spec, args.mode, out=out)
    torch.cuda.synchronize()
    os.environ.pop("HB_NCU_RANGE", None)
    hb.decompress_device(a, f.dims, np.float32)
    torch.cuda.synchronize()


def measure_traffic(args, timeout=240):
    """DRAM bytes (read + write) of the level-1 compress kernels, measured in
    this run: ncu on a child process that compresses the same workload, with
    only the level-1 launches in the profiled range.  None if ncu is absent."""
    import shutil
    ncu = shutil.which("ncu") or "/usr/local/cuda/bin/ncu"
    if not os.path.exists(ncu):
        return None, "ncu not found"
    cmd = [ncu, "--profile-from-start", "off", "--clock-control", "none", "--csv", "--metrics",
           "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum", sys.executable,
           os.path.abspath(__file__), "--probe", "--size", str(args.size), "--kind", args.kind, "--mode", args.mode,
           "--eb", str(args.eb)]
    env = dict(os.environ, HB_NCU_RANGE="")
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, env=env)
    except Exception as e:  # noqa: BLE001
        return None, f"ncu probe failed: {e}"
    import csv
    import io
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    total, kernels, dur = 0.0, set(), 0.0
    rows = [ln for ln in r.stdout.splitlines() if ln.startswith('"')]
    for row in csv.DictReader(io.StringIO("\n".join(rows))):
        m, u, v = row.get("Metric Name"), row.get("Metric Unit"), row.get("Metric Value", "").replace(",", "")
        try:
            v = float(v)
        except ValueError:
            continue
        if m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            total += v * scale.get(u, 1)
            kernels.add(row.get("ID"))
        elif m == "gpu__time_duration.sum":
            dur += v * {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6, "us": 1e-3,
                        "ms": 1.0}.get(u, 1e-6)
    if not kernels:
        return None, "ncu probe returned no level-1 launches (rc %d): %s" % (r.returncode, r.stderr[-300:])
    return {"bytes": int(total), "launches": len(kernels), "ncu_ms": round(dur, 4)}, "measured"


def cpu_baseline(vals_host, args):
    from oracle import oracle
    cores = os.cpu_count() or 1
    oracle.set_threads(cores)
    # bounded sample: leading axis-0 planes of the same field (~10-30 s of CPU work)
    planes = min(vals_host.shape[0], 128)
    sample = np.ascontiguousarray(vals_host[:planes])
    t0 = time.perf_counter()
    reps = 0
    while True:
        blob = oracle.compress(sample, "rel", args.eb, args.mode, 3)
        oracle.decompress(blob)
        reps += 1
        if time.perf_counter() - t0 > 10.0 or reps >= 5:
            break
    dt = time.perf_counter() - t0
    # one host core: a smaller leading slab, one round trip
    oracle.set_threads(1)
    s1 = np.ascontiguousarray(vals_host[:min(vals_host.shape[0], 32)])
    t1 = time.perf_counter()
    oracle.decompress(oracle.compress(s1, "rel", args.eb, args.mode, 3))
    dt1 = time.perf_counter() - t1
    oracle.set_threads(cores)
    return {"value": round(sample.nbytes * reps / dt / 1e9, 4), "unit": "GB/s", "cores": cores, "kind": "port",
            "sample": f"{planes}x{vals_host.shape[1]}x{vals_host.shape[2]} leading slab of the same field, "
                      f"{reps} round trips, oracle/hb_oracle.c OpenMP",
            "one_core": {"value": round(s1.nbytes / dt1 / 1e9, 4), "unit": "GB/s", "cores": 1,
                         "sample": f"{s1.shape[0]}x{s1.shape[1]}x{s1.shape[2]} leading slab, 1 round trip"}}


C5_DIMS = (int(os.environ.get("HB_C5_SIZE", "2048")),) * 3  # (a smaller cube only for smoke tests)
C5_SLABS = 8


def config5(args, world, rank, local, stream):
    """BASELINE configs[4]: 2048^3 f32 turbulence-like field (32 GiB) as 8
    axis-0 slabs of 256x2048x2048, split over the N ranks (strong scaling:
    the volume is fixed, each rank owns 8/N slabs).  Every slab is generated
    on its own GPU from global coordinates (synth.make_modes); per step:
    device min/max of the local slabs + one 2-double all-reduce (global
    rel-eb), compress every local slab, all-gather of the archive sizes
    (container offsets), decompress every local slab.  No field data crosses
    GPUs.  Timed like the headline: CUDA events, barrier, max over ranks."""
    import torch
    import torch.distributed as dist

    import paper_2507_11165_b200 as hb
    from paper_2507_11165_b200 import _lib, slabs, synth
    if C5_SLABS % world:
        return {"unavailable": f"{C5_SLABS} slabs do not split over {world} ranks"}
    per = C5_SLABS // world
    bounds = slabs.slab_bounds(C5_DIMS[0], C5_SLABS)[rank * per:(rank + 1) * per]
    vals = [synth.make_modes((x1 - x0,) + C5_DIMS[1:], seed=2048, x0=x0, global_dims=C5_DIMS) for x0, x1 in bounds]
    fields = [hb.Field(v) for v in vals]
    spec = hb.ErrorBoundSpec("rel", args.eb)
    cap = hb.compress_bound(fields[0].dims, 4)
    out_buf = torch.empty(cap, dtype=torch.uint8, device="cuda")
    rec = torch.empty_like(vals[0])
    grp = dist.group.WORLD if world > 1 else None

    def global_eb():
        if world > 1:
            return slabs.global_eb_distributed(fields, spec, np.float32, grp)
        los, his = zip(*(hb.field.min_max(f) for f in fields))
        return slabs.global_abs_eb(spec, min(los), max(his), np.float32)

    launches = [0]

    def step(ev=None):
        if ev:
            ev[0].record(stream)
        eb = hb.ErrorBoundSpec("abs", global_eb())
        launches[0] += _lib.last_launch_count()
        arcs = []
        for f in fields:
            arcs.append(hb.compress_device(f, eb, args.mode, out=out_buf).clone())
            launches[0] += _lib.last_launch_count()
        if world > 1:
            head, offs, total = slabs.container_layout(C5_DIMS, 3, 4, args.mode, bounds, [a.numel() for a in arcs], grp)
        else:
            total = slabs.header_bytes(C5_SLABS) + sum(a.numel() for a in arcs)
        if ev:
            ev[1].record(stream)
        for f, a in zip(fields, arcs):
            hb.decompress_device(a, f.dims, np.float32, out=rec)
            launches[0] += _lib.last_launch_count()
        if ev:
            ev[2].record(stream)
        return arcs, eb, total

    arcs, eb, total = step()
    err = (rec.double() - vals[-1].double()).abs().max().item()
    assert err <= eb.magnitude, (err, eb.magnitude)
    steps = max(1, min(args.steps, 3))
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)]
    launches[0] = 0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for k in range(steps):
        arcs, eb, total = step(evs[k])
    torch.cuda.synchronize()
    tc = sum(e[0].elapsed_time(e[1]) for e in evs) / 1e3
    td = sum(e[1].elapsed_time(e[2]) for e in evs) / 1e3
    t = torch.tensor([tc + td, tc, td], dtype=torch.float64, device="cpu" if dist.is_initialized() and
                     dist.get_backend() != "nccl" else "cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ttot, tcm, tdm = t.tolist()
    vol = float(np.prod(C5_DIMS)) * 4
    peak, _ = peaks()
    res = {"workload": f"{C5_DIMS[0]}^3 f32 turbulence-like (synth.make_modes), 8 axis-0 slabs of "
                       f"{C5_DIMS[0] // 8}x{C5_DIMS[1]}x{C5_DIMS[2]}, rel-eb {args.eb} (global), {args.mode.upper()}",
           "scaling": "strong",
           "slabs_per_gpu": per, "steps": steps, "warmup": 1,
           "value": round(vol * steps / ttot / 1e9, 3), "unit": "GB/s",
           "compress_gbs": round(vol * steps / tcm / 1e9, 3), "decompress_gbs": round(vol * steps / tdm / 1e9, 3),
           "ms_per_step": round(1e3 * ttot / steps, 3), "cr": round(vol / total, 3), "container_bytes": total,
           "gpu_launches": launches[0],
           "hbm_roofline_frac": round(vol * steps / ttot / 1e9 / (peak * world), 5)}
    del vals, fields, rec, out_buf, arcs
    torch.cuda.empty_cache()
    return res


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2507_11165_b200 as hb
    from paper_2507_11165_b200 import _lib, slabs, synth
    from paper_2507_11165_b200.field import min_max as field_min_max

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # HB_BENCH_BACKEND=gloo (and ranks sharing a GPU) only to exercise the N > 1
    # path on a one-GPU box; the driver's runs use NCCL, one GPU per rank
    backend = os.environ.get("HB_BENCH_BACKEND", "nccl")
    local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    cdev = "cuda" if backend == "nccl" else "cpu"  # collective buffers
    S = args.size
    vals = synth.make_device(args.kind, (S, S, S), seed=2025 + rank)
    f = hb.Field(vals)
    spec = hb.ErrorBoundSpec("rel", args.eb)
    n = f.count
    nbytes = n * 4
    stream = torch.cuda.current_stream()

    out_buf = torch.empty(hb.compress_bound(f.dims, 4), dtype=torch.uint8, device="cuda")
    rec_buf = torch.empty_like(vals)

    def step():
        a = hb.compress_device(f, spec, args.mode, out=out_buf)
        hb.decompress_device(a, f.dims, np.float32, out=rec_buf)
        return a

    # the timed region's profiling mode (only the level-pass marks, the
    # dominant kernel's CUDA events for the roofline) is on for the warm-up
    # too: the compress graph is captured on the third identical call
    _lib.set_profile(2)
    for _ in range(args.warmup):
        arch = step()
    # correctness guard on the timed configuration
    err = (rec_buf.double() - vals.double()).abs().max().item()
    info = hb.section_sizes(arch.cpu().numpy().tobytes())
    assert err <= info["abs_eb"], (err, info["abs_eb"])
    archive_len = arch.numel()

    # timed region: only the level-pass marks (the dominant kernel's CUDA
    # events for the roofline); the full phase table comes from an untimed
    # profiled pass afterwards
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    phases = {}
    launches = 0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        for k in range(args.steps):
            ev[k][0].record(stream)
            if world > 1:
                # slabs of one volume share the global rel-eb: device min/max
                # (k_minmax), 2-float all-reduce, then an abs-eb compress
                lo, hi = field_min_max(f)
                mm = torch.tensor([float(hi), -float(lo)], dtype=torch.float64, device=cdev)
                dist.all_reduce(mm, op=dist.ReduceOp.MAX)
                launches += _lib.last_launch_count()
                eb = slabs.global_abs_eb(spec, np.float32(-mm[1].item()), np.float32(mm[0].item()), np.float32)
                a = hb.compress_device(f, hb.ErrorBoundSpec("abs", eb), args.mode, out=out_buf)
            else:
                a = hb.compress_device(f, spec, args.mode, out=out_buf)
            launches += _lib.last_launch_count()
            for nm, ms in _lib.last_phases():
                phases.setdefault(nm, []).append(ms)
            ev[k][1].record(stream)
            if world > 1:  # slab container: all-gather of archive sizes
                sz = torch.tensor([a.numel()], dtype=torch.int64, device=cdev)
                allsz = [torch.empty_like(sz) for _ in range(world)]
                dist.all_gather(allsz, sz)
            hb.decompress_device(a, f.dims, np.float32, out=rec_buf)
            launches += _lib.last_launch_count()
            for nm, ms in _lib.last_phases():
                phases.setdefault(nm, []).append(ms)
            ev[k][2].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    timed_phases = phases
    phases = {}
    _lib.set_profile(True)
    for _ in range(2):
        a = hb.compress_device(f, spec, args.mode, out=out_buf)
        for nm, ms in _lib.last_phases():
            phases.setdefault(nm, []).append(ms)
        hb.decompress_device(a, f.dims, np.float32, out=rec_buf)
        for nm, ms in _lib.last_phases():
            phases.setdefault(nm, []).append(ms)
    torch.cuda.synchronize()
    _lib.set_profile(False)
    tc = sum(e[0].elapsed_time(e[1]) for e in ev) / 1e3
    td = sum(e[1].elapsed_time(e[2]) for e in ev) / 1e3
    t = torch.tensor([tc + td, tc, td], dtype=torch.float64, device=cdev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ttot, tcm, tdm = t.tolist()
    total_bytes = nbytes * world * args.steps
    value = total_bytes / ttot / 1e9

    # roofline of the dominant kernel (CUDA events around it on the launch stream)
    peak, peak_kind = peaks()
    cand = {k: statistics.mean(v) for k, v in timed_phases.items() if algo_bytes(k, n, 4, archive_len) > 0}
    dom = max(cand, key=cand.get) if cand else None
    roof = None
    if dom:
        ms = cand[dom]
        ab = algo_bytes(dom, n, 4, archive_len)
        ach = ab / (ms / 1e3) / 1e9
        traffic, tsrc = None, "not measured"
        if dom == "level1" and rank == 0 and world == 1 and not args.no_traffic:
            tr, tsrc = measure_traffic(args)
            if tr:
                traffic = tr["bytes"]
                tsrc = f"ncu in this run: {tr['launches']} level-1 launches, {tr['ncu_ms']} ms serialised"
        roof = {"bound": "hbm", "kernel": dom, "achieved": round(ach, 2), "peak": peak, "unit": "GB/s",
                "frac": round(ach / peak, 4), "traffic": traffic, "algo_bytes": int(ab), "ms": round(ms, 4),
                "peak_kind": peak_kind, "traffic_source": tsrc,
                # DRAM bytes actually moved (ncu, profiles/traffic.json) over the same time: the level
                # passes trade f64 class round trips through HBM for halo recompute
                "traffic_gbs": round(traffic / (ms / 1e3) / 1e9, 1) if traffic else None}

    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(1e3 * ttot / args.steps, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32->u8 codes (f64 predictor)",
        "data": "synthetic (GPU-generated GRF-k, SURVEY 8d)",
        "config": {"workload": f"{args.kind} {S}^3 f32 per GPU, rel-eb {args.eb}, {args.mode.upper()} pipeline",
                   "parallelism": f"axis-0 slabs x{world}" if world > 1 else "single GPU",
                   "l2": "input 537 MB > 126 MB L2, no flush needed"},
        "compress_gbs": round(total_bytes / tcm / 1e9, 3), "decompress_gbs": round(total_bytes / tdm / 1e9, 3),
        "cr": round(nbytes / archive_len, 3), "archive_bytes": archive_len,
        "gpu_launches": launches,
        "roofline": roof,
        "phases_ms": {k: round(statistics.mean(v), 4) for k, v in phases.items()},
        "clocks": clk.summary(),
    }

    # end-to-end through the reference-facing API with host (pinned) buffers
    if not args.no_e2e:
        host_in = torch.empty((S, S, S), dtype=torch.float32, pin_memory=True)
        host_in.copy_(vals)
        host_out = torch.empty((S, S, S), dtype=torch.float32, pin_memory=True)
        fh = hb.Field(host_in.numpy())
        blob = None
        for _ in range(1):
            blob = hb.compress(fh, spec, args.mode)
            hb.decompress(blob, out=host_out.numpy())
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            blob = hb.compress(fh, spec, args.mode)
            hb.decompress(blob, out=host_out.numpy())
        torch.cuda.synchronize()
        te = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=cdev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = total_bytes / te.item() / 1e9
        line["e2e"] = {"value": round(e2e, 3), "unit": "GB/s", "h2d_bytes_per_step": nbytes + len(blob),
                       "d2h_bytes_per_step": len(blob) + nbytes}
    if not args.no_config5:
        _lib.release_contexts()  # the 512^3 arena is not needed for the slabs
        torch.cuda.empty_cache()
        line["config5"] = config5(args, world, rank, local, stream)

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(vals.cpu().numpy(), args)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.probe:
        run_probe(args)
        return
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
