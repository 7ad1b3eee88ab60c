"""Summarise ncu reports / launch lists into the text files kept in profiles/.

usage: python profiles/ncu_summary.py launches <launches.csv> <out.txt>
       python profiles/ncu_summary.py report <file.ncu-rep> <out.txt>
"""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "lts__t_sector_hit_rate.pct"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def launches(path, out):
    rows = list(csv.reader(open(path)))
    h = None
    recs = []
    for r in rows:
        if r and r[0] == "ID":
            h = r
            continue
        if h and len(r) == len(h):
            d = dict(zip(h, r))
            if d["Metric Name"] == "gpu__time_duration.sum":
                v = float(d["Metric Value"].replace(",", ""))
                u = d["Metric Unit"]
                us = v / 1e3 if u in ("ns", "nsecond") else (v * 1e3 if u in ("ms", "msecond") else v)
                recs.append((d["Kernel Name"].split("(")[0], us))
    # bench --steps 1 --warmup 1: the last compress (from its k_minmax_init)
    # plus the decompress that follows; torch kernels (bench checks) dropped
    starts = [i for i, (k, _) in enumerate(recs) if "k_minmax_init" in k]
    step = [(k, t) for k, t in recs[starts[-1]:] if "at::" not in k]
    with open(out, "w") as fh:
        fh.write("# one compress + decompress step, 512^3 GRF-k f32 rel 1e-3 CR (ncu --metrics gpu__time_duration.sum,"
                 " cold-cache and serialised: compare shares, not absolutes)\n")
        tot = sum(t for _, t in step)
        for k, t in step:
            fh.write(f"{t:10.1f} us  {100 * t / tot:5.1f}%  {k}\n")
        fh.write(f"total {tot:.1f} us over {len(step)} launches\n")


def report(path, out):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, units = rows[0], rows[1]
    with open(out, "w") as fh:
        for r in rows[2:]:
            d, u = dict(zip(h, r)), dict(zip(h, units))
            fh.write("----\n  Kernel Name: " + d["Kernel Name"][:140] + "\n")
            for k in KEYS:
                if k in d:
                    v, un = d[k], u.get(k, "")
                    if un in SCALE:
                        v, un = f"{float(v.replace(',', '')) * SCALE[un] / 1e6:.3f}", "MB"
                    fh.write(f"  {k}: {v} {un}\n")
            st = [(k.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(d[k].replace(",", "")))
                  for k in h if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
                  and d[k].replace(",", "").replace(".", "", 1).isdigit()]
            tot = sum(v for _, v in st) or 1
            st.sort(key=lambda x: -x[1])
            fh.write("  stall samples: " + ", ".join(f"{k}={100 * v / tot:.0f}%" for k, v in st[:6]) + "\n")


if __name__ == "__main__":
    {"launches": launches, "report": report}[sys.argv[1]](sys.argv[2], sys.argv[3])
