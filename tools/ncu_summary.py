"""Summarise ncu outputs into profiles/<tag>/ (tracked):
  - launch list CSV (gpu__time_duration per launch) -> per-kernel counts, mean/median/min/max time,
    share of the listed time (the list covers the whole bench command: generator, weight pack,
    warm-up, timed steps and the e2e calls, which run the same kernel on host-pipelined chunks)
  - one --set full capture -> key raw metrics + top stall sites
Usage: python tools/ncu_summary.py <tag> <config> [gpurun_out prefix]
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "sm__cycles_elapsed.avg.per_second", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "launch__shared_mem_per_block_dynamic"]


def _csv_rows(path):
    lines = [l for l in open(path) if l.startswith('"')]
    return list(csv.reader(io.StringIO("".join(lines))))


def launches(path):
    rows = _csv_rows(path)
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    d = defaultdict(list)
    for r in rows[1:]:
        v = float(r[vi].replace(",", ""))
        if r[ui] == "us":
            v *= 1e3
        elif r[ui] == "ms":
            v *= 1e6
        name = r[ki].split("(")[0].replace("void ", "").replace("tcbf::<unnamed>::", "")
        d[name].append(v)
    def stats(v):
        v = sorted(v)
        return {"launches": len(v), "mean_us": round(sum(v) / len(v) / 1e3, 3),
                "median_us": round(v[len(v) // 2] / 1e3, 3), "min_us": round(v[0] / 1e3, 3),
                "max_us": round(v[-1] / 1e3, 3)}
    return {k: stats(v) for k, v in d.items()}


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        m = {"kernel": vals[hdr.index("Kernel Name")][:120]}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                m[k] = f"{vals[i]} {units[i]}".strip()
        res.append(m)
    src = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    srows = list(csv.reader(io.StringIO(src)))
    stalls = []
    if len(srows) > 2:
        h = srows[1]
        try:
            si, wi = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
            data = [(int(r[wi] or 0), r[si].strip()) for r in srows[2:] if len(r) > wi and r[wi].isdigit()]
            tot = sum(d[0] for d in data) or 1
            stalls = [f"{100 * n / tot:5.1f}%  {s}" for n, s in sorted(data, reverse=True)[:15]]
        except ValueError:
            pass
    return res, stalls


def main():
    tag, cfg = sys.argv[1], sys.argv[2]
    prefix = sys.argv[3] if len(sys.argv) > 3 else os.path.join(ROOT, "gpurun_out", f"prof_{tag}_{cfg}")
    outdir = os.path.join(ROOT, "profiles", tag)
    os.makedirs(outdir, exist_ok=True)
    summary = {"config": cfg}
    if os.path.exists(prefix + "_launches.csv"):
        L = launches(prefix + "_launches.csv")
        tot = sum(v["mean_us"] * v["launches"] for v in L.values())
        for v in L.values():
            v["share_of_listed_time"] = round(v["mean_us"] * v["launches"] / tot, 3)
        summary["launches"] = L
    if os.path.exists(prefix + "_full.ncu-rep"):
        m, stalls = full(prefix + "_full.ncu-rep")
        summary["full_capture"] = m
        summary["top_stall_sites"] = stalls
    with open(os.path.join(outdir, f"{cfg}.json"), "w") as f:
        json.dump(summary, f, indent=1)
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main()
