"""Record the dram bytes per launch of a profiled kernel (profiles/<tag>/<config>.json, written by
tools/ncu_summary.py from one `ncu --set full` capture) in profiles/traffic.json, which bench.py
reads for the roofline's `traffic` field.

    python tools/traffic_update.py <tag> <config> <plan kernel name>
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bytes(v):
    num, unit = v.split()[:2]
    return float(num.replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit]


def main():
    tag, cfg, kernel = sys.argv[1:4]
    summ = json.load(open(os.path.join(ROOT, "profiles", tag, f"{cfg}.json")))
    cap = summ["full_capture"][0]
    tot = _bytes(cap["dram__bytes_read.sum"]) + _bytes(cap["dram__bytes_write.sum"])
    p = os.path.join(ROOT, "profiles", "traffic.json")
    d = json.load(open(p)) if os.path.exists(p) else {}
    d[cfg] = {"kernel": kernel, "dram_bytes_per_launch": tot,
              "source": f"profiles/{tag}/{cfg}.json (ncu --set full, one launch: {cap['kernel'][:60]})"}
    json.dump(d, open(p, "w"), indent=1)
    print(cfg, kernel, tot)


if __name__ == "__main__":
    main()
