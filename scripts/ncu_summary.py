"""Summarise ncu outputs into profiles/*.json (run here, on the CPU box).

  python scripts/ncu_summary.py launches <launches.csv> <out.json> "<command>"
  python scripts/ncu_summary.py full <report.ncu-rep> <out.json> "<command>" <n_rows> <alg_bytes>
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

import numpy as np


def launches(path, out, cmd):
    txt = open(path).read()
    start = txt.index('"ID"')
    rows = list(csv.DictReader(io.StringIO(txt[start:])))
    per = defaultdict(list)
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        if r["Metric Unit"] in ("nsecond", "ns"):
            v /= 1e3
        elif r["Metric Unit"] == "msecond":
            v *= 1e3
        name = r["Kernel Name"].split("(")[0]
        per[name].append(v)
    tot = sum(sum(v) for v in per.values())
    res = {"command": cmd, "note": "ncu launch list: cold-cache, serialised launches; compare shares",
           "total_us": tot, "kernels": {}}
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        res["kernels"][k] = {"launches": len(v), "median_us": float(np.median(v)),
                             "min_us": float(np.min(v)), "max_us": float(np.max(v)),
                             "share": sum(v) / tot}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


def full(rep, out, cmd, n_rows, alg):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u, v = rows[0], rows[1], rows[2]
    get = {h[i]: (v[i], u[i]) for i in range(len(h))}

    def num(key):
        val, unit = get[key]
        x = float(val.replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3,
                 "usecond": 1, "msecond": 1e3}.get(unit, 1)
        return x * scale

    res = {
        "kernel": get["Kernel Name"][0] if "Kernel Name" in get else None,
        "command": cmd,
        "n_rows": int(n_rows),
        "duration_us": num("gpu__time_duration.sum"),
        "dram_read_bytes": num("dram__bytes_read.sum"),
        "dram_write_bytes": num("dram__bytes_write.sum"),
        "algorithmic_bytes_per_launch": float(alg),
        "registers_per_thread": num("launch__registers_per_thread"),
        "grid": num("launch__grid_size"),
        "block": num("launch__block_size"),
        "issue_active_pct": num("sm__inst_issued.avg.pct_of_peak_sustained_active"),
        "fp64_pipe_pct": num("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
        "dram_throughput_pct": num("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
        "warps_active": num("sm__warps_active.avg.per_cycle_active"),
    }
    res["dram_bytes_per_launch"] = res["dram_read_bytes"] + res["dram_write_bytes"]
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(*sys.argv[2:5])
    else:
        full(*sys.argv[2:7])
