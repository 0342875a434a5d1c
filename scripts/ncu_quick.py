"""Quick look at an ncu report of k_rs_cycle: duration, DRAM bytes, issue,
instructions, and the SASS opcode mix of instructions executed >= 30000 times
(the scan's per-tile loop). python scripts/ncu_quick.py <rep> [--dump file]"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, u, v = r[0], r[1], r[2]
g = {h[i]: (v[i], u[i]) for i in range(len(h))}
for k in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
          "sm__inst_issued.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
          "launch__registers_per_thread"]:
    print(k, g.get(k))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hh = rows[1]
iS, iE, iW = hh.index("Source"), hh.index("Instructions Executed"), hh.index("Warp Stall Sampling (All Samples)")
thr = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 30000
ops, opw, n, tot, stall = Counter(), Counter(), 0, 0, Counter()
lines = []
for x in rows[2:]:
    e = int(x[iE] or 0)
    w = int(x[iW] or 0)
    if e < thr:
        continue
    t = x[iS].split()
    o = t[1] if t[0].startswith("@") else t[0]
    o = o.split(".")[0]
    ops[o] += e
    opw[o] += w
    tot += e
    n = max(n, e)
    lines.append(f"{e:8d} {w:5d} {x[iS]}")
print("loop instructions per warp-tile:", tot / n, "samples", sum(opw.values()))
print(" ".join(f"{k}:{v / n:.0f}" for k, v in ops.most_common(25)))
if "--dump" in sys.argv:
    open(sys.argv[sys.argv.index("--dump") + 1], "w").write("\n".join(lines))
