"""Summarise an `ncu --csv --metrics ...` launch list: per kernel name launches, total µs, share,
DRAM GB/s, tensor %, issue %.  Usage: python tools/launch_table.py launches.csv"""
import csv
import io
import sys
from collections import defaultdict

txt = open(sys.argv[1]).read()
rows = list(csv.reader(io.StringIO("\n".join(l for l in txt.splitlines() if l.startswith('"')))))
h = rows[0]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = defaultdict(dict)
for r in rows[1:]:
    per[int(r[ii])][r[mi]] = float(r[vi].replace(",", "")) if r[vi] else 0.0
    per[int(r[ii])]["name"] = r[ki].split("(")[0].replace("void longer::<unnamed>::", "").replace("void ", "")
agg = defaultdict(lambda: [0, 0.0, 0.0, 0.0, 0.0])
tot = 0.0
for k, m in per.items():
    t = m.get("gpu__time_duration.sum", 0.0)
    a = agg[m["name"]]
    a[0] += 1; a[1] += t; a[2] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
    a[3] += t * m.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", 0)
    a[4] += t * m.get("smsp__issue_active.avg.pct_of_peak_sustained_active", 0)
    tot += t
unit = 1e-3  # gpu__time_duration.sum is in ns
print(f"# {len(per)} launches, sum of kernel durations {tot * unit:.1f} us (serialised, cold: compare shares)")
print(f"{'kernel':44s} {'n':>3s} {'us':>9s} {'share':>6s} {'GB/s':>7s} {'tensor%':>8s} {'issue%':>7s}")
for name, (n, t, by, tw, iw) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{name[:44]:44s} {n:3d} {t * unit:9.1f} {100 * t / tot:5.1f}% {by / t if t else 0:7.0f} {tw / t if t else 0:8.2f} {iw / t if t else 0:7.1f}")
