"""Summarise ncu --set full reports: key metrics + top source lines by warp-stall samples."""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return r[0], r[1], r[2]


for rep in sys.argv[1:]:
    h, units, v = raw(rep)
    name = v[h.index("Kernel Name")][:70]
    print(f"== {rep.split('/')[-1]}: {name}")
    for k in KEYS:
        if k in h:
            print(f"   {k:62s} {v[h.index(k)]:>14s} {units[h.index(k)]}")
    stalls = [(float(v[i] or 0), k) for i, k in enumerate(h)
              if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")]
    print("   stalls per issued instruction: " + ", ".join(
        f"{k[34:-23]}={x:.2f}" for x, k in sorted(stalls, reverse=True)[:7]))
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    open("/tmp/_src.csv", "w").write(src)
    top = subprocess.run([sys.executable, __file__.replace("ncu_summary.py", "ncu_lines.py"), "/tmp/_src.csv", "12"],
                         capture_output=True, text=True).stdout
    print("   top source lines (share of warp-stall samples):")
    for line in top.splitlines():
        print("     " + line)
    print()
