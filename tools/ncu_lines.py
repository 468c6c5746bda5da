"""Per-CUDA-source-line instruction and warp-stall shares from an ncu report's source page.
Usage: python tools/ncu_lines.py report.ncu-rep [n] [kernel-substring]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
if len(sys.argv) > 3:
    cmd += ["-k", sys.argv[3]]
rows = list(csv.reader(io.StringIO(subprocess.run(cmd, capture_output=True, text=True).stdout)))
cur_file, hdr, cur = None, None, None
inst, stall, src = collections.Counter(), collections.Counter(), {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name",):
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None:
        continue
    if r[0] != "":
        cur = (cur_file, r[0])
        src[cur] = r[1].strip()[:80]
    if r[2] == "" or cur is None:
        continue
    try:
        inst[cur] += float(r[7]) if r[7] not in ("", "-") else 0.0
        stall[cur] += float(r[4]) if r[4] not in ("", "-") else 0.0
    except (ValueError, IndexError):      # a source row whose text held the delimiter
        continue
ti, ts = sum(inst.values()) or 1, sum(stall.values()) or 1
print(f"# {ti:.4g} warp instructions, {ts:.0f} stall samples")
print("# top by instructions")
for k, v in inst.most_common(n):
    print(f"{100 * v / ti:5.1f}% inst {100 * stall[k] / ts:5.1f}% stall  {k[0]}:{k[1]}  {src.get(k, '')}")
print("# top by stall samples")
for k, v in stall.most_common(n):
    print(f"{100 * inst[k] / ti:5.1f}% inst {100 * v / ts:5.1f}% stall  {k[0]}:{k[1]}  {src.get(k, '')}")
