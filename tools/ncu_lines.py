"""Top source lines by warp-stall samples from `ncu --page source --csv --print-source cuda,sass`."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
fname, hdr = None, None
agg = []
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or not r or not r[0] or not r[0].isdigit():
        continue
    si = hdr.index("Warp Stall Sampling (All Samples)")
    try:
        samples = int(r[si])
    except ValueError:
        continue
    stalls = {h: r[i] for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h}
    top_stalls = sorted(((int(v), k) for k, v in stalls.items() if v.isdigit()), reverse=True)[:3]
    agg.append((samples, fname, r[0], r[1].strip()[:70], top_stalls))
tot = sum(a[0] for a in agg)
for s, f, ln, src, st in sorted(agg, reverse=True)[:top]:
    print(f"{100 * s / tot:5.1f}% {f}:{ln:5s} {src:70s} {' '.join(f'{k[6:]}={v}' for v, k in st)}")
