"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per step."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
    hdr = rows[hi]
    return hdr, rows[hi + 1:]


def main(path, detail=False, marker="pack_kernel"):
    hdr, data = load(path)
    ki, vi = hdr.index('Kernel Name'), hdr.index('Metric Value')
    gi = hdr.index('Grid Size')
    idx = [i for i, r in enumerate(data) if marker in r[ki]]
    s, e = (idx[-2], idx[-1]) if len(idx) >= 2 else (0, len(data))
    agg = collections.defaultdict(lambda: [0, 0.0])
    tot = 0.0
    for r in data[s:e]:
        v = float(r[vi].replace(',', ''))
        n = r[ki].split('(')[0][:60]
        agg[n][0] += 1
        agg[n][1] += v
        tot += v
        if detail and v > 50000:
            print(f"   {v / 1e3:8.1f} us {r[ki][:50]} grid {r[gi]}")
    for n, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{v / 1e3:9.1f} us {100 * v / tot:5.1f}% x{c:3d} {n}")
    print(f"total {tot / 1e3:.1f} us, {e - s} launches")


if __name__ == "__main__":
    main(sys.argv[1], "-d" in sys.argv)
