"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list by kernel (used for profiles/*.md)."""
import collections
import csv
import re
import sys


def summarize(path, top=30):
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    r = csv.reader(lines)
    hdr = next(r)
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    gi, bi = hdr.index("Grid Size"), hdr.index("Block Size")
    agg = collections.defaultdict(lambda: [0, 0.0, set()])
    for row in r:
        v = float(row[vi].replace(",", ""))
        u = row[ui]
        v = v / 1000.0 if u in ("ns", "nsecond") else (v * 1000 if u in ("ms", "msecond") else v)
        name = re.sub(r"\(.*", "", row[ki]).replace("void ", "").replace("<unnamed>::", "")
        a = agg[name]
        a[0] += 1
        a[1] += v
        a[2].add(row[gi] + "x" + row[bi])
    tot = sum(a[1] for a in agg.values())
    out = [f"total {tot:.1f} us over {sum(a[0] for a in agg.values())} launches", "",
           "| share | total us | launches | avg us | kernel | grid x block |", "|---|---|---|---|---|---|"]
    for k, a in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        out.append(f"| {a[1] / tot * 100:.2f}% | {a[1]:.1f} | {a[0]} | {a[1] / a[0]:.2f} | `{k}` | {' '.join(sorted(a[2]))[:60]} |")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarize(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30))
