"""Summarise an ncu launch list (--metrics gpu__time_duration.sum[,dram__bytes_read.sum,dram__bytes_write.sum] --csv)
by kernel: launches, device time and share, DRAM bytes per launch (used for profiles/*.md and traffic_*.json)."""
import collections
import csv
import json
import re
import sys


def load(path):
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    r = csv.reader(lines)
    hdr = next(r)
    ki, ni, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    gi, bi, ii = hdr.index("Grid Size"), hdr.index("Block Size"), hdr.index("ID")
    launches = collections.OrderedDict()
    for row in r:
        lid = row[ii]
        name = re.sub(r"\(.*", "", row[ki]).replace("void ", "").replace("<unnamed>::", "").strip()
        d = launches.setdefault(lid, {"kernel": name, "cfg": row[gi] + "x" + row[bi], "us": 0.0, "dram": 0.0})
        v = float(row[vi].replace(",", ""))
        u = row[ui]
        if row[ni] == "gpu__time_duration.sum":
            d["us"] = v / 1000.0 if u in ("ns", "nsecond") else (v * 1000 if u in ("ms", "msecond") else v)
        elif row[ni].startswith("dram__bytes"):
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
            d["dram"] += v * scale
    return list(launches.values())


def summarize(path, top=30):
    ls = load(path)
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0, set()])
    for d in ls:
        a = agg[d["kernel"]]
        a[0] += 1
        a[1] += d["us"]
        a[2] += d["dram"]
        a[3].add(d["cfg"])
    tot = sum(a[1] for a in agg.values())
    out = [f"total {tot:.1f} us over {len(ls)} launches (serialised, cold-cache replay: shares, not absolutes)", "",
           "| share | total us | launches | avg us | DRAM MB / launch | kernel | grid x block |",
           "|---|---|---|---|---|---|---|"]
    for k, a in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        out.append(f"| {a[1] / tot * 100:.2f}% | {a[1]:.1f} | {a[0]} | {a[1] / a[0]:.2f} | {a[2] / a[0] / 1e6:.3f} | `{k}` | "
                   f"{' '.join(sorted(a[3]))[:60]} |")
    return "\n".join(out), agg


if __name__ == "__main__":
    text, agg = summarize(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
    print(text)
    if len(sys.argv) > 3:   # kernel-name prefix -> average DRAM bytes per launch (the bench's roofline "traffic")
        pref, cls, out = sys.argv[3], sys.argv[4], sys.argv[5]
        n = sum(a[0] for k, a in agg.items() if k.startswith(pref))
        b = sum(a[2] for k, a in agg.items() if k.startswith(pref))
        json.dump({cls: b / max(n, 1), "launches": n, "source": sys.argv[1]}, open(out, "w"), indent=1)
