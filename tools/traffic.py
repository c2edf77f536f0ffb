"""Per-pass-class DRAM traffic from an ncu launch list (--metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --csv) of one solve, in launch order: the classes of bench.py's rooflines.

  margins        k_heavy<OpMargin> + k_margins<G>            (one margins pass)
  gather_fine    k_heavy<OpGH> [+ k_gather_out<4, 3>] + k_gather_free<G, 1>   (finest gather, A2/A3 over all columns)
  gather_coarse  k_heavy<OpGH> + k_gather_free<G, 0>         (coarse gather over a level list)
  inner_fused    k_inner<...>                                (one relaxation of the persistent inner solver)

Usage: python tools/traffic.py launches.csv out.json
"""
import json
import sys

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.abspath(__file__)))
from launches import load  # noqa: E402


def classify(ls):
    acc = {}
    pending = []   # k_heavy launches waiting for the pass they belong to

    def add(cls, launches):
        a = acc.setdefault(cls, {"passes": 0, "dram": 0.0, "us": 0.0})
        a["passes"] += 1
        a["dram"] += sum(d["dram"] for d in launches)
        a["us"] += sum(d["us"] for d in launches)

    for d in ls:
        k = d["kernel"]
        if k.startswith("k_heavy<OpMargin") or k.startswith("k_heavy<OpGH") or k.startswith("k_gather_out"):
            pending.append(d)   # (k_gather_out<4, 3>: the column sums of the two-pass finest gather)
        elif k.startswith("k_margins"):
            add("margins", pending + [d]); pending = []
        elif k.startswith("k_gather_free") and k.replace(" ", "").split(",")[1].startswith("1"):
            add("gather_fine", pending + [d]); pending = []
        elif k.startswith("k_gather_free"):
            add("gather_coarse", pending + [d]); pending = []
        elif k.startswith("k_inner"):
            add("inner_fused", [d])
        elif k.startswith("k_select"):
            add("select", [d])
    return {c: {"dram_bytes_per_pass": a["dram"] / a["passes"], "passes": a["passes"],
                "us_per_pass_ncu": a["us"] / a["passes"]} for c, a in acc.items()}


if __name__ == "__main__":
    out = classify(load(sys.argv[1]))
    flat = {c: v["dram_bytes_per_pass"] for c, v in out.items()}
    flat["detail"] = out
    flat["source"] = sys.argv[1]
    json.dump(flat, open(sys.argv[2], "w"), indent=1)
    print(json.dumps(out, indent=1))
