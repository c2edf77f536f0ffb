"""A/B of the column engines (ml_set_engine): device time per pass class over warm solves, both engines.

Usage: python tools/engine_ab.py --config 5 [--reps 3]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import mlgen  # noqa: E402
import paper_1607_00315_b200 as ml  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--engines", default="0,1")
    a = ap.parse_args()
    ds = mlgen.make(a.config)
    ctx = ml.Context(ds)
    out = {"config": a.config}
    for eng in [int(x) for x in a.engines.split(",")]:
        ctx.ml_set_engine(eng)
        ctx.ml_solve()
        ctx.ml_profile((1 << 14) - 1)
        ts, F = [], None
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(ctx.stream)
            r = ctx.ml_solve()
            e1.record(ctx.stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
            F = r["F"]
        pr = ctx.ml_profile_read()
        ctx.ml_profile(0)
        out[f"engine{eng}"] = {"ms": sorted(ts)[len(ts) // 2], "F": F, "cycles": r["cycles"],
                               "us_per_pass": {k: round(1e3 * v["ms"] / max(v["passes"], 1), 1)
                                               for k, v in pr.items() if v["passes"]},
                               "ms_per_solve": {k: round(v["ms"] / a.reps, 3) for k, v in pr.items() if v["ms"] > 0}}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
