"""Relaxation trace of one warm solve: level, |C|, |A|, inner iterations, outcome, F change, alpha per relaxation.

Usage: python tools/trace_dump.py --config 5
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
    a = ap.parse_args()
    ds = mlgen.make(a.config)
    ctx = ml.Context(ds)
    ctx.ml_solve()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(ctx.stream)
    rep = ctx.ml_solve()
    e1.record(ctx.stream)
    torch.cuda.synchronize()
    tr = ctx.trace()
    print(json.dumps({"config": a.config, "ms": e0.elapsed_time(e1), "cycles": rep["cycles"],
                      "relaxations": rep["relaxations"]}))
    for r in tr:
        print(f"L{r['level']:2d} nC={r['nC']:9d} nA={r['nA']:8d} it={r['inner_iters']:2d} out={r['outcome']} "
              f"F={r['F_after']:.10e} a={r['alpha']:.4g}")


if __name__ == "__main__":
    main()
