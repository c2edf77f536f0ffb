"""Where the end-to-end time of one step goes (bench.py's e2e leg): pinned H2D of X and y, ml_create (validation,
unit schedules, the heavy-column copy for large X), ml_solve, D2H of w.  CUDA events on the library's stream.

Usage: python tools/e2e_breakdown.py --config 5
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import mlgen  # noqa: E402
import paper_1607_00315_b200 as ml  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    ds = mlgen.make(a.config)
    keep = [np.ascontiguousarray(x) for x in (ds.csr_rowptr, ds.csr_col, ds.csr_val, ds.csc_colptr, ds.csc_row,
                                              ds.csc_val, ds.y)]
    skip = {0, 1, 2} if ds.m <= 8192 else set()
    pinned = [None if k in skip else torch.from_numpy(x).pin_memory() for k, x in enumerate(keep)]
    h2d = sum(t.numel() * t.element_size() for t in pinned if t is not None)
    dev = torch.device("cuda:0")
    out = []
    w_host = torch.empty(ds.n, dtype=torch.float64).pin_memory()
    for rep in range(a.reps + 1):
        st = torch.cuda.current_stream(dev)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ev[0].record(st)
        dev_t = [None if t is None else t.to(dev, non_blocking=True) for t in pinned]   # (H2D alone, for its time)
        ev[1].record(st)
        ctx = ml.Context(ds, device="cuda:0", host_tensors=pinned)   # H2D again + ml_create
        del dev_t
        ev[2].record(st)
        ctx.ml_solve()
        ev[3].record(st)
        w_host.copy_(ctx.ml_get_w(), non_blocking=True)   # D2H into pinned memory (as bench.py's e2e leg)
        ev[4].record(st)
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) * 1e3
        ctx.close()
        if rep:
            out.append({"h2d_ms": ev[0].elapsed_time(ev[1]), "h2d_plus_create_ms": ev[1].elapsed_time(ev[2]),
                        "solve_ms": ev[2].elapsed_time(ev[3]), "d2h_w_ms": ev[3].elapsed_time(ev[4]), "wall_ms": wall})
    med = {k: float(np.median([o[k] for o in out])) for k in out[0]}
    med["create_ms (h2d_plus_create - h2d)"] = med["h2d_plus_create_ms"] - med["h2d_ms"]
    print(json.dumps({"config": a.config, "h2d_bytes": h2d, "h2d_GBs": round(h2d / med["h2d_ms"] / 1e6, 1), **med}))


if __name__ == "__main__":
    main()
