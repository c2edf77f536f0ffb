"""Solve wall time (events) vs the sum of per-class device times: the launch gaps of the host-driven cycle."""
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
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    ds = mlgen.make(a.config)
    ctx = ml.Context(ds)
    for _ in range(2):
        ctx.ml_solve()
    ctx.ml_profile(0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(ctx.stream)
    for _ in range(a.reps):
        rep = ctx.ml_solve()
    e1.record(ctx.stream)
    torch.cuda.synchronize()
    wall = e0.elapsed_time(e1) / a.reps
    l0 = ctx.ml_kernel_launches()
    ctx.ml_profile((1 << 14) - 1)
    ctx.ml_solve()
    launches = ctx.ml_kernel_launches() - l0
    prof = ctx.ml_profile_read()
    dev = {k: round(v["ms"], 3) for k, v in prof.items() if v["ms"] > 0}
    print(json.dumps({"config": a.config, "wall_ms": round(wall, 3), "device_ms": round(sum(dev.values()), 3),
                      "launches": launches, "cycles": rep["cycles"], "relaxations": rep["relaxations"], "classes": dev}))


if __name__ == "__main__":
    main()
