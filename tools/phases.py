"""Per-inner-iteration cost of each phase of the persistent solver (k_inner), from its globaltimer phase marks.

Runs one warm solve, then `--reps` timed solves, and divides the phase totals (block 0, `ml_inner_phases`) by the
inner iterations of the small-|A| (< 2048) and large-|A| relaxations (the relaxation trace).  Phase 7 (outer line
search + update) is reported per relaxation.  ML_LIB=<path> selects an alternative build of libml.so.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import mlgen  # noqa: E402
import paper_1607_00315_b200 as ml  # noqa: E402

NAMES = ["D", "S", "B1+tot", "R", "B2+tot+dec", "sv", "G", "tail/relax"]
# IR_PHDBG builds: sub-phases of the small-|A| iteration in slots 8..15 (NAMES then label the remainders)
SUB = ["D:top+prefetch", "D:direction", "S:zero", "S:scatter", "S:chunk-compute", "S:chunk-sync", "S:producer", "S:tma-wait"]
DBG = ["D:partials", "S:write-partials", "B1+tot", "R", "B2+tot+dec", "sv", "G", "tail/relax"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--tag", default=os.environ.get("ML_LIB", "libml.so"))
    ap.add_argument("--sub", action="store_true", help="the library was built with -DIR_PHDBG")
    ap.add_argument("--gather", action="store_true", help="the library was built with -DGS_PHDBG")
    ap.add_argument("--engine", type=int, default=0, help="ml_set_engine flags (16: heavy path always, 32: never)")
    ap.add_argument("--raw", action="store_true", help="also print the raw phase slots (ns, all solves)")
    a = ap.parse_args()
    ds = mlgen.make(a.config)
    ctx = ml.Context(ds)
    ctx.ml_set_engine(a.engine)
    ctx.ml_solve()
    ctx.ml_inner_phases(reset=True)
    st = ctx.stream
    ts = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        rep = ctx.ml_solve()
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ph = ctx.ml_inner_phases(reset=True)
    if a.raw:
        print(json.dumps({"raw_ns": ph, "heavy": ctx.ml_heavy_info()}))
    prof = ctx.ml_profile_read()   # nonzeros streamed per pass class (device counters, all solves since create)
    tr = ctx.trace()
    its = [0, 0]
    rel = [0, 0]
    for r in tr:
        if r["inner_iters"] <= 0:
            continue
        k = 0 if r["nA"] < 2048 else 1
        its[k] += r["inner_iters"]
        rel[k] += 1
    out = {"config": a.config, "tag": a.tag, "ms": sorted(ts)[len(ts) // 2], "cycles": rep["cycles"], "nnz_touched": rep["nnz_touched"],
           "nnz_per_solve": {k: prof[k]["nnz"] // (a.reps + 1) for k in ("scatter_XAs", "gather_Hs", "gather_fine",
                                                                    "gather_coarse", "margins") if prof[k]["nnz"]}}
    if a.gather:   # k_gather_small phases (slots 8..13), per launch (relaxations incl. converged-level skips)
        nl = sum(1 for r in tr if r["level"] > 0) or 1   # coarse-level launches only
        names = ["setup+rD", "stream", "flags+partials", "grid.sync", "totals+offsets", "compaction", "stream:tma-wait"]
        out["gather_us_per_launch"] = {names[j]: round(ph[8 + j] / 1e3 / a.reps / nl, 2) for j in range(7)}
        print(json.dumps(out))
        return
    if a.sub:
        out["rows"] = [[r["level"], r["nA"], r["inner_iters"], int(r["alpha"]), round(r["F_before"] / 1e3, 1)]
                       for r in tr]   # debug build: F_before = us in k_inner (block 0), alpha = iterations run
        us = [x / 1e3 / a.reps for x in ph]
        n = max(its[0], 1)
        out["small_sub_us_per_iter"] = {**{DBG[j]: round(us[j] / n, 2) for j in range(7)},
                                        **{SUB[j]: round(us[8 + j] / n, 2) for j in range(8)}}
        out["small_tail_us_per_relax"] = round(us[7] / max(rel[0], 1), 2)
        print(json.dumps(out))
        return
    for k, nm in ((0, "small"), (1, "large")):
        if its[k] == 0:
            continue
        us = [ph[8 * k + j] / 1e3 / a.reps for j in range(8)]
        out[nm] = {"relax": rel[k], "iters": its[k],
                   "us_per_iter": {NAMES[j]: round(us[j] / its[k], 2) for j in range(7)},
                   "us_tail_per_relax": round(us[7] / rel[k], 2),
                   "ms_total": round(sum(us) / 1e3, 3)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
