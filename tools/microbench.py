"""Micro-benchmarks of single libml passes on a BASELINE config (CUDA events, warm L2 unless --flush)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import mlgen  # noqa: E402
import paper_1607_00315_b200 as ml  # noqa: E402


def timeit(fn, reps, stream, flush=None):
    ts = []
    for _ in range(3):
        fn()
    for _ in range(reps):
        if flush is not None:
            flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--ncols", type=int, default=3000)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--flush", action="store_true")
    a = ap.parse_args()
    ds = mlgen.make(a.config)
    ctx = ml.Context(ds)
    st = ctx.stream
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda") if a.flush else None
    rng = np.random.default_rng(0)
    C = np.sort(rng.choice(ds.n, min(a.ncols, ds.n), replace=False)).astype(np.int32)
    lens = np.diff(ds.csc_colptr)
    nnzC = int(lens[C].sum())
    Ct = torch.from_numpy(C).cuda()
    v = torch.randn(len(C), dtype=torch.float64, device="cuda")
    ctx.ml_eval_f_grad(want_g=False, want_h=False)
    out = {}
    t = timeit(lambda: ctx.ml_hessvec(Ct, v), a.reps, st, flush)
    out["hessvec_C"] = {"ms": t, "nnz": nnzC, "GBs_X2passes": 2 * 8 * nnzC / t / 1e6}
    t = timeit(lambda: ctx.ml_diag_hess(Ct), a.reps, st, flush)
    out["diag_C"] = {"ms": t, "GBs": 8 * nnzC / t / 1e6}
    t = timeit(lambda: ctx.ml_diag_hess(None), a.reps, st, flush)
    out["diag_all"] = {"ms": t, "GBs": 8 * ds.nnz / t / 1e6}
    t = timeit(lambda: ctx.ml_eval_f_grad(want_g=False, want_h=False), a.reps, st, flush)
    out["margins_all"] = {"ms": t, "GBs": 8 * ds.nnz / t / 1e6}
    vall = torch.randn(ds.n, dtype=torch.float64, device="cuda")
    t = timeit(lambda: ctx.ml_hessvec(None, vall), a.reps, st, flush)
    out["hessvec_all"] = {"ms": t, "GBs_X2passes": 2 * 8 * ds.nnz / t / 1e6}
    ctx.ml_inner_phases(reset=True)
    t = timeit(lambda: ctx.ml_solve(), 3, st)
    ph = ctx.ml_inner_phases(reset=True)
    out["solve"] = {"ms": t, "inner_phase_ms_small_A": [round(x / 6e6, 3) for x in ph[:8]], "inner_phase_ms_large_A": [round(x / 6e6, 3) for x in ph[8:16]]}
    print(json.dumps({"config": a.config, "ncols": len(C), "flush": a.flush, **out}))


if __name__ == "__main__":
    main()
