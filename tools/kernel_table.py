"""Per-kernel (API pass) timings on a BASELINE config: warm (inputs left in L2 by the previous repetition) and cold
(L2 flushed by writing 256 MB before each repetition), p10 / median / p90 over --reps repetitions, CUDA events on the
library's stream.  GB/s = algorithmic bytes (8 B per nonzero streamed, the pass's vectors once) / time.

Usage: python tools/kernel_table.py --config 5 [--reps 20] > gpurun_out/kernels_cfg5.json
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import mlgen  # noqa: E402
import paper_1607_00315_b200 as ml  # noqa: E402


def times(fn, reps, stream, flush):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        if flush is not None:
            flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return np.array(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    ds = mlgen.make(a.config)
    m, n, nnz = ds.m, ds.n, ds.nnz
    ctx = ml.Context(ds)
    st = ctx.stream
    ctx.ml_solve()   # the solution's support: the C of the restricted passes
    w = ctx.ml_get_w()
    S = torch.nonzero(w).flatten().to(torch.int32)
    lens = np.diff(ds.csc_colptr.astype(np.int64))
    Sh = S.cpu().numpy()
    nnzS = int(lens[Sh].sum())
    vS = torch.randn(len(Sh), dtype=torch.float64, device="cuda")
    vall = torch.randn(n, dtype=torch.float64, device="cuda")
    ctx.ml_eval_f_grad(want_g=False, want_h=False)
    _, g, h = ctx.ml_eval_f_grad(S)
    _, gall, _ = ctx.ml_eval_f_grad()
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
    import ctypes
    sel_out = torch.zeros(n, dtype=torch.int32, device="cuda")
    sel_n = ctypes.c_int64()

    def select():   # (the C call with a preallocated output: the binding's allocation is not the library's)
        ml.load().ml_select_coarse(ctx.h, ctypes.c_void_p(gall.data_ptr()), 2 * len(Sh),
                                   ctypes.c_void_p(sel_out.data_ptr()), ctypes.byref(sel_n))

    # (name, call, algorithmic bytes: X bytes + vectors)
    cases = [
        ("A1 margins (CSR, all rows)", lambda: ctx.ml_eval_f_grad(want_g=False, want_h=False),
         8 * nnz + 4 * (m + 1) + m + 24 * m),
        ("A1+A2 eval_f_grad (all columns)", lambda: ctx.ml_eval_f_grad(),
         (8 * nnz + 4 * (m + 1) + m + 24 * m) + (8 * nnz + 8 * (n + 1) + 16 * m + 16 * n)),
        ("A2 diag_hess (all columns)", lambda: ctx.ml_diag_hess(None), 8 * nnz + 8 * (n + 1) + 8 * m + 8 * n),
        ("A2 diag_hess (support)", lambda: ctx.ml_diag_hess(S), 8 * nnzS + 12 * len(Sh) + 8 * m),
        ("A5 hessvec (support)", lambda: ctx.ml_hessvec(S, vS), 2 * 8 * nnzS + 24 * len(Sh) + 24 * m),
        ("A5 hessvec (all columns)", lambda: ctx.ml_hessvec(None, vall), 2 * 8 * nnz + 24 * n + 24 * m),
        ("A8 select_coarse (all n, k = 2|S|)", select, 8 * n + 4 * 2 * len(Sh)),
    ]
    out = {"config": a.config, "m": m, "n": n, "nnz": nnz, "support": len(Sh), "nnz_support": nnzS,
           "reps": a.reps, "kernels": []}
    for name, fn, nbytes in cases:
        row = {"kernel": name, "algorithmic_MB": round(nbytes / 1e6, 2)}
        for mode, fl in (("warm", None), ("cold", flush)):
            t = times(fn, a.reps, st, fl)
            p10, p50, p90 = (float(np.percentile(t, q)) for q in (10, 50, 90))
            row[mode] = {"ms_p10": round(p10, 4), "ms_p50": round(p50, 4), "ms_p90": round(p90, 4),
                         "GBs_p50": round(nbytes / p50 / 1e6, 1), "pct_of_6530": round(100 * nbytes / p50 / 1e6 / 6530, 1)}
        out["kernels"].append(row)
    hv = out["kernels"][4]["warm"]["ms_p50"]
    out["hessvec_per_s_support_warm"] = round(1e3 / hv, 1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
