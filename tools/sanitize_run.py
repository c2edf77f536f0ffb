"""Small end-to-end exercise of every libml entry point (for compute-sanitizer runs)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import mlgen  # noqa: E402
import paper_1607_00315_b200 as ml  # noqa: E402


def run(ds, opts=None, engine=0):
    ctx = ml.Context(ds)
    if engine:
        ctx.ml_set_engine(engine)
    rng = np.random.default_rng(0)
    w = np.zeros(ds.n)
    idx = rng.choice(ds.n, max(1, ds.n // 10), replace=False)
    w[idx] = rng.normal(0, 0.1, len(idx))
    ctx.ml_set_w(torch.from_numpy(w).cuda())
    F, g, h = ctx.ml_eval_f_grad()
    C = torch.from_numpy(np.sort(rng.choice(ds.n, max(1, ds.n // 3), replace=False)).astype(np.int32)).cuda()
    ctx.ml_eval_f_grad(C)
    ctx.ml_diag_hess(C)
    ctx.ml_hessvec(C, torch.randn(C.numel(), dtype=torch.float64, device="cuda"))
    ctx.ml_select_coarse(g, ds.n // 4)
    gC = g[C.long()].contiguous()
    hC = h[C.long()].contiguous()
    ctx.ml_shrink_linesearch(C, gC, h=hC)
    r = ctx.ml_solve(opts or ml.default_opts())
    torch.cuda.synchronize()
    print(ds.name, "ok", r["status"], r["cycles"], r["kappa"])


if __name__ == "__main__":
    run(mlgen.make(1))
    run(mlgen.make(2, m=300, n=3000))                      # small-m paths (TMA smem passes, persistent inner)
    run(mlgen.make(3, m=20000, n=30000))                   # large-m paths (atomic scatter, heavy units)
    run(mlgen.random_sparse(777, 1301, 0.02, seed=5, empty_rows=9, empty_cols=40))
    run(mlgen.onehot(3000, 3)[0])
    run(mlgen.make(1), ml.default_opts(inner_cg=2))
    # short columns on the large-m path (thread-per-column tiles, two-pass finest gather), then the heavy-column path
    # forced on (padded row-major copy, vector loads)
    run(mlgen.make(5, m=12000, n=120000))
    run(mlgen.make(5, m=12000, n=120000), engine=1 << 4)
    run(mlgen.make(4, m=20000, n=40000), engine=1 << 4)
    run(mlgen.make(2, m=300, n=3000), ml.default_opts(continuation=1))
    run(mlgen.make(3, m=20000, n=30000), ml.default_opts(continuation=1))
