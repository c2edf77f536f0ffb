"""Full-size solve parity for one BASELINE config outside the test suite (cfg 5's oracle solve takes minutes):
GPU vs oracle F, kappa, supports outside the band ||g_j| - lambda| < 1e-4.  Prints one JSON line."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import mlgen  # noqa: E402
import oracle  # noqa: E402
import paper_1607_00315_b200 as ml  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    a = ap.parse_args()
    ds = mlgen.make(a.config)
    ctx = ml.Context(ds)
    r_g = ctx.ml_solve()
    w_g = ctx.ml_get_w().cpu().numpy()
    o = oracle.Oracle(ds)
    t0 = time.perf_counter()
    r_o = o.solve()
    t_o = time.perf_counter() - t0
    w_o = o.get_w()
    _, g_o, _ = o.eval_f_grad()
    band = np.abs(np.abs(g_o) - ds.lam) < 1e-4
    mism = int(np.sum(((w_g != 0) != (w_o != 0)) & ~band))
    out = {"config": a.config, "F_gpu": r_g["F"], "F_oracle": r_o["F"], "F_rel": abs(r_g["F"] - r_o["F"]) / abs(r_o["F"]),
           "kappa_gpu": r_g["kappa"], "kappa_oracle": r_o["kappa"], "cycles_gpu": r_g["cycles"], "cycles_oracle": r_o["cycles"],
           "nnz_w_gpu": r_g["nnz_w"], "nnz_w_oracle": r_o["nnz_w"], "support_mismatch_outside_band": mism,
           "band_columns": int(band.sum()), "oracle_seconds": round(t_o, 1),
           "pass": bool(abs(r_g["F"] - r_o["F"]) <= 1e-6 * abs(r_o["F"]) and r_g["kappa"] <= 1e-6 and mism == 0)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
