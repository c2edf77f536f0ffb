"""Solve a BASELINE config and write w (and the trace) to an .npy file: compare two builds of libml bit for bit
(ML_LIB=<path> selects the build).  Usage: python tools/bitcmp.py --config 2 --out a.npy"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import mlgen  # noqa: E402
import paper_1607_00315_b200 as ml  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    ds = mlgen.make(a.config)
    ctx = ml.Context(ds)
    rep = ctx.ml_solve()
    w = ctx.ml_get_w().cpu().numpy()
    tr = np.array([[r["F_before"], r["F_after"], r["alpha"]] for r in ctx.trace()])
    np.save(a.out, np.concatenate([w, tr.ravel(), [rep["F"], rep["kappa"]]]))
    print(a.config, rep["cycles"], rep["F"], rep["kappa"])


if __name__ == "__main__":
    main()
