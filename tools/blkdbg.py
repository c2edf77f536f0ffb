"""Per-block balance of the large-m persistent solver's S (X_A s) and G (X_A^T sv) work, from a -DIR_BLKDBG build
(tph[0..5]: sum / max / 2^62 - min over blocks of each block's S and G work in a launch, before the grid barriers).

Usage: nvcc ... -DIR_BLKDBG -o paper_1607_00315_b200/libml_blkdbg.so; ML_LIB=.../libml_blkdbg.so python tools/blkdbg.py --config 5
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
    ctx.ml_inner_phases(reset=True)
    r = ctx.ml_solve()
    torch.cuda.synchronize()
    ph = ctx.ml_inner_phases(reset=True)
    nl = sum(1 for t in ctx.trace() if t["inner_iters"] > 0)
    G = min(torch.cuda.get_device_properties(0).multi_processor_count, 160)
    out = {"config": a.config, "launches": nl, "blocks": G}
    for k, nm in ((0, "S"), (3, "G")):
        out[nm] = {"avg_us_per_launch": round(ph[k] / 1e3 / (G * nl), 1), "max_us": round(ph[k + 1] / 1e3, 1),
                   "min_us": round(((1 << 62) - ph[k + 2]) / 1e3, 1)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
