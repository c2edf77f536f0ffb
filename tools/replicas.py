"""Batched replicas: P contexts of the same problem, each on its own stream and host thread, each
with its cooperative kernels capped at SMs / P CTAs (ml_set_sm_share), solving side by side.  Reports solves per
second against P = 1 on the whole GPU (wall clock around all threads, device synchronised on both sides)."""
import argparse
import json
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import mlgen  # noqa: E402
import paper_1607_00315_b200 as ml  # noqa: E402


def run(ds, P, solves):
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    streams = [torch.cuda.Stream() for _ in range(P)]
    ctxs = [ml.Context(ds, stream=s) for s in streams]
    for c in ctxs:
        c.ml_set_sm_share(sms // P)
        c.ml_solve()
    torch.cuda.synchronize()
    reps = [[] for _ in range(P)]

    def work(k):
        for _ in range(solves):
            reps[k].append(ctxs[k].ml_solve())

    th = [threading.Thread(target=work, args=(k,)) for k in range(P)]
    t0 = time.perf_counter()
    for t in th:
        t.start()
    for t in th:
        t.join()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    ok = all(r["status"] == 0 and r["kappa"] <= 1e-6 for rs in reps for r in rs)
    nnz = sum(r["nnz_touched"] for rs in reps for r in rs)
    return {"replicas": P, "blocks_each": sms // P, "solves": P * solves, "seconds": round(dt, 4),
            "solves_per_s": round(P * solves / dt, 1), "ms_per_solve_each": round(dt / solves * 1e3, 3),
            "x_gbs": round(8.0 * nnz / dt / 1e9, 1), "all_converged": ok, "F": reps[0][-1]["F"]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--solves", type=int, default=40)
    ap.add_argument("--replicas", default="1,2,4,8")
    a = ap.parse_args()
    ds = mlgen.make(a.config)
    for P in [int(x) for x in a.replicas.split(",")]:
        print(json.dumps({"workload": ds.name, **run(ds, P, a.solves)}))


if __name__ == "__main__":
    main()
