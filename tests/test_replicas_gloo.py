"""The N > 1 host path of bench.py (replicas only, DESIGN 8.4) on CPU with gloo, world size 2: the timing barrier,
the max-over-ranks time, the whole-job byte sum, and the reference arm running on rank 0 only."""
import os
import socket
import sys

import pytest
import torch
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, q):
    os.environ.update({"MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port), "RANK": str(rank),
                       "WORLD_SIZE": str(ws), "LOCAL_RANK": str(rank)})
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    import bench
    r, w, _ = bench.dist_setup(ws, backend="gloo")
    bench.barrier(w)
    # rank k streamed (k + 1) GB in (10 + 5 k) ms
    value, t_max = bench.aggregate(float(r + 1) * 1e9, 10.0 + 5.0 * r, w, torch.device("cpu"))
    ref = bench.run_reference(type("A", (), {"config": 1, "warmup": 1, "steps": 1, "gpus": w})()) if r == 1 else "skip"
    q.put((r, value, t_max, ref))
    dist.destroy_process_group()


def test_two_replicas_gloo():
    ws, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, q)) for r in range(ws)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in range(ws))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r, value, t_max, _ in out:
        assert t_max == pytest.approx(15.0)
        assert value == pytest.approx(3e9 / 15e-3 / 1e9)   # (1 + 2) GB / 15 ms, the same on every rank
    assert out[1][3] is None   # the reference arm does no work on rank != 0
