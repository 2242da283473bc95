"""The N > 1 path of bench.py on CPU: two ranks over gloo (127.0.0.1).  Every
rank works on its own seeded batch (weak scaling, no data-path collective);
only the timings are reduced (max over ranks) and rank 0 reports."""
import io
import os
import socket
import sys
from contextlib import redirect_stdout

import pytest
import torch
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update({"RANK": str(rank), "WORLD_SIZE": str(world), "LOCAL_RANK": str(rank),
                       "MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port)})
    sys.path.insert(0, ROOT)
    import bench
    import workloads
    import torch.distributed as dist

    class A:  # the subset of bench arguments the reference arm reads
        gpus, steps, warmup, config, ref_seconds, scale = world, 1, 1, 2, 1.0, 0.001

    r, w, _ = bench.dist_init(A)
    out = {"rank": r, "world": w, "backend": dist.get_backend()}
    # timings: each rank reports its own, the job sees the max
    out["reduced"] = bench.reduce_max([10.0 + r, 3.0 * (r + 1), 1.0], w)
    out["gbs"] = bench.job_gbs(w, 1_000_000_000, 4, out["reduced"][0])
    # per-rank data: seeded by rank, different batches, same shape
    x = workloads.generate(2, scale=0.001, seed=r)
    out["x_sum"] = int(x.to(torch.int64).sum())
    out["x_n"] = x.numel()
    # reference arm: rank 0 alone prints its line
    buf = io.StringIO()
    with redirect_stdout(buf):
        bench.run_reference(A, r, w)
    out["ref_lines"] = [l for l in buf.getvalue().splitlines() if l.startswith("{")]
    dist.barrier()
    dist.destroy_process_group()
    q.put(out)


def test_two_ranks_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=240) for _ in procs), key=lambda d: d["rank"])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [d["world"] for d in res] == [2, 2]
    assert all(d["backend"] == "gloo" for d in res)
    for d in res:  # max over ranks, identical on every rank
        assert d["reduced"] == [11.0, 6.0, 1.0]
        assert d["gbs"] == pytest.approx(2 * 1e9 * 4 / (11.0e-3) / 1e9)
    assert res[0]["x_n"] == res[1]["x_n"] and res[0]["x_sum"] != res[1]["x_sum"]
    assert len(res[0]["ref_lines"]) == 1 and res[1]["ref_lines"] == []
