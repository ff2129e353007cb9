"""bench.py's N > 1 plumbing (replicas, max-over-ranks device time) on CPU with gloo, world 2.
The GPU box has one GPU, so the multi-rank path is covered here (no collective on the data
path: each replica builds and applies its own H-hat; only the timing is reduced)."""
import os
import socket
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch.distributed as tdist
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    ms = bench.max_over_ranks(10.0 + 5.0 * rank)          # rank 1 is the slow one
    tdist.barrier()
    out.put((rank, ms, bench.job_gbps(1_000_000_000, 4, world, ms)))
    tdist.destroy_process_group()


def test_max_over_ranks_and_job_throughput_gloo_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ms, gbps in res:
        assert ms == 15.0                                   # every rank sees the max
        assert gbps == pytest.approx(1e9 * 4 * 2 / 0.015 / 1e9)


def test_single_process_identity():
    sys.path.insert(0, ROOT)
    import bench
    assert bench.max_over_ranks(3.5) == 3.5
    assert bench.job_gbps(2_000_000_000, 10, 1, 20.0) == pytest.approx(1000.0)


def test_reference_arm_rank_nonzero_is_silent(capsys):
    sys.path.insert(0, ROOT)
    import bench

    class A:
        config, nrhs, steps, warmup = "2d_tiny", 1, 1, 3
    assert bench.run_reference(A(), rank=1, world=2) is None
    assert capsys.readouterr().out == ""
