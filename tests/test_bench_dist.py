"""bench.py's multi-process plumbing on the CPU (gloo, world size 2): one replica per
rank, barrier, timing reduced as the max over ranks, distinct replica seeds, and the
reference arm running on rank 0 only (replicas only, no data-path
collective)."""
import os
import socket
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(RANK=str(rank), LOCAL_RANK=str(rank), WORLD_SIZE=str(world),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    import bench
    import paper_2605_18254_b200 as srm
    w, r, loc, pg = bench.dist_setup()
    assert (w, r, loc) == (world, rank, rank) and pg is not None
    bench.barrier(pg)
    m = bench.max_over_ranks(pg, 10.0 + rank)  # per-rank device ms -> job time
    seed = srm.mix_seed(20260101, rank)        # the replica seed run_b200 uses
    # the reference arm: rank != 0 exits without work
    class A:  # minimal args
        steps, warmup = 1, 0
    rc = bench.run_reference(A, bench.CONFIGS["cfg1"], w, r, pg) if r != 0 else None
    out.put((rank, m, seed, rc))
    pg.destroy_process_group()


def test_two_rank_gloo_plumbing():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=240) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [m for _, m, _, _ in res] == [11.0, 11.0]       # max over ranks
    assert res[0][2] != res[1][2]                          # independent replicas
    assert res[1][3] == 0                                  # reference arm: rank 1 idle
