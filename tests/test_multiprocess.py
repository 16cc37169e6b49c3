"""Multi-process host logic on CPU (gloo, world_size 2).

Each rank takes its stream range from the C-ABI partitioner (xg_partition),
generates its slice with the ORACLE (the checker; the device path is covered
by the gpu tests), and the ranks' slices gathered in rank order must equal
the single-process fill -- the schedule-independence test of
proj/tests/test_parallel.cpp:132-143 lifted to processes.  The Monte Carlo
workload's one collective (a uint64 hit-count sum) is exercised the same way.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, total, per, q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist

    import paper_1108_0486_b200 as xg
    from oracle import Oracle

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    first, count = xg.partition(total, world, rank)
    o = Oracle()
    o.threads = 2
    words = o.ensemble(1, count, first_stream=first).fill_u32(per)
    # gather the variable-size slices in rank order
    gathered = [None] * world
    dist.all_gather_object(gathered, (first, count, words))
    sizes = [(f, c) for f, c, _ in gathered]
    slices = [w for _, _, w in gathered]
    # Monte Carlo hit count: per-rank count + one all-reduce (sum)
    hits = torch.tensor([int(o.ensemble(1, count, first_stream=first).mc_hits(320).sum())],
                        dtype=torch.int64)
    dist.all_reduce(hits)
    if rank == 0:
        q.put((np.concatenate(slices), int(hits.item()), sizes))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,total", [(2, 64), (2, 7)])
def test_gloo_partitioned_fill_equals_single(world, total, oracle):
    per = 300
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, total, per, q)) for r in range(world)]
    for p in procs:
        p.start()
    words, hits, sizes = q.get(timeout=60)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    single = oracle.ensemble(1, total).fill_u32(per)
    assert np.array_equal(words, single)
    assert hits == int(oracle.ensemble(1, total).mc_hits(320).sum())
    assert sum(c for _, c in sizes) == total


def _bench_worker(rank, world, port, q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist

    import bench

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    t = bench.max_over_ranks(float(rank + 1) * 1.5, world)
    geo = {wl: bench.workload_geometry(wl, world, rank)
           for wl in ("fill_u32", "fill_f64", "fill_2p34", "mc_pi")}
    gathered = [None] * world
    dist.all_gather_object(gathered, geo)
    if rank == 0:
        q.put((t, gathered))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_bench_multirank_logic(world):
    """bench.py's N>1 bookkeeping on gloo: max-over-ranks timing and the
    per-rank stream slices (weak: disjoint 2^14-stream blocks; strong: a
    partition of one global ensemble) that make up the job."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    t, geos = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert t == 1.5 * world
    for wl, total_streams in (("fill_2p34", 1 << 18), ("mc_pi", 1 << 17)):
        spans = [g[wl] for g in geos]
        pos = 0
        for first, count, per, scaling, job in spans:
            assert first == pos and scaling == "strong"
            pos += count
        assert pos == total_streams
        assert spans[0][4] == (1 << 34 if wl == "fill_2p34" else 1 << 41)
    firsts = sorted(g["fill_u32"][0] for g in geos)
    assert firsts == [r * (1 << 14) for r in range(world)]
    assert all(g["fill_u32"][4] == (1 << 30) * world for g in geos)
    assert all(g["fill_f64"][4] == (1 << 31) * world for g in geos)
