"""Multi-process host logic on CPU (gloo, world_size 2).

Each rank takes its stream range from the C-ABI partitioner (xg_partition),
generates its slice with the ORACLE (the checker; the device path is covered
by the gpu tests), and the ranks' slices gathered in rank order must equal
the single-process fill -- the schedule-independence test of
proj/tests/test_parallel.cpp:132-143 lifted to processes.  The Monte Carlo
workload's one collective (a uint64 hit-count sum) is exercised the same way.
"""
import json
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


def _bench_cmd(*args, env=None):
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    e = dict(os.environ)
    e.pop("WORLD_SIZE", None)
    e.update(env or {})
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), *args], capture_output=True,
                       text=True, timeout=900, env=e, cwd="/tmp")
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    _bench_cmd.stdout = r.stdout
    return r.returncode, (json.loads(lines[-1]) if lines else None), r.stderr


def test_bench_self_launches_n_ranks_dry_run():
    """`python bench.py --gpus 2` outside torchrun re-launches itself with 2
    ranks (torch.distributed.run, 127.0.0.1) -- the driver's own command is
    an N-rank job; the dry run checks world, slices and max-over-ranks on CPU."""
    rc, line, err = _bench_cmd("--gpus", "2", "--dry-run")
    assert rc == 0, err[-2000:]
    assert line["n_gpus"] == 2 and line["comm"]["nranks"] == 2
    assert line["max_over_ranks"] == 2.0
    assert [s["fill_2p34"][0] for s in line["slices"]] == [0, 1 << 17]


def _gpu_slice_worker(rank, world, port, q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist

    import paper_1108_0486_b200 as xg
    from paper_1108_0486_b200.digest import row_digests

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    first, count = xg.partition(1000, world, rank)
    e = xg.BlockEnsemble(xg.xorgensgp32_params(), 1, count, 63, first_stream=first)
    x, s, ws = row_digests(e.fill_u32(4096))
    hits = torch.tensor([int(xg.BlockEnsemble(xg.xorgensgp32_params(), 1, count, 63,
                                              first_stream=first).mc_pi(320).item())])
    dist.all_reduce(hits)
    g = [None] * world
    dist.all_gather_object(g, (first, x, s, ws))
    if rank == 0:
        q.put((g, int(hits.item())))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_gloo_ranks_generate_slices_on_the_gpu(world):
    """Ranks (sharing one GPU) generate their partition slices with the GPU
    path; the digests gathered in rank order equal the single-process fill's,
    and the all-reduced MC count equals the single ensemble's."""
    import torch

    import paper_1108_0486_b200 as xg
    from paper_1108_0486_b200.digest import row_digests

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_slice_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    g, hits = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    e = xg.BlockEnsemble(xg.xorgensgp32_params(), 1, 1000, 63)
    x, s, ws = row_digests(e.fill_u32(4096))
    assert [f for f, *_ in g] == [xg.partition(1000, world, r)[0] for r in range(world)]
    assert np.array_equal(np.concatenate([t[1] for t in g]), x)
    assert np.array_equal(np.concatenate([t[2] for t in g]), s)
    assert np.array_equal(np.concatenate([t[3] for t in g]), ws)
    assert hits == int(xg.BlockEnsemble(xg.xorgensgp32_params(), 1, 1000, 63).mc_pi(320).item())
    del torch


@pytest.mark.gpu
@pytest.mark.parametrize("workload", ["fill_u32", "fill_2p34", "mc_pi"])
def test_bench_two_ranks_self_launched_gloo(workload):
    """The driver's N = 2 command through the self-launch path, two gloo ranks
    on one GPU: n_gpus 2, and every rank's slice passes the full-size parity
    check (tests/golden/full_size.json)."""
    rc, line, err = _bench_cmd("--gpus", "2", "--workload", workload, "--steps", "3", "--warmup", "3",
                               "--no-cpu", "--no-e2e", "--no-extra", "--sustained-s", "0",
                               env={"XG_BENCH_BACKEND": "gloo"})
    assert rc == 0, err[-3000:]
    assert line["n_gpus"] == 2 and line["comm"]["nranks"] == 2
    assert line["parity"]["checked"] and line["parity"]["ok"], line["parity"]
    if workload == "mc_pi":
        assert line["mc"]["allreduce_in_step"]


@pytest.mark.gpu
def test_bench_default_line_contract():
    """The driver's default command (short): one JSON line with the contract
    keys, a roofline with the measured write ceiling, the sustained leg, e2e
    with the copied bytes, and every BASELINE config in extra_workloads with
    its roofline and a passing full-size parity check."""
    rc, line, err = _bench_cmd("--gpus", "1", "--steps", "3", "--warmup", "3", "--sustained-s", "0.3",
                               "--no-cpu")
    assert rc == 0, err[-3000:]
    # stdout is the one JSON line (NCCL's log is forwarded to stderr)
    assert _bench_cmd.stdout.strip().count("\n") == 0, _bench_cmd.stdout[:2000]
    # N = 1 runs the job's collective through a one-rank NCCL communicator
    assert line["comm"]["backend"] == "nccl" and line["comm"]["nranks"] == 1, line["comm"]
    assert "NCCL INFO" in err and "nRanks 1" in err
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "gpu_launches", "clocks", "roofline",
              "e2e", "parity", "sustained", "extra_workloads"):
        assert k in line, k
    assert line["n_gpus"] == 1 and line["gpu_launches"] == 3
    r = line["roofline"]
    assert r["bound"] == "hbm" and r["frac"] > 0.5 and r["write_ceiling_gbs"] > 1000
    assert line["e2e"]["d2h_bytes_per_step"] == 4 << 30 and line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["parity"]["checked"] and line["parity"]["ok"]
    assert set(line["extra_workloads"]) == {"fill_f32", "fill_f64", "fill_2p34", "mc_pi", "stream1"}
    for name, e in line["extra_workloads"].items():
        assert e["parity"]["checked"] and e["parity"]["ok"], name
        assert e["roofline"]["frac"] and e["roofline"]["frac"] > (0.2 if name == "stream1" else 0.5), name
    assert abs(line["extra_workloads"]["mc_pi"]["mc"]["pi_estimate"] - 3.14159265) < 1e-4
    assert line["extra_workloads"]["mc_pi"]["mc"]["allreduce_in_step"]
    for name in ("fill_f32", "fill_f64", "mc_pi", "stream1"):
        e2e = line["extra_workloads"][name]["e2e"]
        assert e2e["value"] > 0 and e2e["h2d_bytes_per_step"] == 0, name
    assert line["extra_workloads"]["fill_f64"]["e2e"]["d2h_bytes_per_step"] == 8 << 30
