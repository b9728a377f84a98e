"""World-size-2 `gloo` run of the multi-GPU decomposition on CPU:
bench.py splits the batched workload's own systems (cfg3) into disjoint
contiguous per-rank ranges with no data-path collective, single-system workloads run as replicas,
and the whole-job time is the max over ranks (the only collective)."""

import dataclasses
import hashlib
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, world: int, port: int, out):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        from paper_2201_09827_b200 import problems

        spec = dataclasses.replace(problems.CONFIGS["cfg3"], batch=5)
        idx = list(bench.shard_systems(spec, rank, world))
        a, b = bench._inputs(spec, rank, world)
        digest = hashlib.sha256(a.tobytes() + b.tobytes()).hexdigest()
        first_ok = bool(np.array_equal(a[0], problems.config_problem(spec, idx[0])[0]))
        single = list(bench.shard_systems(problems.CONFIGS["cfg2a"], rank, world))
        tmax = bench.max_over_ranks(1.5 + rank, dist, "cpu")
        gathered = [None] * world
        dist.all_gather_object(gathered, (idx, digest, first_ok, single, tmax))
        if rank == 0:
            out.put(gathered)
    finally:
        dist.destroy_process_group()


def test_two_rank_sharding_and_timing():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (i0, d0, ok0, s0, t0), (i1, d1, ok1, s1, t1) = res
    # cfg3: the configuration's systems split into disjoint, contiguous shards
    # (ceil(batch / world) each); each rank built its own systems
    assert i0 == [0, 1, 2] and i1 == [3, 4]
    assert ok0 and ok1 and d0 != d1
    # single-system workload: replicas of the same system
    assert s0 == s1 == [0]
    # the whole-job time is the slowest rank's
    assert t0 == t1 == 2.5


def _sweep_worker(rank: int, world: int, port: int, out):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2201_09827_b200 import harness
        from paper_2201_09827_b200.precision import PrecisionTriple
        from paper_2201_09827_b200.refine import Method

        # mtx problems that do not exist: each rank records its own in-row
        # errors without touching a GPU, so the deal + gather logic is what runs
        refs = [harness.Problem.from_text(f"mtx:/nonexistent/p{i}_r.mtx") for i in range(5)]
        spec = harness.SweepSpec(refs, [Method.GMRES_IR, Method.RGMRES_IR],
                                 PrecisionTriple.parse("single", "double", "quad"), m=16, k=4)
        rows = harness.run_sweep_ranks(spec)
        out.put((rank, [(r["problem_id"], r["method"], r["k"]) for r in rows]))
    finally:
        dist.destroy_process_group()


def test_two_rank_sweep_deal_and_gather():
    """run_sweep_ranks: problems dealt round-robin, every rank gets all rows in
    spec order (same order as the single-process run_sweep)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sweep_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = [(f"p{i}_r", m, k) for i in range(5) for m, k in (("gmres-ir", 0), ("rgmres-ir", 4))]
    assert got[0] == want and got[1] == want
