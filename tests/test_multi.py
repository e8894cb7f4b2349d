"""The N>1 path of bench.py (source-sharded replicas) on CPU with
gloo, world size 2: the only collectives are the max of the per-rank step time
and the sum of the per-rank traversed edges (metric bookkeeping, not data path)."""
import os
import socket

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    ms = 1.0 + 2.0 * rank            # rank 1 is slower
    t = bench.replica_max(ms, world, dist, "cpu")
    e = bench.replica_sum(1e9 * (rank + 1), world, dist, "cpu")   # ranks traverse different edges
    v = bench.replica_value(e, t)
    out[rank] = (t, v)
    dist.barrier()
    dist.destroy_process_group()


def test_replica_timing_is_max_over_ranks():
    world = 2
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    for r in range(world):
        t, v = out[r]
        assert t == 3.0                       # max over ranks, every rank agrees
        assert abs(v - 3e9 / 3e-3 / 1e9) < 1e-9  # (1e9 + 2e9) edges / 3 ms


def test_single_rank_identity():
    import bench
    assert bench.replica_max(1.5, 1) == 1.5
    assert bench.replica_sum(7.0, 1) == 7.0
    assert bench.replica_value(2e9, 2.0) == pytest.approx(1000.0)


def test_source_sharding():
    """Rank r takes entries [8r, 8r+8) of the sequential seeded sample: disjoint
    shards, rank 0's equal the N=1 sources; a single-source config repeats."""
    import bench
    import graphgen
    import numpy as np
    cand = np.arange(10_000)
    one = graphgen.choose_sources(cand, 8, 102)
    four = graphgen.choose_sources(cand, 32, 102)
    assert four[:8] == one
    shards = [bench.shard_sources(four, r, 4, 8) for r in range(4)]
    assert shards[0] == one and len({s for sh in shards for s in sh}) == 32
    assert bench.shard_sources([0], 3, 4, 1) == [0]


def test_reference_arm_nonzero_rank_prints_nothing(monkeypatch):
    import bench

    class A:
        workload, algo, steps, warmup = "c1", "bfs", 1, 0
    assert bench.run_reference(A, rank=1, world=2) is None


def test_reference_arm_cpu_c1():
    """--impl reference on CPU: the oracle on c1 (graph built on the host)."""
    import bench

    class A:
        workload, algo, steps, warmup = "c1", "bfs", 1, 0
    out = bench.run_reference(A, rank=0, world=1)
    assert out["impl"] == "reference" and out["value"] > 0 and out["unit"] == "GTEPS"
    assert out["e2e"]["h2d_bytes_per_step"] == 0 and out["cpu_baseline"]["kind"] == "oracle"
