"""Trajectory sharding across ranks (world size 2, gloo, CPU).

The per-rank runner is the CPU oracle here (tests may use it); the dispatcher
itself never imports the oracle.  The merged records of a 2-rank run must be
byte-identical to a single-process run of the same trajectory indices
(counter-based RNG: records are independent of the rank count)."""
import os
import socket

import numpy as np
import pytest

from paper_2111_02396_b200 import dispatch


def test_shard_partitions_indices():
    for total in (0, 1, 7, 10000):
        for world in (1, 2, 3, 8):
            seen = []
            for r in range(world):
                b, s, c = dispatch.shard(total, r, world)
                seen += [b + s * j for j in range(c)]
            assert sorted(seen) == list(range(total))


def test_merge_and_aggregate():
    parts = [{"x": np.arange(0, 10, 2)[:, None] * 1.0}, {"x": np.arange(1, 10, 2)[:, None] * 1.0}]
    m = dispatch.merge_records(parts, 10)
    assert (m["x"][:, 0] == np.arange(10)).all()
    mean, se = dispatch.aggregate(m["x"])
    assert mean[0] == 4.5 and abs(se[0] - np.arange(10).std(ddof=1) / np.sqrt(10)) < 1e-15


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, total, q):
    import torch.distributed as dist
    import oracle
    import workloads
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    c = workloads.random_circuit(5, 5, seed=2, noise="both", p=0.05, t1_ns=400.0, tphi_ns=700.0, readout=True)

    def runner(begin, stride, count):
        r = oracle.run_trajectories(c, seed=41, traj_begin=begin, stride=stride, traj_count=count, shots=2,
                                    threads=1)
        return {"bits": r["bits"], "kraus": r["kraus"], "obs": r["obs"]}

    merged = dispatch.run_sharded(runner, total)
    if rank == 0:
        q.put({k: v.copy() for k, v in merged.items()})
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_matches_single_process():
    import multiprocessing as mp
    import oracle
    import workloads
    total = 23
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, total, q)) for r in range(2)]
    for p in ps:
        p.start()
    merged = q.get(timeout=240)
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    c = workloads.random_circuit(5, 5, seed=2, noise="both", p=0.05, t1_ns=400.0, tphi_ns=700.0, readout=True)
    ref = oracle.run_trajectories(c, seed=41, traj_count=total, shots=2)
    assert (merged["bits"] == ref["bits"]).all()
    assert (merged["kraus"] == ref["kraus"]).all()
    assert np.array_equal(merged["obs"], ref["obs"])
