"""Multi-GPU trajectory dispatcher (trajectory mode).

Quantum trajectories are independent Monte Carlo samples ("embarrassingly
parallelizable").  Rank r of N runs trajectories t = r + N*j of
the job (interleaved, which balances the variable number of conventional
channels), with no communication until the end: one all-gather of the
per-trajectory records (bitstrings, Kraus indices, observables) and a
deterministic host merge in trajectory order.  The counter-based RNG makes
every record independent of N, so the merged output is identical for N = 1,
2, 4, 8.

The collective runs through torch.distributed (NCCL on GPUs, gloo in the CPU
tests); the per-rank work is any `runner(begin, stride, count) -> dict of
numpy arrays with leading dimension count` (normally
qtraj.Context.run_trajectories bound to a plan and state buffer).
"""
from __future__ import annotations

from typing import Callable, Dict, Optional

import numpy as np


def shard(total: int, rank: int, world: int):
    """(traj_begin, traj_stride, count) of `rank` for a job of `total` trajectories."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    count = (total - rank + world - 1) // world if total > rank else 0
    return rank, world, count


def merge_records(parts, total: int) -> Dict[str, np.ndarray]:
    """parts[r] = dict of arrays for rank r (rows j <-> trajectory r + N*j).
    Returns arrays with rows in trajectory order 0..total-1."""
    world = len(parts)
    keys = [k for k in parts[0] if isinstance(parts[0][k], np.ndarray)]
    out = {}
    for k in keys:
        shape = parts[0][k].shape[1:]
        arr = np.zeros((total,) + shape, dtype=parts[0][k].dtype)
        for r, p in enumerate(parts):
            arr[r::world] = p[k]
        out[k] = arr
    return out


def aggregate(obs: np.ndarray):
    """Mean and standard error (sample sd / sqrt(r)) per observable."""
    r = obs.shape[0]
    mean = obs.mean(axis=0)
    se = obs.std(axis=0, ddof=1) / np.sqrt(r) if r > 1 else np.full_like(mean, np.nan)
    return mean, se


def aggregate_sets(obs: np.ndarray, n_sets: int, traj_begin: int = 0):
    """Parameter sweeps: rows are trajectories traj_begin, traj_begin + 1, ...
    (merged, trajectory order); trajectory t ran parameter set t mod n_sets.
    Returns (mean, stderr), each [n_sets, n_obs]."""
    t = traj_begin + np.arange(obs.shape[0])
    out = [aggregate(obs[t % n_sets == s]) for s in range(n_sets)]
    return np.stack([m for m, _ in out]), np.stack([e for _, e in out])


def _gather_rows(t, group, world):
    """all_gather of a [count_r, ...] tensor whose counts differ by at most 1 across ranks."""
    import torch
    import torch.distributed as dist
    n = torch.tensor([t.shape[0]], device=t.device, dtype=torch.int64)
    ns = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(ns, n, group=group)
    mx = int(max(int(x.item()) for x in ns))
    pad = torch.zeros((mx,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    pad[: t.shape[0]] = t
    bufs = [torch.zeros_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    return [b[: int(c.item())] for b, c in zip(bufs, ns)]


def run_sharded(runner: Callable[[int, int, int], Dict[str, np.ndarray]], total: int,
                group=None, device=None) -> Optional[Dict[str, np.ndarray]]:
    """Run this rank's shard and all-gather the records.  Every rank returns the
    merged records in trajectory order (None fields are dropped)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    begin, stride, count = shard(total, rank, world)
    mine = {k: v for k, v in runner(begin, stride, count).items() if isinstance(v, np.ndarray)}
    if world == 1:
        return merge_records([mine], total)
    parts = [dict() for _ in range(world)]
    for k in sorted(mine):
        a = np.ascontiguousarray(mine[k])
        dt = a.dtype
        if dt == np.uint64:  # torch has no uint64 collectives: move the bits as int64
            a = a.view(np.int64)
        t = torch.from_numpy(a)
        if device is not None:
            t = t.to(device)
        got = _gather_rows(t, group, world)
        for r, g in enumerate(got):
            v = g.cpu().numpy()
            parts[r][k] = v.view(np.uint64) if dt == np.uint64 else v
    return merge_records(parts, total)
