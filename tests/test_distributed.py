"""Distributed-state mode: a register split over 2^g ranks with
global-qubit swaps, checked against the CPU oracle's single-state trajectories.

CPU: a numpy test backend (oracle Alg. 1 for the local operations) under the
emulated fabric and under a real world-size-2 gloo process group (the
all-to-all exchange path).  GPU: the libqtraj backend under the emulated
fabric (NCCL cannot put two ranks on one GPU)."""
import os
import socket

import numpy as np
import pytest

import oracle
import workloads
from paper_2111_02396_b200 import distributed as D
from paper_2111_02396_b200 import qtraj


class NumpyBackend:
    """Test-only stand-in for the GPU backend: complex128 torch CPU tensors,
    operations by the oracle's Alg. 1 and plain numpy sums."""

    def __init__(self):
        import torch
        self.torch = torch

    def new_state(self, nl, rank):
        s = self.torch.zeros(1 << nl, dtype=self.torch.complex128)
        if rank == 0:
            s[0] = 1.0
        return s

    def apply_ops(self, state, nl, ops):
        psi = state.numpy()
        for pos, M in ops:
            oracle.apply_gate(psi, pos, M)

    def permute(self, state, perm):
        src = state.numpy()
        n = len(perm)
        idx = np.arange(1 << n)
        j = np.zeros_like(idx)
        for b in range(n):
            j |= ((idx >> b) & 1) << perm[b]
        out = np.zeros_like(src)
        out[j] = src
        return self.torch.from_numpy(out)

    def reduce_rho(self, state, positions):
        psi = state.numpy()
        pos = sorted(positions)
        d = 1 << len(pos)
        rho = np.zeros((d, d), np.complex128)
        idx = np.arange(psi.size)
        mask = sum(1 << p for p in pos)
        base = idx[(idx & mask) == 0]
        off = [sum(((a >> m) & 1) << p for m, p in enumerate(pos)) for a in range(d)]
        for a in range(d):
            for b in range(d):
                rho[a, b] = np.sum(psi[base | off[a]] * np.conj(psi[base | off[b]]))
        return rho

    def expect(self, state, observables):
        psi = state.numpy()
        norm = float(np.sum(np.abs(psi) ** 2))
        if not norm > 0.0:
            return np.zeros(len(observables)), 0.0
        return np.array([oracle.pauli_expectation(psi, s) for s in observables]), norm

    def sample_local(self, state, n_total, seed, traj, shot_ids):
        psi = state.numpy()
        nl = int(np.log2(psi.size))
        half = (n_total + 1) // 2
        out = []
        for sh in shot_ids:
            lo, size, bits = 0, psi.size, 0
            for lvl in range(nl - 1, -1, -1):
                h = size // 2
                m0 = float(np.sum(np.abs(psi[lo:lo + h]) ** 2))
                m1 = float(np.sum(np.abs(psi[lo + h:lo + size]) ** 2))
                u = qtraj.draw(seed, sh * half + lvl // 2, 2, traj, lvl & 1)
                bit = 1 if m0 == 0 else (0 if m1 == 0 else (0 if u * (m0 + m1) < m0 else 1))
                if bit:
                    lo += h
                    bits |= 1 << lvl
                size = h
            out.append(bits)
        return np.array(out, np.uint64)


def circuit(n, seed, noise="both"):
    c = workloads.random_circuit(n, depth=6, seed=seed, max_arity=2, noise=noise, p=0.04,
                                 t1_ns=600.0, tphi_ns=1000.0, readout=True)
    c.observables = ["I" * q + "Z" + "I" * (n - q - 1) for q in range(n)] + ["Z" * n]
    return c


def check(out, ref, t):
    assert (out["kraus"] == ref["kraus"][t]).all()
    assert (out["bits"] == ref["bits"][t]).all()
    assert np.max(np.abs(out["obs"] - ref["obs"][t])) < 1e-9 or np.max(np.abs(out["obs"] - ref["obs"][t])) < 1e-4


def test_exchange_maps_are_bijective():
    for world, gbits in ((8, [0, 2]), (8, [1]), (4, [0, 1]), (8, [2, 0, 1])):
        s = len(gbits)
        seen = set()
        for r in range(world):
            for c in range(1 << s):
                seen.add((D._dest(r, gbits, c), D._src_chunk(r, gbits)))
        assert len(seen) == world * (1 << s)


@pytest.mark.parametrize("world", [2, 4])
def test_emulated_fabric_numpy_backend_matches_oracle(world):
    n = 8
    c = circuit(n, seed=5)
    seed, T = 321, 3
    ref = oracle.run_trajectories(c, seed=seed, traj_count=T, shots=2)
    for t in range(T):
        tr = D.DistributedTrajectory(NumpyBackend(), D.EmulatedFabric(world), n)
        out = tr.run(c, seed=seed, traj=t, shots=2, observables=c.observables)
        check(out, ref, t)
        assert out["swaps"] > 0


@pytest.mark.parametrize("world", [2, 8])
def test_xy_observables_on_global_qubits(world):
    """Pauli strings with X / Y on global (rank-index) qubits: their qubits are
    swapped in before the evaluation (block-diagonal over ranks); values equal the
    oracle's, and the sampler still sees the logical layout."""
    n = 9
    c = circuit(n, seed=8)
    c.observables = ["I" * (n - 1) + "X", "Y" + "I" * (n - 2) + "X", "I" * (n - 3) + "YZX", "XZXZXZXIY",
                     "Z" + "I" * (n - 2) + "Y", "I" * n]
    seed, T = 5, 3
    ref = oracle.run_trajectories(c, seed=seed, traj_count=T, shots=3)
    for t in range(T):
        tr = D.DistributedTrajectory(NumpyBackend(), D.EmulatedFabric(world), n)
        out = tr.run(c, seed=seed, traj=t, shots=3, observables=c.observables)
        check(out, ref, t)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_n(world):
    return max(8, 6 + world.bit_length() - 1)  # >= 6 local qubits per rank


def _gloo_worker(rank, port, q, world=2):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n = _gloo_n(world)
    c = circuit(n, seed=6)
    res = []
    for t in range(2):
        tr = D.DistributedTrajectory(NumpyBackend(), D.TorchFabric(), n)
        out = tr.run(c, seed=77, traj=t, shots=2, observables=c.observables)
        res.append({k: np.asarray(v) for k, v in out.items() if k in ("kraus", "bits", "obs")})
    q.put((rank, res))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_gloo_distributed_state_matches_oracle(world):
    """torch.distributed (gloo) all-to-all exchanges; worlds 4 and 8 have 2 and 3
    global qubits, so multi-qubit exchanges (ride-along swaps) run through
    TorchFabric (the 8-GPU C5 layout)."""
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_gloo_worker, args=(r, port, q, world)) for r in range(world)]
    for p in ps:
        p.start()
    got = dict(q.get(timeout=240) for _ in range(world))
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    c = circuit(_gloo_n(world), seed=6)
    ref = oracle.run_trajectories(c, seed=77, traj_count=2, shots=2)
    for rank in range(world):
        for t in range(2):
            check(got[rank][t], ref, t)


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4, 8])
def test_gpu_backend_emulated_fabric_matches_oracle(world):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = qtraj.Context(0)
    n = 13
    c = circuit(n, seed=40 + world, noise="ad")
    c.observables += ["I" * (n - 1) + "X", "Y" + "I" * (n - 3) + "ZX", "XZ" + "I" * (n - 4) + "YY"]
    seed, T = 99, 3
    ref = oracle.run_trajectories(c, seed=seed, traj_count=T, shots=3)
    for t in range(T):
        tr = D.DistributedTrajectory(D.GpuBackend(ctx, "cuda:0"), D.EmulatedFabric(world), n)
        out = tr.run(c, seed=seed, traj=t, shots=3, observables=c.observables)
        assert (out["kraus"] == ref["kraus"][t]).all()
        bad = [s for s in range(3) if out["bits"][s] != ref["bits"][t][s] and ref["sample_margin"][t][s] >= 1e-4]
        assert not bad
        assert np.max(np.abs(out["obs"] - ref["obs"][t])) < 1e-4


def _gpu_gloo_worker(rank, port, q, world, n):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ctx = qtraj.Context(0)
    c = circuit(n, seed=41, noise="ad")
    c.observables += ["I" * (n - 1) + "X", "Y" + "I" * (n - 3) + "ZX"]
    res = []
    for t in range(2):
        tr = D.DistributedTrajectory(D.GpuBackend(ctx, "cuda:0"), D.TorchFabric(), n)
        out = tr.run(c, seed=91, traj=t, shots=3, observables=c.observables)
        res.append({k: np.asarray(v) for k, v in out.items() if k in ("kraus", "bits", "obs", "sample_margin")})
    q.put((rank, res))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_gpu_backend_torch_fabric_two_processes():
    """The production pairing GpuBackend + TorchFabric: two processes (ranks) on one GPU,
    gloo all-to-all with the CUDA states staged through the host (NCCL on multi-GPU
    nodes); both ranks reproduce the oracle's trajectories."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import multiprocessing as mp
    n, world = 14, 2
    mctx = mp.get_context("spawn")
    q = mctx.Queue()
    port = _free_port()
    ps = [mctx.Process(target=_gpu_gloo_worker, args=(r, port, q, world, n)) for r in range(world)]
    for p in ps:
        p.start()
    got = dict(q.get(timeout=300) for _ in range(world))
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    c = circuit(n, seed=41, noise="ad")
    c.observables += ["I" * (n - 1) + "X", "Y" + "I" * (n - 3) + "ZX"]
    ref = oracle.run_trajectories(c, seed=91, traj_count=2, shots=3)
    for rank in range(world):
        for t in range(2):
            out = got[rank][t]
            assert (out["kraus"] == ref["kraus"][t]).all()
            bad = [s for s in range(3) if out["bits"][s] != ref["bits"][t][s] and ref["sample_margin"][t][s] >= 1e-4]
            assert not bad
            assert np.max(np.abs(out["obs"] - ref["obs"][t])) < 1e-4


@pytest.mark.parametrize("world", [2, 4])
def test_overlapped_exchange_defers_and_matches(world):
    """Pending local operations that commute with a swap are applied per received chunk
    (overlapping the exchange); the result equals the flush-everything-first schedule and
    the oracle, and some operations were actually deferred."""
    n = 8
    c = circuit(n, seed=9)
    seed = 55
    ref = oracle.run_trajectories(c, seed=seed, traj_count=1, shots=2)
    outs = {}
    for ov in (False, True):
        tr = D.DistributedTrajectory(NumpyBackend(), D.EmulatedFabric(world), n)
        tr.overlap = ov
        outs[ov] = tr.run(c, seed=seed, traj=0, shots=2, observables=c.observables)
        if ov:
            assert tr.deferred_ops > 0
    check(outs[True], ref, 0)
    assert (outs[True]["kraus"] == outs[False]["kraus"]).all()
    assert (outs[True]["bits"] == outs[False]["bits"]).all()
    assert np.max(np.abs(np.asarray(outs[True]["obs"]) - np.asarray(outs[False]["obs"]))) < 1e-10
