"""GPU parity on the degenerate and boundary cases of the method (through the C
ABI, against the CPU oracle): empty and identity-only circuits, the smallest
registers (tile = the whole state), the tile-size boundary n = 12 / 13,
channels on high qubits (outside the coalesced low qubits), every channel
conventional (s = 0: projective channels), zero
trajectories, zero shots, ragged batches, trajectories addressed far into the
index space, and the maximum shot count per trajectory."""
import numpy as np
import pytest

import oracle
import workloads
from workloads import Channel, Circuit, Gate, channels, gates

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2111_02396_b200 import qtraj  # noqa: E402
from test_gpu_parity import compare, run_both  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2111_02396_b200 import build as B
    B.build()
    return qtraj.Context(0)


@pytest.mark.parametrize("n", [1, 2, 3, 12, 13])
def test_empty_circuit(ctx, n):
    """No operations: every sample is 0...0, <Z_q> = 1, the state is |0...0>."""
    c = Circuit(n_qubits=n, moments=[])
    c.observables = ["Z" * n, "X" + "I" * (n - 1)]
    ref, out, state = run_both(ctx, c, seed=3, T=5, shots=3)
    assert np.all(out["bits"] == 0)
    assert np.allclose(out["obs"][:, 0], 1.0) and np.allclose(out["obs"][:, 1], 0.0, atol=1e-12)
    compare(ref, out, state)


def test_identity_only_circuit(ctx):
    """Identity gates and identity channels are skipped by the planner (no pass)
    and change nothing."""
    n = 6
    c = Circuit(n_qubits=n, moments=[[Gate((q,), np.eye(2)) for q in range(n)],
                                     [Channel((0,), [np.eye(2)])], [Gate((1, 4), np.eye(4))]])
    c.observables = ["Z" * n]
    ref, out, state = run_both(ctx, c, seed=3, T=4, shots=2)
    assert np.all(out["bits"] == 0)
    compare(ref, out, state)


@pytest.mark.parametrize("n", [1, 2, 3, 4])
def test_smallest_registers(ctx, n):
    """Registers smaller than the coalescing run (tile = the whole state)."""
    c = workloads.random_circuit(n, depth=8, seed=40 + n, max_arity=min(2, n), noise="both", p=0.05,
                                 t1_ns=400.0, tphi_ns=700.0, readout=True)
    ref, out, state = run_both(ctx, c, seed=17, T=64, shots=4)
    assert compare(ref, out, state) == 0


@pytest.mark.parametrize("n", [12, 13])
def test_tile_boundary(ctx, n):
    """n = T (one tile per state) and n = T + 1 (two tiles)."""
    c = workloads.random_circuit(n, depth=6, seed=n, noise="both", p=0.03, t1_ns=600.0, tphi_ns=900.0,
                                 readout=True)
    ref, out, state = run_both(ctx, c, seed=5, T=8, shots=2)
    assert compare(ref, out, state) == 0


def test_channels_on_high_qubits(ctx):
    """Conventional channels on the highest qubits (their rho_Q is reduced on a
    tile that excludes the low qubits' partners) and a 2-qubit channel spanning
    a low and a high qubit."""
    n = 15
    rng = np.random.default_rng(2)
    moms = []
    for layer in range(4):
        moms.append([Gate((q,), workloads.haar_unitary(rng, 2)) for q in range(n)])
        moms.append([Gate((0, 14), workloads.haar_unitary(rng, 4)), Gate((7, 13), workloads.haar_unitary(rng, 4))])
        moms.append([Channel((14,), channels.amplitude_damp(0.3)), Channel((13,), channels.phase_damp(0.4))])
        moms.append([Channel((1, 12), [np.kron(a, b) for a in channels.amplitude_damp(0.2)
                                       for b in channels.amplitude_damp(0.25)])])
    c = Circuit(n_qubits=n, moments=moms, observables=["I" * 14 + "Z", "Z" + "I" * 13 + "X"])
    ref, out, state = run_both(ctx, c, seed=8, T=12, shots=2)
    assert (ref["branch"] == 1).any()  # the conventional branch is exercised
    assert compare(ref, out, state) == 0


def test_every_channel_conventional(ctx):
    """Projective pairs {|0><0|, |1><1|} have sigma_min(K_i)^2 = 0, so s = 0 and
    every channel takes Alg. 2's second loop."""
    n = 5
    rng = np.random.default_rng(4)
    moms = []
    for layer in range(3):
        moms.append([Gate((q,), workloads.haar_unitary(rng, 2)) for q in range(n)])
        moms.append([Gate((0, 1), workloads.haar_unitary(rng, 4)), Gate((2, 3), workloads.haar_unitary(rng, 4))])
        moms.append([Channel((q,), channels.measure()) for q in range(n)])
    c = Circuit(n_qubits=n, moments=moms, observables=["ZZZZZ"])
    ref, out, state = run_both(ctx, c, seed=12, T=32, shots=1)
    assert (ref["branch"] == 1).all()
    assert compare(ref, out, state) == 0


def test_zero_trajectories_and_zero_shots(ctx):
    c = workloads.random_circuit(6, depth=4, seed=1, noise="depol", p=0.05)
    plan = qtraj.Plan(qtraj.Circuit.from_description(c), max_fused=4)
    state = torch.zeros(4 << 6, dtype=torch.complex64, device="cuda")
    out = ctx.run_trajectories(plan, state, seed=1, traj_count=0, shots=1, batch=4)
    assert out["bits"].shape == (0, 1)
    ref = oracle.run_trajectories(c, seed=1, traj_count=6, shots=0)
    out = ctx.run_trajectories(plan, state, seed=1, traj_count=6, shots=0, batch=4)
    assert out["bits"].shape == (6, 0)
    assert np.array_equal(out["kraus"], ref["kraus"])


@pytest.mark.parametrize("batch", [1, 5, 7])
def test_ragged_batches_far_indices(ctx, batch):
    """traj_count not a multiple of the batch, trajectories addressed from 2^40:
    records depend on (seed, t) only."""
    c = workloads.random_circuit(9, depth=5, seed=77, noise="both", p=0.04, t1_ns=500.0, tphi_ns=800.0,
                                 readout=True)
    ref, out, _ = run_both(ctx, c, seed=99, T=17, shots=2, batch=batch, traj_begin=(1 << 40) + 3, stride=11)
    assert compare(ref, out, None, check_states=False) == 0


def test_many_shots_per_trajectory(ctx):
    """1024 shots of one final state: identical to the oracle's chain-rule samples."""
    c = workloads.random_circuit(10, depth=6, seed=5, noise="depol", p=0.02, readout=True)
    ref, out, state = run_both(ctx, c, seed=21, T=3, shots=1024)
    assert compare(ref, out, state) == 0


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("n", [7, 14])
def test_three_qubit_conventional_channels(ctx, n, mode):
    """3-qubit non-mixture channels (products of amplitude damping, 8 Kraus
    operators of 8 x 8): rho_Q is 8 x 8 on the device; in the conventional mode
     a 3-qubit depolarizing channel (64 Paulis) is reduced too."""
    rng = np.random.default_rng(n + 10 * mode)
    ad = [np.kron(np.kron(a, b), c) for a in channels.amplitude_damp(0.3) for b in channels.amplitude_damp(0.2)
          for c in channels.amplitude_damp(0.25)]
    P = [np.eye(2), gates.X(), gates.Y(), gates.Z()]
    r = 0.05
    dep3 = [np.sqrt(1 - r) * np.eye(8)] + [np.sqrt(r / 63) * np.kron(np.kron(P[i], P[j]), P[k])
                                          for i in range(4) for j in range(4) for k in range(4) if (i, j, k) != (0, 0, 0)]
    moms = []
    for layer in range(3):
        moms.append([Gate((q,), workloads.haar_unitary(rng, 2)) for q in range(n)])
        moms.append([Gate((0, n - 1), workloads.haar_unitary(rng, 4)), Gate((2, 3), workloads.haar_unitary(rng, 4))])
        moms.append([Channel((1, n - 2, 4), ad), Channel((0, 3, n - 1), dep3)])
    c = Circuit(n_qubits=n, moments=moms, observables=["Z" * n, "X" + "I" * (n - 2) + "Z"])
    ref, out, state = run_both(ctx, c, seed=23, T=16, shots=2, mode=mode)
    assert (ref["branch"] == 1).any()
    assert compare(ref, out, state) == 0


def parity_projectors(q):
    """{P_even, P_odd} on q qubits (parity of the computational-basis bits): a
    projective (s = 0, always conventional) q-qubit channel."""
    d = 2 ** q
    par = np.array([bin(i).count("1") & 1 for i in range(d)])
    return [np.diag((par == 0).astype(float)).astype(np.complex128), np.diag((par == 1).astype(float)).astype(np.complex128)]


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("n", [9, 13])
def test_four_to_six_qubit_conventional_channels(ctx, n, mode):
    """Alg. 2 lines 13-21 for channels on 4 and 6 qubits (P:203-212 hold for any q):
    a 4-qubit product of amplitude damping (16 Kraus operators of 16 x 16, non-mixture)
    and a 6-qubit parity-projective channel (s = 0); rho_Q up to 64 x 64 on the device.
    Both modes; the conventional mode also reduces a 4-qubit depolarizing mixture."""
    rng = np.random.default_rng(n + 100 * mode)
    a1, a2 = channels.amplitude_damp(0.3), channels.amplitude_damp(0.15)
    ad4 = [np.kron(np.kron(np.kron(a, b), c), d) for a in a1 for b in a2 for c in a1 for d in a2]
    proj6 = parity_projectors(6)
    dep1 = channels.depolarize(0.04)
    moms = []
    for layer in range(3):
        moms.append([Gate((q,), workloads.haar_unitary(rng, 2)) for q in range(n)])
        moms.append([Gate((0, n - 1), workloads.haar_unitary(rng, 4)), Gate((2, 3), workloads.haar_unitary(rng, 4))])
        moms.append([Channel((1, n - 2, 4, 5), ad4)])
        moms.append([Channel(tuple(range(n - 6, n))[::-1], proj6), Channel((0,), dep1)])
    c = Circuit(n_qubits=n, moments=moms, observables=["Z" * n, "X" + "I" * (n - 2) + "Z"])
    ref, out, state = run_both(ctx, c, seed=29, T=12, shots=2, mode=mode)
    assert (ref["branch"] == 1).any()
    assert compare(ref, out, state) == 0


@pytest.mark.parametrize("nq", [1, 2, 3, 4, 5, 6])
def test_reduce_rho_up_to_six_qubits(ctx, nq):
    """qt_reduce_rho (distributed-state building block) for 1..6 qubits vs numpy:
    rho_Q[a][b] = sum_rest psi[rest, a] conj(psi[rest, b]), index bit m <-> m-th
    lowest listed qubit."""
    n = 14
    rng = np.random.default_rng(nq)
    psi = rng.standard_normal(2 ** n) + 1j * rng.standard_normal(2 ** n)
    psi = (psi / np.linalg.norm(psi)).astype(np.complex64)
    qs = sorted(int(x) for x in rng.choice(n, size=nq, replace=False))
    st = torch.from_numpy(psi).cuda()
    rho = ctx.reduce_rho(st, qs)
    t = psi.astype(np.complex128).reshape([2] * n)  # axis i <-> qubit n-1-i
    axes = [n - 1 - q for q in qs]
    rest = [a for a in range(n) if a not in axes]
    # matrix index bit m <-> qubits[m] (ascending): the most significant index bit is qs[-1]
    tt = np.transpose(t, rest + axes[::-1]).reshape(-1, 2 ** nq)
    want = tt.T @ tt.conj()
    assert np.allclose(rho, want, atol=1e-6), np.abs(rho - want).max()
