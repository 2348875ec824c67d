"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle.

Criteria (BASELINE.json north_star): identical Kraus branch choices and
sampled bitstrings; amplitudes within 1e-5 relative L2 (fp32 state, A11 of
SURVEY 8(c)); observables within 1e-4.  Decision mismatches are accepted only
when the oracle's margin for that decision is below 1e-4 ("explained",
SURVEY 8(c) "Marginal decisions"); any unexplained mismatch fails.
"""
import numpy as np
import pytest

import oracle
import workloads
from workloads import Channel, Circuit, Gate, channels, gates

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2111_02396_b200 import qtraj  # noqa: E402

AMP_TOL = 1e-5
OBS_TOL = 1e-4
MARGIN = 1e-4


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2111_02396_b200 import build as B
    B.build()
    return qtraj.Context(0)


def rel_l2(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def rand_state(rng, n):
    v = rng.standard_normal(2 ** n) + 1j * rng.standard_normal(2 ** n)
    return v / np.linalg.norm(v)


def to_dev(psi):
    return torch.from_numpy(psi.astype(np.complex64)).cuda()


def placements(n, k, rng):
    out = [list(range(k)), list(range(n - k, n))]  # all-low, all-high
    for _ in range(3):
        out.append([int(x) for x in rng.choice(n, size=k, replace=False)])
    out.append(list(range(n - k, n))[::-1])  # unsorted (Kronecker order)
    return out


# ---------------------------------------------------------------------------
# K1: Alg. 1 on single gates, every k and placement class
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("n", [6, 10, 13, 16])
@pytest.mark.parametrize("k", [1, 2, 3, 4, 5, 6])
def test_apply_gate_matches_oracle(ctx, n, k):
    if k > n:
        pytest.skip()
    rng = np.random.default_rng(10 * n + k)
    for qs in placements(n, k, rng):
        U = workloads.haar_unitary(rng, 2 ** k)
        psi = rand_state(rng, n)
        ref = oracle.apply_gate(psi.copy(), qs, U)
        d = to_dev(psi)
        ctx.apply_gate(d, qs, U)
        got = d.cpu().numpy().astype(np.complex128)
        assert rel_l2(got, ref) < AMP_TOL, (qs, rel_l2(got, ref))


def test_all_placements_n10_k2(ctx):
    rng = np.random.default_rng(3)
    n = 10
    for a in range(n):
        for b in range(n):
            if a == b:
                continue
            U = workloads.haar_unitary(rng, 4)
            psi = rand_state(rng, n)
            ref = oracle.apply_gate(psi.copy(), [a, b], U)
            d = to_dev(psi)
            ctx.apply_gate(d, [a, b], U)
            assert rel_l2(d.cpu().numpy().astype(np.complex128), ref) < AMP_TOL


# ---------------------------------------------------------------------------
# Trajectories (Alg. 2) vs the oracle, element by element
# ---------------------------------------------------------------------------
def run_both(ctx, c, seed, T, shots=1, f=4, batch=0, one_gate=False, traj_begin=0, stride=1, tensor_cores=0,
             mode=0):
    ref = oracle.run_trajectories(c, seed=seed, traj_begin=traj_begin, stride=stride, traj_count=T,
                                  shots=shots, want_states=True, mode=mode)
    assert ref["rc"] == 0
    plan = qtraj.Plan(qtraj.Circuit.from_description(c), max_fused=f, one_gate_per_pass=one_gate,
                      tensor_cores=tensor_cores)
    if batch == 0:
        batch = T  # one batch: the state buffer then holds every final state
    state = torch.zeros(batch << c.n_qubits, dtype=torch.complex64, device="cuda")
    out = ctx.run_trajectories(plan, state, seed=seed, traj_count=T, traj_begin=traj_begin,
                               traj_stride=stride, shots=shots, batch=batch, observables=c.observables,
                               mode=mode)
    torch.cuda.synchronize()
    return ref, out, state


def compare(ref, out, state=None, check_states=True):
    # Kraus choices: every channel is recorded (workloads default record=True)
    bad_k = np.argwhere(out["kraus"] != ref["kraus"])
    unexplained = [(t, c) for t, c in bad_k if ref["kraus_margin"][t, c] >= MARGIN]
    assert not unexplained, f"unexplained Kraus mismatches {unexplained[:5]}"
    diverged = set(int(t) for t, _ in bad_k)
    bad_b = np.argwhere(out["bits"] != ref["bits"])
    unexplained = [(t, s) for t, s in bad_b if int(t) not in diverged and ref["sample_margin"][t, s] >= MARGIN]
    assert not unexplained, f"unexplained sample mismatches {unexplained[:5]}"
    keep = [t for t in range(len(ref["bits"])) if t not in diverged]
    if len(ref["obs"][0]):
        assert np.max(np.abs(out["obs"][keep] - ref["obs"][keep])) < OBS_TOL
    if check_states and state is not None:
        T = ref["states"].shape[0]
        psi = state.view(-1, ref["states"].shape[1])[:T].cpu().numpy().astype(np.complex128)
        for t in keep:
            p = psi[t] / np.linalg.norm(psi[t])
            assert rel_l2(p, ref["states"][t]) < AMP_TOL, (t, rel_l2(p, ref["states"][t]))
    return len(diverged)


def test_ghz4_config1(ctx):
    c = workloads.ghz4_depolarized(0.01)
    ref, out, state = run_both(ctx, c, seed=workloads.trajectory_seed(1), T=1000, shots=1)
    assert compare(ref, out, state) == 0
    assert list(np.bincount(out["kraus"].ravel(), minlength=4)) == [6935, 20, 22, 23]
    assert out["stats"]["reductions"] == 0  # unitary mixtures: never conventional


@pytest.mark.parametrize("noise", ["depol", "decay", "both", "ad", "pd"])
@pytest.mark.parametrize("n", [5, 9, 12, 14])
def test_random_noisy_trajectories(ctx, noise, n):
    c = workloads.random_circuit(n, depth=8, seed=100 + n, noise=noise, p=0.03,
                                 t1_ns=600.0, tphi_ns=1100.0, readout=True)
    c.observables = c.observables[:3] + ["X" * min(n, 3) + "I" * (n - min(n, 3)),
                                         "I" * (n - 2) + "YZ"]
    ref, out, state = run_both(ctx, c, seed=7 + n, T=24, shots=3)
    compare(ref, out, state)
    if noise in ("decay", "both", "ad", "pd"):
        assert out["stats"]["reductions"] > 0


@pytest.mark.parametrize("tensor_cores", [-1, 1])
@pytest.mark.parametrize("n", [12, 14])
def test_tensor_core_and_cuda_core_paths(ctx, n, tensor_cores):
    """K1 on tcgen05 (3xTF32, gates padded to 4 qubits) and on FP32 CUDA cores."""
    c = workloads.random_circuit(n, depth=10, seed=300 + n, max_arity=2, noise="both", p=0.03,
                                 t1_ns=700.0, tphi_ns=1200.0, readout=True)
    ref, out, state = run_both(ctx, c, seed=17, T=10, shots=2, tensor_cores=tensor_cores)
    compare(ref, out, state)


@pytest.mark.parametrize("n", [5, 12])
def test_conventional_mode_parity(ctx, n):
    """NEXT-1: the conventional trajectory algorithm -- every channel is
    reduced on the device -- against the oracle's conventional mode."""
    c = workloads.random_circuit(n, depth=5, seed=400 + n, noise="both", p=0.03, t1_ns=900.0, tphi_ns=1500.0,
                                 readout=True)
    ref, out, state = run_both(ctx, c, seed=5, T=6, shots=2, mode=1)
    compare(ref, out, state)
    assert out["stats"]["reductions"] == 6 * c.n_channels


@pytest.mark.parametrize("f", [2, 3, 4, 5, 6])
def test_fuse_sizes_same_results(ctx, f):
    c = workloads.random_circuit(13, depth=10, seed=55, max_arity=2, noise="both", p=0.02,
                                 t1_ns=900.0, tphi_ns=1500.0)
    ref, out, state = run_both(ctx, c, seed=3, T=8, shots=2, f=f)
    compare(ref, out, state)


def test_one_gate_per_pass_mode(ctx):
    c = workloads.random_circuit(14, depth=6, seed=8, noise="decay", t1_ns=700.0, tphi_ns=1200.0)
    ref, out, state = run_both(ctx, c, seed=4, T=6, shots=1, one_gate=True)
    compare(ref, out, state)


def test_batching_and_trajectory_addressing(ctx):
    c = workloads.random_circuit(12, depth=6, seed=9, noise="both", p=0.04, t1_ns=500.0, tphi_ns=900.0,
                                 readout=True)
    ref, out, _ = run_both(ctx, c, seed=11, T=20, shots=2, batch=3, traj_begin=5, stride=3)
    compare(ref, out, None, check_states=False)


def test_three_qubit_gates_and_mixed_arity(ctx):
    c = workloads.random_circuit(13, depth=6, seed=21, max_arity=3, noise="depol", p=0.05)
    ref, out, state = run_both(ctx, c, seed=2, T=6, shots=1, f=4)
    compare(ref, out, state)


def test_sample_and_expectation_standalone(ctx):
    rng = np.random.default_rng(5)
    for n in (4, 12, 15):
        psi = rand_state(rng, n)
        d = to_dev(psi)
        got = ctx.sample_bitstrings(d, seed=9, traj=2, shots=64)
        ref, mg = oracle.sample_state(psi.astype(np.complex64).astype(np.complex128), seed=9, traj=2, shots=64)
        bad = [(i) for i in np.flatnonzero(got != ref) if mg[i] >= MARGIN]
        assert not bad
        obs = ["Z" + "I" * (n - 1), "X" * n, "I" * (n - 2) + "XY", "Y" + "Z" * (n - 1)]
        ev = ctx.expectation_value(d, obs)
        for k, s in enumerate(obs):
            assert abs(ev[k] - oracle.pauli_expectation(psi, s)) < OBS_TOL


def test_sample_block_sum_heap(ctx):
    """Registers of >= 2^10 tiles sample their global levels through the block-sum heap
    (kernels.cu blocksum_heap_kernel): bitstrings identical to the oracle's chain rule,
    standalone (n = 24) and at the end of trajectories (n = 23, 4 shots each)."""
    rng = np.random.default_rng(8)
    n = 24
    psi = rand_state(rng, n)
    got = ctx.sample_bitstrings(to_dev(psi), seed=4, traj=7, shots=256)
    ref, mg = oracle.sample_state(psi.astype(np.complex64).astype(np.complex128), seed=4, traj=7, shots=256)
    assert not [i for i in np.flatnonzero(got != ref) if mg[i] >= MARGIN]
    c = workloads.random_circuit(23, depth=3, seed=31, max_arity=2, noise="depol", p=0.02)
    ref, out, state = run_both(ctx, c, seed=3, T=2, shots=4, f=4)
    compare(ref, out, state)


def test_read_only_final_pass_repeatable(ctx):
    """n = 23 (1024 tiles of 2^13): the read-only final pass (block sums + observables)
    runs items whose tile loads land while the other warpgroup works.  Completion of those
    loads once raced (partial tiles on ~1 item in 4000, slot 0's observables off by up to
    3e-3): six repeated 4-trajectory runs must all match the oracle."""
    n, T = 23, 4
    c = workloads.random_circuit(n, depth=3, seed=31, max_arity=2, noise="depol", p=0.02)
    ref = oracle.run_trajectories(c, seed=3, traj_count=T, shots=1)
    plan = qtraj.Plan(qtraj.Circuit.from_description(c), max_fused=4)
    for _ in range(6):
        state = torch.zeros(T << n, dtype=torch.complex64, device="cuda")
        out = ctx.run_trajectories(plan, state, seed=3, traj_count=T, shots=1, observables=c.observables, batch=T)
        torch.cuda.synchronize()
        assert np.max(np.abs(out["obs"] - ref["obs"])) < OBS_TOL


def test_config2_sample_of_trajectories(ctx):
    """C2 (20 q Sycamore-style + QCS-like noise) on 4 trajectory indices spread
    over [0, 1e4): the launch configuration bench.py times (f=4, tiles)."""
    c = workloads.sycamore_grid_qcs(config=2)
    seed = workloads.trajectory_seed(2)
    ref = oracle.run_trajectories(c, seed=seed, traj_begin=17, stride=2477, traj_count=4, shots=1,
                                  want_states=True)
    plan = qtraj.Plan(qtraj.Circuit.from_description(c), max_fused=4)
    state = torch.zeros(4 << 20, dtype=torch.complex64, device="cuda")
    out = ctx.run_trajectories(plan, state, seed=seed, traj_count=4, traj_begin=17, traj_stride=2477,
                               shots=1, observables=c.observables)
    torch.cuda.synchronize()
    compare(ref, out, state)


def test_config2_full_batch_launch(ctx):
    """C2 in bench.py's launch configuration: one full batch of 384 slots (3 GiB of
    state, byte offsets past 2^31), trajectories t = 17 + 26 j; slots 0, 127, 255
    and 383 are checked against the oracle one by one, and every slot's records
    are a valid Kraus index with a normalised state."""
    c = workloads.sycamore_grid_qcs(config=2)
    seed = workloads.trajectory_seed(2)
    B = 384
    plan = qtraj.Plan(qtraj.Circuit.from_description(c), max_fused=4)
    state = torch.zeros(B << 20, dtype=torch.complex64, device="cuda")
    out = ctx.run_trajectories(plan, state, seed=seed, traj_count=B, traj_begin=17, traj_stride=26, batch=B,
                               shots=1, observables=c.observables)
    torch.cuda.synchronize()
    kmax = np.array([len(op.kraus) for op in c.ops() if hasattr(op, "kraus")])
    assert np.all((out["kraus"] >= 0) & (out["kraus"] < kmax[None, :]))
    norms = torch.linalg.vector_norm(state.view(B, -1), dim=1).cpu().numpy()
    assert np.all(np.isfinite(norms)) and np.all(norms > 0)
    for j in (0, 127, 255, 383):
        ref = oracle.run_trajectories(c, seed=seed, traj_begin=17 + 26 * j, traj_count=1, shots=1,
                                      want_states=True)
        sub = {"kraus": out["kraus"][j:j + 1], "bits": out["bits"][j:j + 1], "obs": out["obs"][j:j + 1]}
        compare(ref, sub, state.view(B, -1)[j], check_states=True)


# ---------------------------------------------------------------------------
# K1 f16 tensor-core runs: the tile scale (DESIGN R11) under norm growth,
# tiny amplitudes and all-zero tiles; chains of 4-qubit operators applied with
# qt_apply_plan vs the oracle's Alg. 1 one operator at a time.
# ---------------------------------------------------------------------------
def _chain(rng, n_ops, low=12, k=4):
    ops = []
    prev = None
    for _ in range(n_ops):
        while True:
            qs = sorted(int(x) for x in rng.choice(low, k, replace=False))
            if qs != prev:
                break
        prev = qs
        ops.append((qs, workloads.haar_unitary(rng, 2 ** k)))
    return ops


def _apply_chain(ctx, psi, ops, n, f=4):
    c = qtraj.Circuit(n)
    for m, (qs, M) in enumerate(ops):
        c.add_matrix(m, qs, M)
    plan = qtraj.Plan(c, max_fused=f, tensor_cores=1)
    d = to_dev(psi)
    ctx.apply_plan(plan, d)
    ref = psi.copy()
    for qs, M in ops:
        ref = oracle.apply_gate(ref, qs, M)
    return d.cpu().numpy().astype(np.complex128), ref


@pytest.mark.parametrize("scale", [1.0, 3.0, 40.0])
def test_tc_run_norm_growth(ctx, scale):
    """Non-unitary operators (qt_add_matrix, as distributed mode's 1/sqrt(p)
    picks) grow the tile norm by up to scale^4: runs split and widen their
    scale headroom (2^shift) instead of overflowing the f16 operands."""
    n = 14
    rng = np.random.default_rng(7)
    ops = _chain(rng, 12)
    ops = [(qs, M * (scale if i % 3 == 0 else 1.0)) for i, (qs, M) in enumerate(ops)]
    got, ref = _apply_chain(ctx, rand_state(rng, n), ops, n)
    assert np.all(np.isfinite(got))
    assert rel_l2(got, ref) < AMP_TOL, rel_l2(got, ref)


@pytest.mark.parametrize("amp", [1e-25, 1e-3, 1e3])
def test_tc_run_amplitude_range(ctx, amp):
    """The power-of-two tile scale keeps 22 significant bits whatever the
    amplitude magnitude (unnormalised states, tiny per-rank norms)."""
    n = 14
    rng = np.random.default_rng(11)
    got, ref = _apply_chain(ctx, rand_state(rng, n) * amp, _chain(rng, 10), n)
    assert rel_l2(got, ref) < AMP_TOL, rel_l2(got, ref)


@pytest.mark.parametrize("k", [5, 6])
@pytest.mark.parametrize("amp", [1e-25, 1.0, 1e3])
def test_tc_wide_gates_amplitude_range(ctx, k, amp):
    """5- and 6-qubit tensor-core gates (f16 hi/lo GEMMs, tile scale per gate):
    chains of Haar k-qubit operators on high and low qubits, any amplitude scale."""
    n = 15
    rng = np.random.default_rng(20 + k)
    ops = _chain(rng, 5, low=n, k=k)
    got, ref = _apply_chain(ctx, rand_state(rng, n) * amp, ops, n, f=k)
    assert rel_l2(got, ref) < AMP_TOL, rel_l2(got, ref)


@pytest.mark.parametrize("k", [5, 6])
def test_tc_wide_gates_norm_growth(ctx, k):
    """Non-unitary k-qubit operators (norm up to 40) on the wide tensor-core path."""
    n = 14
    rng = np.random.default_rng(30 + k)
    ops = [(qs, M * (40.0 if i % 2 == 0 else 1.0)) for i, (qs, M) in enumerate(_chain(rng, 4, low=n, k=k))]
    got, ref = _apply_chain(ctx, rand_state(rng, n), ops, n, f=k)
    assert np.all(np.isfinite(got))
    assert rel_l2(got, ref) < AMP_TOL, rel_l2(got, ref)


@pytest.mark.parametrize("f", [5, 6])
@pytest.mark.parametrize("tensor_cores", [-1, 1])
def test_wide_fused_gates_trajectories(ctx, f, tensor_cores):
    """Noisy trajectories with fused gates of up to f = 5 / 6 qubits (3-qubit
    operators included) on tcgen05 (f16 hi/lo, padded to f qubits) and on CUDA
    cores: identical Kraus choices and samples, states within 1e-5."""
    c = workloads.random_circuit(14, depth=8, seed=500 + f, max_arity=3, noise="both", p=0.03,
                                 t1_ns=800.0, tphi_ns=1400.0, readout=True)
    ref, out, state = run_both(ctx, c, seed=19, T=8, shots=2, f=f, tensor_cores=tensor_cores)
    compare(ref, out, state)


@pytest.mark.parametrize("n", [6, 8, 11])
@pytest.mark.parametrize("f", [5, 6])
def test_wide_gates_small_registers(ctx, n, f):
    """5- and 6-qubit operations on registers smaller than a tile (whole-state
    tiles with 2^5 / 2^6 amplitudes per thread)."""
    c = workloads.random_circuit(n, depth=5, seed=3 * n + f, max_arity=f, noise="both", p=0.03, t1_ns=600.0,
                                 tphi_ns=900.0, readout=True)
    rng = np.random.default_rng(n + f)
    wide = tuple(int(q) for q in rng.permutation(n)[:f])  # unsorted: Kronecker order exercised
    c.moments.insert(2, [Gate(wide, workloads.haar_unitary(rng, 2 ** f))])
    ref, out, state = run_both(ctx, c, seed=19, T=8, shots=2, f=f)
    assert compare(ref, out, state) == 0


def test_tc_run_zero_tiles(ctx):
    """Tiles that are entirely zero (max component 0) stay exactly zero."""
    n = 14
    rng = np.random.default_rng(12)
    psi = rand_state(rng, n)
    psi[np.arange(2 ** n) & (1 << 13) != 0] = 0  # qubit 13 (outside every tile of the chain) in |0>
    psi /= np.linalg.norm(psi)
    got, ref = _apply_chain(ctx, psi, _chain(rng, 8), n)
    assert np.all(got[np.arange(2 ** n) & (1 << 13) != 0] == 0)
    assert rel_l2(got, ref) < AMP_TOL, rel_l2(got, ref)


# ---------------------------------------------------------------------------
# NEXT-3: mid-circuit measurements (keyed projector channels, always the
# conventional branch) -- identical outcomes, samples and states
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("n", [5, 14])
def test_mid_circuit_measurement_parity(ctx, n):
    rng = np.random.default_rng(40 + n)
    c = workloads.random_circuit(n, depth=6, seed=40 + n, max_arity=2, noise="depol")
    moms = []
    for i, m in enumerate(c.moments):
        moms.append(m)
        if i % 3 == 2:
            moms.append([workloads.measurement(int(q)) for q in rng.choice(n, 2, replace=False)])
    c.moments = moms
    ref, out, state = run_both(ctx, c, seed=123, T=24, shots=2)
    assert compare(ref, out, state) == 0


# ---------------------------------------------------------------------------
# C4 (32 qubits on one GPU, SURVEY 8(c) pins): no oracle state fits, so a
# mirror circuit (C then C^dagger) must return |0...0>
# ---------------------------------------------------------------------------
def test_mirror_circuit_32_qubits(ctx):
    n = 32
    if torch.cuda.get_device_properties(0).total_memory < (40 << 30):
        pytest.skip("needs a 32 GiB state")
    rng = np.random.default_rng(32)
    fwd = []
    for layer in range(6):
        qs = rng.permutation(n)
        for i in range(0, n - 1, 2):
            fwd.append(((int(qs[i]), int(qs[i + 1])), workloads.haar_unitary(rng, 4)))
    c = qtraj.Circuit(n)
    m = 0
    for qs, U in fwd:
        c.add_gate(m, list(qs), U)
        m += 1
    for qs, U in reversed(fwd):
        c.add_gate(m, list(qs), U.conj().T)
        m += 1
    plan = qtraj.Plan(c, max_fused=4)
    state = torch.zeros(1 << n, dtype=torch.complex64, device="cuda")
    out = ctx.run_trajectories(plan, state, seed=1, traj_count=1, batch=1, shots=8, observables=["Z" * 4])
    torch.cuda.synchronize()
    a0 = state[0].item()
    assert abs(abs(a0) - 1.0) < 1e-4, a0
    assert np.all(out["bits"] == 0)
    del state
    torch.cuda.empty_cache()


def test_calibrated_qcs_noise_model_parity(ctx):
    """NEXT-2: a circuit with the calibrated approximate QCS noise model
    (workloads/noise_model.py: Z-phase + fSim coherent errors, depolarizing
    remainder of the XEB budget, decay from T1 / eps_inc, readout)."""
    from workloads import noise_model as nm
    c = workloads.sycamore_grid_qcs(rows=3, cols=4, cycles=4, config=2, noise=False)
    pairs = sorted({tuple(op.qubits) for op in c.ops() if len(op.qubits) == 2})
    noisy = nm.synthetic_calibration(c.n_qubits, pairs, seed=8).noisy(c)
    noisy.observables = ["Z" + "I" * (c.n_qubits - 1), "I" * (c.n_qubits - 1) + "Z"]
    ref, out, state = run_both(ctx, noisy, seed=77, T=32)
    assert compare(ref, out, state) == 0


# ---------------------------------------------------------------------------
# Experimental TMA-pipelined kernel on 11-qubit tiles (tile_pass_v3.cu, tile_bits = 11)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("case", ["unitary", "depol", "damping", "c2"])
def test_tile_pass_v3_matches_oracle(ctx, case):
    if case == "unitary":
        c, T = workloads.random_circuit(14, depth=6, seed=3, noise="none"), 4
    elif case == "depol":
        c, T = workloads.random_circuit(16, depth=6, seed=4, noise="depol", p=0.02), 6
    elif case == "damping":
        c, T = workloads.random_circuit(14, depth=6, seed=5, noise="both", p=0.02, t1_ns=800.0, tphi_ns=1500.0,
                                        readout=True), 8
    else:
        c, T = workloads.sycamore_grid_qcs(config=2), 8
    ref = oracle.run_trajectories(c, seed=7, traj_count=T, shots=2, want_states=True)
    plan = qtraj.Plan(qtraj.Circuit.from_description(c), max_fused=4, tile_bits=11)
    assert plan.info(7, 0)["kernel"] == 11
    state = torch.zeros(T << c.n_qubits, dtype=torch.complex64, device="cuda")
    out = ctx.run_trajectories(plan, state, seed=7, traj_count=T, shots=2, batch=T, observables=c.observables)
    torch.cuda.synchronize()
    compare(ref, out, state)


def test_tile_pass_v3_measurement_and_readout(ctx):
    """tile_bits = 11 with mid-circuit measurements (projector channels, always the
    conventional branch: rho_Q epilogue + device choice) and readout error."""
    n, T = 14, 12
    rng = np.random.default_rng(41)
    c = workloads.random_circuit(n, depth=6, seed=41, max_arity=2, noise="depol", readout=True)
    moms = []
    for i, m in enumerate(c.moments):
        moms.append(m)
        if i % 3 == 2:
            moms.append([workloads.measurement(int(q)) for q in rng.choice(n, 2, replace=False)])
    c.moments = moms
    ref = oracle.run_trajectories(c, seed=9, traj_count=T, shots=3, want_states=True)
    plan = qtraj.Plan(qtraj.Circuit.from_description(c), max_fused=4, tile_bits=11)
    state = torch.zeros(T << n, dtype=torch.complex64, device="cuda")
    out = ctx.run_trajectories(plan, state, seed=9, traj_count=T, shots=3, batch=T, observables=c.observables)
    torch.cuda.synchronize()
    assert compare(ref, out, state) == 0
