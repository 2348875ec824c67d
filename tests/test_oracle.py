"""Pins for the CPU oracle (oracle/), against things other than itself.

Each test names what fixes the expected value: a published KAT, a closed form
from the paper, a textbook identity, an independent library routine, or a
statistical bound.  CPU only (-m "not gpu").
"""
import os

import numpy as np
import pytest

import oracle
from oracle import dm
import workloads
from workloads import Channel, Circuit, Gate, channels, gates

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# --------------------------------------------------------------------------
# Independent dense application via numpy tensor contraction (not Alg. 1).
# --------------------------------------------------------------------------
def dense_apply(psi, qubits, U):
    n = int(np.log2(psi.size))
    k = len(qubits)
    T = psi.reshape((2,) * n)  # axis a <-> qubit n-1-a
    Ut = U.reshape((2,) * (2 * k))  # (out_0..out_{k-1}, in_0..in_{k-1}); index 0 = MSB = qubits[0]
    axes = [n - 1 - q for q in qubits]
    out = np.tensordot(Ut, T, axes=(list(range(k, 2 * k)), axes))
    out = np.moveaxis(out, list(range(k)), axes)
    return out.reshape(-1)


def rand_state(rng, n):
    v = rng.standard_normal(2 ** n) + 1j * rng.standard_normal(2 ** n)
    return v / np.linalg.norm(v)


# --------------------------------------------------------------------------
# RNG
# --------------------------------------------------------------------------
def test_philox_known_answers():
    rows = [l.split() for l in open(os.path.join(GOLDEN, "philox_kat.txt")) if l.strip() and l[0] != "#"]
    assert len(rows) == 3
    for r in rows:
        v = [int(x, 16) for x in r]
        assert oracle.philox(v[0:4], v[4:6]) == v[6:10]


def _golden_rng():
    """Parse tests/golden/rng_contract.txt (written by tools/gen_rng_golden.py, a third
    Philox implementation): list of (purpose, traj, shot, [(ordinal, half)], values)."""
    path = os.path.join(os.path.dirname(__file__), "golden", "rng_contract.txt")
    rows, n = [], 4
    half_n = (n + 1) // 2
    for ln in open(path):
        if ln.startswith("#") or "->" not in ln:
            continue
        head, vals = ln.split("->")
        vals = vals.split()
        f = head.split()
        kv = dict(x.split("=") for x in f if "=" in x)
        if f[0] == "channel":
            t = int(kv["traj"])
            if "ordinals" in f:
                rows.append((oracle.PURPOSE_CHANNEL, t, [(c, 0) for c in range(3)], [float(v) for v in vals]))
            else:
                rows.append((oracle.PURPOSE_CHANNEL, t, [(int(f[-1]), 0)], [float(v) for v in vals]))
        elif f[0] == "sample":
            t, sh = int(kv["traj"]), int(kv["shot"])
            rows.append((oracle.PURPOSE_SAMPLE, t, [(sh * half_n + l // 2, l % 2) for l in (3, 2, 1, 0)],
                         [float(v) for v in vals]))
        elif f[0] == "readout":
            t, sh = int(kv["traj"]), int(kv["shot"])
            rows.append((oracle.PURPOSE_READOUT, t, [(sh * half_n + q // 2, q % 2) for q in range(4)],
                         [float(v) for v in vals]))
    return rows


def test_rng_contract_golden():
    """Oracle draws = the golden vectors of an independent third Philox (CHANNEL,
    SAMPLE at shots 0..3, READOUT ordinals shot * ceil(n/2) + q/2, a trajectory index
    above 2^32), plus the Random123-style block of (ordinal 0, CHANNEL)."""
    seed = 0x23962112
    assert oracle.philox([0, 1, 0, 0], [seed, 0]) == [0x861C02A8, 0xB8423366, 0x81CEF5B7, 0x5D2ED471]
    rows = _golden_rng()
    assert len(rows) >= 9
    for purpose, t, ords, vals in rows:
        for (o, h), v in zip(ords, vals):
            assert oracle.uniform(seed, o, purpose, t, h) == v, (purpose, t, o, h)


def test_rng_golden_generator_reproduces_file():
    """The committed golden file is exactly what tools/gen_rng_golden.py writes."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "tools", "gen_rng_golden.py"), "--check"])
    assert r.returncode == 0


def test_library_host_rng_matches_golden():
    """The product's own Philox (csrc/philox.hpp, host side of libqtraj, qt_draw) gives
    the same golden draws (the device copy is the same header; parity tests cover it)."""
    from paper_2111_02396_b200 import qtraj
    seed = 0x23962112
    for purpose, t, ords, vals in _golden_rng():
        for (o, h), v in zip(ords, vals):
            assert qtraj.draw(seed, o, purpose, t, h) == v


def test_u53_range_and_resolution():
    assert oracle.u53(0, 0) == 0.0
    top = oracle.u53(0xFFFFFFFF, 0xFFFFFFFF)
    assert top < 1.0 and top == 1.0 - 2.0 ** -53
    assert oracle.u53(0, 1 << 6) == 2.0 ** -53


# --------------------------------------------------------------------------
# Alg. 1
# --------------------------------------------------------------------------
def test_x_on_zero_is_one():
    psi = np.zeros(2, np.complex128); psi[0] = 1
    oracle.apply_gate(psi, [0], gates.X())
    assert np.allclose(psi, [0, 1])


def test_h_involution():
    rng = np.random.default_rng(1)
    psi = rand_state(rng, 4); ref = psi.copy()
    for q in range(4):
        oracle.apply_gate(psi, [q], gates.H()); oracle.apply_gate(psi, [q], gates.H())
    assert np.allclose(psi, ref, atol=1e-14)


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5, 6])
def test_alg1_matches_tensor_contraction(k):
    rng = np.random.default_rng(100 + k)
    n = 8
    for trial in range(4):
        qs = [int(x) for x in rng.choice(n, size=k, replace=False)]
        U = workloads.haar_unitary(rng, 2 ** k)
        psi = rand_state(rng, n)
        ref = dense_apply(psi.copy(), qs, U)
        oracle.apply_gate(psi, qs, U)
        assert np.max(np.abs(psi - ref)) < 1e-13
        assert abs(np.linalg.norm(psi) - 1) < 1e-13  # unitary preserves norm


def test_cnot_unsorted_qubits_kronecker_order():
    # CNOT(3, 1): control = qubit 3 (listed first = matrix MSB).
    psi = np.zeros(16, np.complex128); psi[1 << 3] = 1  # |q3=1>
    oracle.apply_gate(psi, [3, 1], gates.CNOT())
    assert psi[(1 << 3) | (1 << 1)] == 1


def test_ghz_amplitudes_and_mirror():
    n = 6
    psi = np.zeros(2 ** n, np.complex128); psi[0] = 1
    oracle.apply_gate(psi, [0], gates.H())
    for q in range(n - 1):
        oracle.apply_gate(psi, [q, q + 1], gates.CNOT())
    exp = np.zeros(2 ** n); exp[0] = exp[-1] = 1 / np.sqrt(2)
    assert np.allclose(psi, exp, atol=1e-15)
    # mirror circuit C then C^dag returns |0...0>
    rng = np.random.default_rng(7)
    ops = []
    for _ in range(20):
        k = int(rng.integers(1, 4))
        qs = [int(x) for x in rng.choice(n, size=k, replace=False)]
        ops.append((qs, workloads.haar_unitary(rng, 2 ** k)))
    psi = np.zeros(2 ** n, np.complex128); psi[0] = 1
    for qs, U in ops:
        oracle.apply_gate(psi, qs, U)
    for qs, U in reversed(ops):
        oracle.apply_gate(psi, qs, U.conj().T)
    assert abs(psi[0] - 1) < 1e-12 and np.linalg.norm(psi[1:]) < 1e-12


# --------------------------------------------------------------------------
# Lower bounds p-bar = sigma_min(K)^2
# --------------------------------------------------------------------------
def test_sigma_min_closed_forms():
    assert abs(oracle.sigma_min_sq(np.sqrt(0.9) * np.eye(2)) - 0.9) < 1e-12
    g = 0.19
    assert abs(oracle.sigma_min_sq(np.diag([1, np.sqrt(1 - g)])) - 0.81) < 1e-12
    assert oracle.sigma_min_sq(np.array([[0, 0.3], [0, 0]])) < 1e-14


@pytest.mark.parametrize("d", [2, 4, 8, 16, 64])
def test_sigma_min_matches_numpy_svd(d):
    rng = np.random.default_rng(d)
    for _ in range(3):
        K = rng.standard_normal((d, d)) + 1j * rng.standard_normal((d, d))
        ref = np.linalg.svd(K, compute_uv=False).min() ** 2
        assert abs(oracle.sigma_min_sq(K) - ref) < 1e-10 * max(1.0, ref)


def test_unitary_mixture_flags():
    assert oracle.is_unitary_mixture(channels.depolarize(0.01))
    assert oracle.is_unitary_mixture(channels.depolarize2(0.01))
    assert oracle.is_unitary_mixture(channels.bit_flip(0.2))
    assert not oracle.is_unitary_mixture(channels.amplitude_damp(0.1))
    assert not oracle.is_unitary_mixture(channels.decay_dephase(32, 15e3, 30e3))


# --------------------------------------------------------------------------
# Channel inputs vs the paper's closed forms (pins workloads + dm together)
# --------------------------------------------------------------------------
def test_decay_channel_closed_form_P398():
    t, T1, Tphi = 32.0, 15e3, 30e3
    T2 = 1 / (1 / (2 * T1) + 1 / Tphi)
    rng = np.random.default_rng(3)
    a = rand_state(rng, 1)
    rho = np.outer(a, a.conj())
    Ks = channels.decay_dephase(t, T1, Tphi)
    out = sum(K @ rho @ K.conj().T for K in Ks)
    exp = np.array([[1 - rho[1, 1] * np.exp(-t / T1), rho[0, 1] * np.exp(-t / T2)],
                    [rho[1, 0] * np.exp(-t / T2), rho[1, 1] * np.exp(-t / T1)]])
    assert np.allclose(out, exp, atol=1e-15)
    assert np.allclose(sum(K.conj().T @ K for K in Ks), np.eye(2), atol=1e-15)


def test_depolarizing_closed_form_P432():
    p = 0.07
    rng = np.random.default_rng(4)
    a = rand_state(rng, 1); rho = np.outer(a, a.conj())
    out = sum(K @ rho @ K.conj().T for K in channels.depolarize(p))
    assert np.allclose(out, (1 - 4 * p / 3) * rho + (4 * p / 3) * np.eye(2) / 2, atol=1e-15)
    r = 0.05
    b = rand_state(rng, 2); rho2 = np.outer(b, b.conj())
    out2 = sum(K @ rho2 @ K.conj().T for K in channels.depolarize2(r))
    # E_dep with D=4: (1-r) rho + r/15 sum_{mu != 0} P rho P
    P = gates.paulis()
    ref = (1 - r) * rho2 + r / 15 * sum(np.kron(P[a_], P[b_]) @ rho2 @ np.kron(P[a_], P[b_])
                                        for a_ in range(4) for b_ in range(4) if a_ or b_)
    assert np.allclose(out2, ref, atol=1e-15)


def test_dm_embed_matches_tensor_contraction():
    rng = np.random.default_rng(11)
    n = 5
    for k in (1, 2, 3):
        qs = [int(x) for x in rng.choice(n, size=k, replace=False)]
        U = workloads.haar_unitary(rng, 2 ** k)
        psi = rand_state(rng, n)
        assert np.allclose(dm.embed(U, qs, n) @ psi, dense_apply(psi, qs, U), atol=1e-13)


# --------------------------------------------------------------------------
# Config 1 (GHZ-4 + depolarize 0.01): closed forms and golden histogram
# --------------------------------------------------------------------------
def test_ghz4_density_matrix_closed_forms():
    p = 0.01
    c = workloads.ghz4_depolarized(p)
    rho = dm.evolve(c)
    lam = 1 - 4 * p / 3
    # Z(x)4 sees 5 depolarizing factors: qubit 0 twice (H, CX01) and qubits
    # 1,2,3 after the CX that maps their parity ... closed forms:
    assert abs(dm.expectation(rho, "ZZZZ") - lam ** 5) < 1e-12
    assert abs(dm.expectation(rho, "XXXX") - lam ** 7) < 1e-12
    for s in ("ZIII", "IZII", "IIZI", "IIIZ"):
        assert abs(dm.expectation(rho, s)) < 1e-12
    probs = dm.outcome_probabilities(rho)
    assert abs(probs[0] - 0.4803524582) < 1e-9 and abs(probs[15] - 0.4803524582) < 1e-9
    assert abs(sum(probs[1:15]) - 0.0392950835) < 1e-9


def test_density_matrix_readout_path_closed_form_and_trajectories():
    """dm.outcome_probabilities with readout error (reading R14): on |1>|0>
    the recorded distribution is the product of the two confusion rows in closed
    form; on a noisy 3-qubit circuit the oracle's trajectory bitstrings (readout
    applied) follow it (chi-square)."""
    rho = np.zeros((4, 4)); rho[1, 1] = 1.0  # qubit 0 = 1, qubit 1 = 0
    p00, p11 = np.array([0.1, 0.2]), np.array([0.3, 0.05])
    probs = dm.outcome_probabilities(rho, p00, p11)
    # qubit 0 (|1>): recorded 0 with p11[0]; qubit 1 (|0>): recorded 1 with p00[1]
    want = {1: (1 - 0.3) * (1 - 0.2), 0: 0.3 * (1 - 0.2), 3: (1 - 0.3) * 0.2, 2: 0.3 * 0.2}
    for x, w in want.items():
        assert abs(probs[x] - w) < 1e-15
    c = workloads.random_circuit(3, depth=4, seed=9, noise="both", p=0.05, t1_ns=900.0, tphi_ns=1500.0,
                                 readout=True)
    rho = dm.evolve(c)
    pr = dm.outcome_probabilities(rho, c.p00, c.p11)
    R = 40000
    r = oracle.run_trajectories(c, seed=5, traj_count=R, shots=1)
    hist = np.bincount(r["bits"][:, 0].astype(np.int64), minlength=8)
    m = pr > 0
    chi2 = (((hist[m] - R * pr[m]) ** 2) / (R * pr[m])).sum()
    assert chi2 < 7 + 6 * np.sqrt(14)


def test_ghz4_trajectories_golden_histogram_and_stats():
    c = workloads.ghz4_depolarized(0.01)
    seed = workloads.trajectory_seed(1)
    assert seed == 0x23962112
    r = oracle.run_trajectories(c, seed=seed, traj_count=1000, shots=1)
    assert r["rc"] == 0
    assert list(np.bincount(r["kraus"].ravel(), minlength=4)) == [6935, 20, 22, 23]
    assert (r["branch"] == 0).all()  # unitary mixtures: always deferred
    r2 = oracle.run_trajectories(c, seed=seed, traj_count=20000, shots=1)
    rho = dm.evolve(c)
    for k, s in enumerate(c.observables):
        v = r2["obs"][:, k]
        se = max(v.std(ddof=1) / np.sqrt(len(v)), 1e-3)
        assert abs(v.mean() - dm.expectation(rho, s)) < 4 * se + 1e-9


# --------------------------------------------------------------------------
# Alg. 2: trajectory average == density matrix, conventional branch
# --------------------------------------------------------------------------
@pytest.mark.parametrize("noise", ["depol", "decay", "both", "ad"])
def test_trajectory_average_matches_density_matrix(noise):
    n = 4
    c = workloads.random_circuit(n, depth=5, seed=21, noise=noise, p=0.08,
                                 t1_ns=400.0, tphi_ns=800.0, t_ns=32.0)
    c.observables = ["ZIII", "IZII", "IIZI", "IIIZ", "XXII", "IYYI", "ZZZZ"]
    R = 6000
    r = oracle.run_trajectories(c, seed=77, traj_count=R, shots=1)
    assert r["rc"] == 0
    rho = dm.evolve(c)
    for k, s in enumerate(c.observables):
        v = r["obs"][:, k]
        se = v.std(ddof=1) / np.sqrt(R)
        assert abs(v.mean() - dm.expectation(rho, s)) < 4 * se + 1e-9, (s, v.mean(), dm.expectation(rho, s))
    if noise in ("decay", "both", "ad"):
        assert (r["branch"] == 1).any()  # the conventional branch was exercised
    # bitstring histogram vs diag(rho): chi-square with a generous bound
    probs = dm.outcome_probabilities(rho)
    hist = np.bincount(r["bits"].ravel().astype(np.int64), minlength=2 ** n)
    mask = probs * R > 5
    chi2 = (((hist[mask] - R * probs[mask]) ** 2) / (R * probs[mask])).sum()
    assert chi2 < mask.sum() + 6 * np.sqrt(2 * mask.sum())


def test_kraus_selection_frequencies_chi_square():
    # single qubit in a fixed superposition, one amplitude-damping channel:
    # p_0 = 1 - g |b|^2, p_1 = g |b|^2 (p_i = <Psi|K_i^dag K_i|Psi>)
    g = 0.3
    a, b = np.sqrt(0.4), np.sqrt(0.6)
    U = np.array([[a, -b], [b, a]], np.complex128)
    c = Circuit(1, [[Gate((0,), U)], [Channel((0,), channels.amplitude_damp(g))]])
    R = 100000
    r = oracle.run_trajectories(c, seed=5, traj_count=R, shots=0)
    counts = np.bincount(r["kraus"][:, 0], minlength=2)
    p1 = g * b * b
    exp = np.array([1 - p1, p1]) * R
    chi2 = (((counts - exp) ** 2) / exp).sum()
    assert chi2 < 6.63  # chi-square, 1 dof, alpha = 0.01
    # deferral rate == s = pbar_0 = 1 - g (binomial, 4 sigma)
    defer = (r["branch"][:, 0] == 0).mean()
    assert abs(defer - (1 - g)) < 4 * np.sqrt(g * (1 - g) / R)


def test_amplitude_damping_decay_law():
    # P(1) after m applications on |1> = (1 - g)^m
    g, m = 0.1, 6
    mom = [[Gate((0,), gates.X())]] + [[Channel((0,), channels.amplitude_damp(g))] for _ in range(m)]
    c = Circuit(1, mom)
    R = 40000
    r = oracle.run_trajectories(c, seed=9, traj_count=R, shots=1)
    frac1 = (r["bits"][:, 0] == 1).mean()
    p = (1 - g) ** m
    assert abs(frac1 - p) < 4 * np.sqrt(p * (1 - p) / R)


def test_bit_flip_p1_deterministic_and_identity_channel():
    c = Circuit(1, [[Gate((0,), gates.X())], [Channel((0,), channels.bit_flip(1.0))]])
    r = oracle.run_trajectories(c, seed=1, traj_count=200, shots=1)
    assert (r["bits"] == 0).all()
    c2 = Circuit(1, [[Gate((0,), gates.H())], [Channel((0,), [np.eye(2, dtype=complex)])]])
    r2 = oracle.run_trajectories(c2, seed=1, traj_count=50, shots=0)
    assert (r2["kraus"] == 0).all() and (r2["branch"] == 0).all()


def test_deterministic_and_index_addressable():
    c = workloads.random_circuit(5, 6, seed=3, noise="both", p=0.05, t1_ns=500.0, tphi_ns=900.0)
    a = oracle.run_trajectories(c, seed=123, traj_begin=0, traj_count=40, shots=2, threads=1)
    b = oracle.run_trajectories(c, seed=123, traj_begin=10, traj_count=10, shots=2, threads=4)
    assert (a["kraus"][10:20] == b["kraus"]).all() and (a["bits"][10:20] == b["bits"]).all()
    s = oracle.run_trajectories(c, seed=123, traj_begin=1, stride=3, traj_count=5, shots=2)
    assert (a["bits"][1:16:3] == s["bits"]).all()


# --------------------------------------------------------------------------
# Sampler (reading R13) and readout
# --------------------------------------------------------------------------
def test_sampler_h_binomial_and_zero_mass():
    psi = np.array([1, 1], np.complex128) / np.sqrt(2)
    bits, _ = oracle.sample_state(psi, seed=2, traj=0, shots=100000)
    f = bits.mean()
    assert abs(f - 0.5) < 3 * np.sqrt(0.25 / 100000)
    bell = np.zeros(4, np.complex128); bell[0] = bell[3] = 1 / np.sqrt(2)
    bits, _ = oracle.sample_state(bell, seed=2, traj=1, shots=5000)
    assert set(np.unique(bits)) <= {0, 3}
    one = np.zeros(8, np.complex128); one[5] = 1j
    bits, _ = oracle.sample_state(one, seed=2, traj=1, shots=300)
    assert (bits == 5).all()


def test_sampler_distribution_chi_square():
    rng = np.random.default_rng(8)
    n = 5
    psi = rand_state(rng, n)
    S = 200000
    bits, _ = oracle.sample_state(psi, seed=4, traj=3, shots=S)
    hist = np.bincount(bits.astype(np.int64), minlength=2 ** n)
    p = np.abs(psi) ** 2
    chi2 = (((hist - S * p) ** 2) / (S * p)).sum()
    assert chi2 < 31 + 6 * np.sqrt(62)
    # unnormalized input gives the same samples (norm invariance)
    bits2, _ = oracle.sample_state(psi * 3.0, seed=4, traj=3, shots=1000)
    assert (bits2 == bits[:1000]).all()


def _chain_rule_bruteforce(psi, seed, traj, shot, draw):
    """Reading R13 written out by enumeration (independent of oracle.c): masses of the
    two children of the current prefix summed over ALL 2^n probabilities that carry
    the prefix, one fresh uniform per level (SAMPLE ordinal shot * ceil(n/2) + l // 2,
    half l % 2, from the third Philox of tools/gen_rng_golden.py)."""
    n = int(np.log2(psi.size))
    p = np.abs(np.asarray(psi, np.complex128)) ** 2
    idx = np.arange(psi.size)
    half_n = (n + 1) // 2
    prefix = 0
    for l in range(n - 1, -1, -1):
        hi = ((idx >> (l + 1)) << (l + 1)) == prefix  # indices with the chosen bits above l
        m0 = p[hi & (((idx >> l) & 1) == 0)].sum()
        m1 = p[hi & (((idx >> l) & 1) == 1)].sum()
        u = draw(seed, shot * half_n + l // 2, 2, traj, l % 2)
        if m0 == 0.0:
            bit = 1
        elif m1 == 0.0:
            bit = 0
        else:
            bit = 0 if u * (m0 + m1) < m0 else 1
        prefix |= bit << l
    return prefix


def test_sampler_chain_rule_bruteforce_enumeration():
    """Every oracle sample equals the brute-force enumeration of the chain-rule map
    (n <= 10; Porter-Thomas-like, GHZ-like and basis states, i.e. zero-mass branches),
    up to decisions whose margin is below 1e-12 (different fp64 summation orders)."""
    import importlib.util
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("gen_rng_golden", os.path.join(root, "tools", "gen_rng_golden.py"))
    g = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(g)
    rng = np.random.default_rng(12)
    states = []
    for n in (1, 3, 6, 10):
        states.append(rand_state(rng, n))
    ghz = np.zeros(2 ** 7, np.complex128); ghz[0] = ghz[-1] = np.sqrt(0.5)
    basis = np.zeros(2 ** 5, np.complex128); basis[19] = 1.0
    sparse = rand_state(rng, 8) * (rng.random(256) < 0.1)
    states += [ghz, basis, sparse / np.linalg.norm(sparse)]
    checked = 0
    for k, psi in enumerate(states):
        shots = 40
        bits, margins = oracle.sample_state(psi, seed=0x5EED + k, traj=3 + k, shots=shots)
        for sh in range(shots):
            want = _chain_rule_bruteforce(psi, 0x5EED + k, 3 + k, sh, g.draw)
            if margins[sh] >= 1e-12:
                assert int(bits[sh]) == want, (k, sh)
                checked += 1
    assert checked > 250


def test_chain_rule_map_measure_equals_probability():
    """The chain-rule map sends the uniform measure on [0,1)^n to |psi|^2 exactly:
    enumerate a 64-point midpoint grid per level on n = 2 and count outcomes."""
    psi = np.array([0.5, 0.5j, np.sqrt(0.375), -np.sqrt(0.125)], np.complex128)
    p = np.abs(psi) ** 2
    G = 64
    grid = (np.arange(G) + 0.5) / G
    counts = np.zeros(4)
    for u1 in grid:          # level 1 (the MSB) first
        m0, m1 = p[0] + p[1], p[2] + p[3]
        b1 = 0 if u1 * (m0 + m1) < m0 else 1
        for u0 in grid:
            c0, c1 = p[2 * b1], p[2 * b1 + 1]
            b0 = 0 if u0 * (c0 + c1) < c0 else 1
            counts[2 * b1 + b0] += 1
    assert np.allclose(counts / G ** 2, p, atol=1.0 / G)


def test_readout_flips():
    c = Circuit(3, [[Gate((1,), gates.X())]])
    c.p00 = np.array([1.0, 0.0, 0.0]); c.p11 = np.array([0.0, 1.0, 0.0])
    r = oracle.run_trajectories(c, seed=3, traj_count=100, shots=2)
    assert (r["bits_raw"] == 2).all() and (r["bits"] == 1).all()
    c.p00 = np.array([0.0, 0.0, 0.3]); c.p11 = np.zeros(3)
    R = 20000
    r = oracle.run_trajectories(c, seed=3, traj_count=R, shots=1)
    f = ((r["bits"][:, 0] >> 2) & 1).mean()
    assert abs(f - 0.3) < 4 * np.sqrt(0.21 / R)


def test_pauli_expectations_textbook():
    bell = np.zeros(4, np.complex128); bell[0] = bell[3] = 1 / np.sqrt(2)
    assert abs(oracle.pauli_expectation(bell, "XX") - 1) < 1e-14
    assert abs(oracle.pauli_expectation(bell, "YY") + 1) < 1e-14
    assert abs(oracle.pauli_expectation(bell, "ZZ") - 1) < 1e-14
    assert abs(oracle.pauli_expectation(bell, "ZI")) < 1e-14
    plus = np.array([1, 1], np.complex128) / np.sqrt(2)
    assert abs(oracle.pauli_expectation(plus, "Z")) < 1e-14
    rng = np.random.default_rng(12)
    psi = rand_state(rng, 3)
    for s in ("XYZ", "IZX", "YYI"):
        ref = np.vdot(psi, dm.pauli_matrix(s) @ psi).real
        assert abs(oracle.pauli_expectation(psi, s) - ref) < 1e-13


def test_estimator_stderr_scaling():
    # Monte Carlo error ~ 1/sqrt(r)
    c = Circuit(1, [[Gate((0,), gates.H())], [Channel((0,), channels.depolarize(0.3))]])
    c.observables = ["X"]
    v = oracle.run_trajectories(c, seed=31, traj_count=10000, shots=0)["obs"][:, 0]
    se_big = v.std(ddof=1) / np.sqrt(10000)
    se_small = v[:100].std(ddof=1) / np.sqrt(100)
    assert 0.066 <= se_big / se_small <= 0.15


# --------------------------------------------------------------------------
# Conventional trajectory algorithm (NEXT-1): same distribution as Alg. 2
# --------------------------------------------------------------------------
def test_conventional_mode_matches_density_matrix():
    n = 4
    c = workloads.random_circuit(n, depth=5, seed=23, noise="both", p=0.06, t1_ns=500.0, tphi_ns=900.0)
    c.observables = ["ZIII", "IZII", "XXII", "IYYI", "ZZZZ"]
    R = 6000
    r = oracle.run_trajectories(c, seed=78, traj_count=R, shots=1, mode=1)
    assert r["rc"] == 0
    assert (r["branch"] == 1).all()  # every channel computes its probabilities
    rho = dm.evolve(c)
    for k, s in enumerate(c.observables):
        v = r["obs"][:, k]
        se = v.std(ddof=1) / np.sqrt(R)
        assert abs(v.mean() - dm.expectation(rho, s)) < 4 * se + 1e-9


def test_conventional_mode_kraus_frequencies():
    # depolarizing is a unitary mixture: in conventional mode it is sampled by p_i
    c = Circuit(1, [[Gate((0,), gates.H())], [Channel((0,), channels.depolarize(0.3))]])
    R = 60000
    r = oracle.run_trajectories(c, seed=8, traj_count=R, shots=0, mode=1)
    counts = np.bincount(r["kraus"][:, 0], minlength=4)
    exp = np.array([0.7, 0.1, 0.1, 0.1]) * R
    assert (((counts - exp) ** 2) / exp).sum() < 11.34  # chi-square 3 dof, alpha = 0.01


def test_range_parallel_mode_matches_trajectory_parallel_mode():
    """Oracle parallel mode (ii) (the Alg. 1 outer loop split into
    fixed index ranges, for n >= 24) gives exactly the results of mode (i): same Kraus
    choices, margins, samples, observables and states, bit for bit (fixed range-sum
    order in both modes)."""
    c = workloads.random_circuit(13, depth=6, seed=21, noise="both", p=0.03, t1_ns=600.0, tphi_ns=900.0,
                                 readout=True)
    a = oracle.run_trajectories(c, seed=8, traj_count=3, shots=3, want_states=True, threads=3)
    b = oracle.run_trajectories(c, seed=8, traj_count=3, shots=3, want_states=True, threads=5,
                                range_parallel=True)
    assert a["rc"] == 0 and b["rc"] == 0
    assert (a["branch"] == 1).any()
    for k in ("kraus", "branch", "kraus_margin", "bits", "bits_raw", "sample_margin", "obs", "states"):
        assert np.array_equal(a[k], b[k]), k
