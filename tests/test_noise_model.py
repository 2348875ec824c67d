"""NEXT-2 pins: the calibrated QCS noise-model builder (workloads/noise_model.py)
against the paper's formulas and textbook
identities.  CPU only."""
import numpy as np
import pytest

import oracle
import workloads
from workloads import gates
from workloads import noise_model as nm


def superop(kraus):
    return sum(np.kron(K, K.conj()) for K in kraus)


def apply(kraus, rho):
    return sum(K @ rho @ K.conj().T for K in kraus)


def rand_rho(rng, d):
    a = rng.standard_normal((d, d)) + 1j * rng.standard_normal((d, d))
    r = a @ a.conj().T
    return r / np.trace(r)


@pytest.mark.parametrize("T1,eps,t", [(15e3, 1e-3, 25.0), (30e3, 4e-4, 25.0), (12e3, 2e-3, 32.0)])
def test_eps_inc_is_the_average_error_of_the_decay_channel(T1, eps, t):
    """P:369 inverted for T_phi and fed to the channel of P:397-409 gives back
    eps_inc as the channel's average gate error, up to O(t^2)."""
    Tphi = nm.t_phi_from_eps_inc(eps, t, T1)
    K = nm.decay_channel(t, T1, Tphi)
    assert np.allclose(sum(k.conj().T @ k for k in K), np.eye(2), atol=1e-14)
    got = nm.average_error(K)
    assert abs(got - eps) <= 10 * (t / min(T1, Tphi)) ** 2 + 1e-12, (got, eps)


def test_decay_channel_closed_form_P398():
    rng = np.random.default_rng(1)
    t, T1, Tphi = 40.0, 9e3, 7e3
    T2 = 1 / (1 / (2 * T1) + 1 / Tphi)
    rho = rand_rho(rng, 2)
    e1, e2 = np.exp(-t / T1), np.exp(-t / T2)
    exact = np.array([[1 - rho[1, 1] * e1, rho[0, 1] * e2], [rho[1, 0] * e2, rho[1, 1] * e1]])
    assert np.allclose(apply(nm.decay_channel(t, T1, Tphi), rho), exact, atol=1e-14)


@pytest.mark.parametrize("n", [1, 2])
@pytest.mark.parametrize("eps", [0.0, 0.03, 0.5])
def test_eq1_depolarizing_D_n(n, eps):
    """Eq. 1: D_n[eps](rho) = (1 - eps) rho + eps I / 2^n; trace preserving; equal
    to E_dep of P:432 with r_dep = eps (1 - 1/D^2) (reading A17)."""
    rng = np.random.default_rng(n)
    d = 2 ** n
    K = nm.depolarize_n(eps, n)
    assert len(K) == d * d
    assert np.allclose(sum(k.conj().T @ k for k in K), np.eye(d), atol=1e-13)
    rho = rand_rho(rng, d)
    assert np.allclose(apply(K, rho), (1 - eps) * rho + eps * np.eye(d) / d, atol=1e-13)
    r = eps * (1 - 1 / d ** 2)
    E = workloads.channels.depolarize(r) if n == 1 else workloads.channels.depolarize2(r)
    assert np.allclose(superop(K), superop(E), atol=1e-13)


def test_eq2_uzz_unitary():
    U = nm.u_zz(0.7, 10.0)
    assert np.allclose(U.conj().T @ U, np.eye(4))
    assert np.allclose(np.diag(U)[:3], 1) and np.isclose(np.angle(np.diag(U)[3]), np.angle(np.exp(-2j * np.pi * 7.0)))


def test_r_ent_closed_form_fsim():
    """N4 with no Z phases: 1 - |Tr fSim(dt, dp)|^2 / 16 = 1 - |1 + 2 cos dt + e^{-i dp}|^2 / 16."""
    for dt, dp in [(0.0, 0.0), (0.03, -0.02), (0.1, 0.2)]:
        M = nm.QCSNoiseModel(qubits={0: nm.QubitCal(1e4, 1e-3, 1e-3), 1: nm.QubitCal(1e4, 1e-3, 1e-3)},
                             pairs={(0, 1): nm.PairCal(0.01, dt, dp)})
        exact = 1 - abs(1 + 2 * np.cos(dt) + np.exp(-1j * dp)) ** 2 / 16
        assert np.isclose(M.r_ent((0, 1)), exact, atol=1e-15)


def test_error_budget_P436():
    """The depolarizing remainder makes the noisy two-qubit gate's total Pauli
    error (coherent errors, depolarizing, decay on both qubits) equal the
    calibrated XEB Pauli error, to first order."""
    M = nm.synthetic_calibration(2, [(0, 1)], seed=3)
    p = (0, 1)
    rdep = M.r_dep_2q(p)
    assert rdep > 0
    Uc = M.coherent_2q(p)
    dep = workloads.channels.depolarize2(rdep)
    d0, d1 = M.decay(0, M.t_2q), M.decay(1, M.t_2q)
    deco = [np.kron(a, b) for a in d0 for b in d1]
    total = [D @ E @ Uc for D in deco for E in dep]
    got = nm.pauli_error(total)
    want = M.pairs[p].xeb_pauli
    assert abs(got - want) < 0.05 * want, (got, want)


def test_noisy_circuit_is_valid_and_runs():
    """The builder's circuits pass the library's unitarity / CPTP validation and
    run through the oracle; decay on every qubit after every moment (A16)."""
    from paper_2111_02396_b200 import qtraj
    c = workloads.sycamore_grid_qcs(rows=2, cols=3, cycles=3, config=2, noise=False)
    pairs = sorted({tuple(op.qubits) for op in c.ops() if len(op.qubits) == 2})
    M = nm.synthetic_calibration(c.n_qubits, pairs, seed=5)
    noisy = M.noisy(c)
    qtraj.Circuit.from_description(noisy)  # validation happens on upload
    n_decay = sum(1 for op in noisy.ops() if getattr(op, "name", "") == "decay")
    assert n_decay == c.n_qubits * len(c.moments)
    r = oracle.run_trajectories(noisy, seed=2, traj_count=20)
    assert r["rc"] == 0 and np.all(r["status"] == 0)


def test_coherent_error_z_phases_before_and_after_P424():
    """P:424 puts the Z phase errors before AND after the fSim gate.  The inserted error
    unitary E (applied after the ideal gate G) must give E G = Z_a fSim(th + dth, ph + dph)
    Z_b, checked through the fSim composition law on a gate that does not commute with
    Z x I (sqrt-iSWAP-like fSim(pi/4, 0)), with different phases on the two qubits."""
    th0, ph0 = np.pi / 4, 0.0
    G = workloads.gates.fsim(th0, ph0)
    pc = nm.PairCal(0.01, d_theta=0.03, d_phi=-0.02, z_before=(0.05, -0.04), z_after=(0.02, 0.07))
    M = nm.QCSNoiseModel(qubits={0: nm.QubitCal(1e4, 1e-3, 1e-3), 1: nm.QubitCal(1e4, 1e-3, 1e-3)},
                         pairs={(0, 1): pc})
    E = M.coherent_2q((0, 1), G)
    ez = lambda a: np.diag([np.exp(1j * a), np.exp(-1j * a)])  # e^{i a Z}
    zb = np.kron(ez(0.05), ez(-0.04))
    za = np.kron(ez(0.02), ez(0.07))
    want = za @ workloads.gates.fsim(th0 + 0.03, ph0 - 0.02) @ zb
    got = E @ G
    k = np.vdot(want.ravel(), got.ravel())
    assert abs(abs(k) - 4) < 1e-9, k  # equal up to a global phase
    assert np.allclose(got, want * (k / abs(k)), atol=1e-12)
    # the phases do not commute through G: the old placement (all after G) differs
    assert not np.allclose(M.coherent_2q((0, 1)) @ G, got, atol=1e-6)
