"""NEXT-3: mid-circuit measurement as keyed projector channels (SURVEY
8(c) A12) and the circuit file format.  CPU pins of the oracle's behaviour:
collapse, perfect correlations, the always-conventional branch (sigma_min of a
projector is 0, so s = 0), agreement with the density-matrix evolution
(measurement = dephasing on average), and JSON round trips."""
import numpy as np

import oracle
from oracle import dm
import workloads
from workloads import Circuit, Gate, gates

H = gates.H()
CX = gates.CNOT()  # control = first listed qubit (Kronecker order)


def binom_ok(k, n, p, z=5.0):
    return abs(k - n * p) <= z * np.sqrt(n * p * (1 - p)) + 1


def test_measurement_collapses_the_state():
    """H M H on |0>: the record is uniform and, after the collapse, the final
    sample is uniform and independent of it; without M the final bit is 0."""
    T = 4000
    c = Circuit(n_qubits=1, moments=[[Gate((0,), H)], [workloads.measurement(0)], [Gate((0,), H)]])
    r = oracle.run_trajectories(c, seed=5, traj_count=T)
    assert r["rc"] == 0
    rec = r["kraus"][:, 0]
    assert np.all(r["branch"][:, 0] == 1)  # always the conventional branch (s = 0)
    assert binom_ok(int(rec.sum()), T, 0.5)
    bits = r["bits"][:, 0].astype(np.int64)
    assert binom_ok(int(bits.sum()), T, 0.5)
    assert binom_ok(int((bits == rec).sum()), T, 0.5)
    c0 = Circuit(n_qubits=1, moments=[[Gate((0,), H)], [Gate((0,), H)]])
    assert np.all(oracle.run_trajectories(c0, seed=5, traj_count=200)["bits"] == 0)


def test_bell_measurements_are_correlated():
    """Bell pair: the two mid-circuit outcomes agree in every trajectory, the
    final sample repeats them, and each outcome is uniform."""
    T = 2000
    c = Circuit(n_qubits=2, moments=[[Gate((0,), H)], [Gate((0, 1), CX)],
                                     [workloads.measurement(0)], [workloads.measurement(1)]])
    r = oracle.run_trajectories(c, seed=9, traj_count=T)
    a, b = r["kraus"][:, 0], r["kraus"][:, 1]
    assert np.all(a == b)
    bits = r["bits"][:, 0].astype(np.int64)
    assert np.all(bits == a * 3)
    assert binom_ok(int(a.sum()), T, 0.5)


def test_measurement_trajectories_match_density_matrix():
    """Averaged over trajectories, a measurement is complete dephasing: <Z_i>
    and the outcome distribution of a noisy 3-qubit circuit with mid-circuit
    measurements match the density-matrix oracle within 4 sigma."""
    rng = np.random.default_rng(3)
    n = 3
    moms = []
    for layer in range(4):
        moms.append([Gate((q,), workloads.haar_unitary(rng, 2)) for q in range(n)])
        moms.append([Gate((0, 1), workloads.haar_unitary(rng, 4))])
        moms.append([workloads.Channel((q,), workloads.channels.depolarize(0.02)) for q in range(n)])
        if layer % 2 == 0:
            moms.append([workloads.measurement(layer % n)])
    c = Circuit(n_qubits=n, moments=moms, observables=["ZII", "IZI", "IIZ"])
    rho = dm.evolve(c)
    T = 6000
    r = oracle.run_trajectories(c, seed=21, traj_count=T)
    for i, s in enumerate(c.observables):
        exact = dm.expectation(rho, s)
        m = r["obs"][:, i]
        assert abs(m.mean() - exact) <= 4 * m.std() / np.sqrt(T) + 1e-3, (s, m.mean(), exact)
    probs = dm.outcome_probabilities(rho)
    hist = np.bincount(r["bits"][:, 0].astype(np.int64), minlength=2 ** n)
    for k in range(2 ** n):
        assert binom_ok(int(hist[k]), T, float(probs[k]))


def test_circuit_json_round_trip():
    """The circuit file format reproduces the circuit exactly (flattened arrays
    and oracle results identical)."""
    c = workloads.sycamore_grid_qcs(rows=2, cols=3, cycles=3, config=2)
    c.moments.append([workloads.measurement(q) for q in range(3)])
    c2 = workloads.circuit_from_json(workloads.circuit_to_json(c))
    f1, f2 = workloads.flatten(c), workloads.flatten(c2)
    for k in f1:
        assert np.array_equal(np.asarray(f1[k]), np.asarray(f2[k])), k
    assert np.array_equal(c.p00, c2.p00) and np.array_equal(c.p11, c2.p11)
    assert c.observables == c2.observables
    r1 = oracle.run_trajectories(c, seed=4, traj_count=50)
    r2 = oracle.run_trajectories(c2, seed=4, traj_count=50)
    assert np.array_equal(r1["kraus"], r2["kraus"]) and np.array_equal(r1["bits"], r2["bits"])
