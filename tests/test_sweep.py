"""NEXT-4: parameter sweeps ("simulating parametrized circuits for many
different choices of parameters ... embarrassingly parallelizable").  A sweep
gate carries one unitary per parameter set; trajectory t of a run applies set
t mod n_sets (include/qtraj.h qt_add_gate_sweep).  Sweep gates draw no random
numbers, so set s of a sweep is, trajectory by trajectory, the plain circuit of
set s (workloads.resolve_set) at trajectories t = s (mod n_sets).

CPU: the oracle on resolved circuits against the QAOA p = 1 closed form
(Wang, Hadfield, Jiang, Rieffel, PRA 97, 022304 (2018), Thm. 1, triangle-free
graphs; our cost unitary exp(-i gamma ZZ) is theirs at gamma_W = -2 gamma), the
host planner of the sweep against the planner of each resolved circuit, ABI
validation, the circuit file format.  GPU: parity of one sweep launch with the
oracle run on every resolved circuit."""
import numpy as np
import pytest

import oracle
import workloads
from oracle import dm
from paper_2111_02396_b200 import build as B
from paper_2111_02396_b200 import qtraj


@pytest.fixture(scope="module", autouse=True)
def built():
    B.build()
    qtraj.lib()


def _angles(S, layers, seed):
    rng = np.random.default_rng(seed)
    return rng.uniform(0, np.pi, (S, layers)).tolist(), rng.uniform(0, np.pi / 2, (S, layers)).tolist()


def _edges_and_degrees(rows, cols):
    pat = workloads._grid_couplers(rows, cols)
    edges = [e for k in "ABCD" for e in pat[k]]
    deg = np.zeros(rows * cols, int)
    for a, b in edges:
        deg[a] += 1
        deg[b] += 1
    return edges, deg


@pytest.mark.parametrize("rows,cols", [(2, 3), (3, 3)])
def test_qaoa_p1_closed_form(rows, cols):
    """Noiseless p = 1 QAOA on a grid (triangle-free): <Z_u Z_v> =
    1/2 sin(4 beta) sin(2 gamma) (cos^d(2 gamma) + cos^e(2 gamma)), d = deg(u) - 1,
    e = deg(v) - 1, for every parameter set of the sweep."""
    gam, bet = _angles(5, 1, seed=11)
    c = workloads.qaoa_grid_sweep(rows, cols, 1, gam, bet, depol=0.0)
    assert workloads.n_sets(c) == 5
    edges, deg = _edges_and_degrees(rows, cols)
    for s in range(5):
        r = oracle.run_trajectories(workloads.resolve_set(c, s), seed=3, traj_begin=s, traj_count=1)
        g, b = gam[s][0], bet[s][0]
        for (u, v), val in zip(edges, r["obs"][0]):
            cf = 0.5 * np.sin(4 * b) * np.sin(2 * g) * (np.cos(2 * g) ** (deg[u] - 1) + np.cos(2 * g) ** (deg[v] - 1))
            assert abs(val - cf) < 1e-12


def test_noisy_sweep_trajectories_match_density_matrix():
    """Noisy sweep (depolarizing + amplitude damping): per parameter set, the
    trajectory mean of every <Z_u Z_v> matches the density-matrix oracle of the
    resolved circuit within 4 sigma."""
    S, T = 3, 1500
    gam, bet = _angles(S, 2, seed=5)
    c = workloads.qaoa_grid_sweep(2, 2, 2, gam, bet, depol=0.02, amp_damp=0.05)
    for s in range(S):
        cs = workloads.resolve_set(c, s)
        r = oracle.run_trajectories(cs, seed=21, traj_begin=s, stride=S, traj_count=T)
        assert r["rc"] == 0
        rho = dm.evolve(cs)
        for j, pstr in enumerate(cs.observables):
            exact = dm.expectation(rho, pstr)
            mean, sd = r["obs"][:, j].mean(), r["obs"][:, j].std(ddof=1)
            assert abs(mean - exact) <= 4 * sd / np.sqrt(T) + 1e-12, (s, pstr, mean, exact)


def test_planner_sweep_equals_resolved_circuits():
    """Host planning of trajectory t of the sweep = planning of trajectory t of
    the circuit of set t mod S (same passes, fused gates, deferrals)."""
    S = 4
    gam, bet = _angles(S, 2, seed=2)
    c = workloads.qaoa_grid_sweep(3, 4, 2, gam, bet, depol=0.01, amp_damp=0.02)
    qc = qtraj.Circuit.from_description(c)
    assert qc.num_sets == S
    plan = qtraj.Plan(qc, max_fused=4)
    plans = [qtraj.Plan(qtraj.Circuit.from_description(workloads.resolve_set(c, s)), max_fused=4) for s in range(S)]
    for t in range(40):
        assert plan.info(17, t) == plans[t % S].info(17, t)


def test_sweep_validation():
    c = qtraj.Circuit(3)
    U = [workloads.gates.rz(0.1), workloads.gates.rz(0.2)]
    c.add_gate_sweep(0, [0], U)
    assert c.num_sets == 2
    with pytest.raises(qtraj.QtError):  # different number of sets
        c.add_gate_sweep(0, [1], U + [workloads.gates.rz(0.3)])
    with pytest.raises(qtraj.QtError):  # a non-unitary set
        c.add_gate_sweep(1, [1], [workloads.gates.rz(0.1), 2 * np.eye(2)])
    with pytest.raises(qtraj.QtError):  # qubit reused in a moment
        c.add_gate_sweep(0, [0], U)
    assert qtraj.Circuit(2).num_sets == 1


def test_sweep_json_round_trip():
    gam, bet = _angles(3, 1, seed=9)
    c = workloads.qaoa_grid_sweep(2, 3, 1, gam, bet)
    c2 = workloads.circuit_from_json(workloads.circuit_to_json(c))
    assert workloads.n_sets(c2) == 3
    for s in range(3):
        f1 = workloads.flatten(workloads.resolve_set(c, s))
        f2 = workloads.flatten(workloads.resolve_set(c2, s))
        for k in f1:
            assert np.array_equal(np.asarray(f1[k]), np.asarray(f2[k])), k


@pytest.mark.gpu
@pytest.mark.parametrize("rows,cols,f", [(2, 3, 4), (3, 4, 4), (3, 5, 6)])
def test_sweep_gpu_parity(rows, cols, f):
    """One launch runs every parameter set: each trajectory equals the oracle's
    trajectory of its resolved circuit (Kraus choices and bitstrings identical,
    observables within 1e-4, states within 1e-5 relative L2)."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    S, per = 4, 6
    T = S * per
    gam, bet = _angles(S, 3, seed=rows * cols)
    c = workloads.qaoa_grid_sweep(rows, cols, 3, gam, bet, depol=0.01, amp_damp=0.03)
    ctx = qtraj.Context(0)
    plan = qtraj.Plan(qtraj.Circuit.from_description(c), max_fused=f)
    n = c.n_qubits
    state = torch.zeros(T << n, dtype=torch.complex64, device="cuda")
    out = ctx.run_trajectories(plan, state, seed=31, traj_count=T, shots=2, batch=T, observables=c.observables)
    torch.cuda.synchronize()
    psi = state.view(T, -1).cpu().numpy().astype(np.complex128)
    for s in range(S):
        ref = oracle.run_trajectories(workloads.resolve_set(c, s), seed=31, traj_begin=s, stride=S,
                                      traj_count=per, shots=2, want_states=True)
        idx = np.arange(s, T, S)
        assert np.array_equal(out["kraus"][idx], ref["kraus"])
        assert np.array_equal(out["bits"][idx], ref["bits"])
        assert np.max(np.abs(out["obs"][idx] - ref["obs"])) < 1e-4
        for j, t in enumerate(idx):
            p = psi[t] / np.linalg.norm(psi[t])
            assert np.linalg.norm(p - ref["states"][j]) / np.linalg.norm(ref["states"][j]) < 1e-5


def test_aggregate_sets_groups_by_parameter_set():
    from paper_2111_02396_b200 import dispatch
    obs = np.arange(12, dtype=np.float64).reshape(12, 1)  # trajectories 5..16
    mean, se = dispatch.aggregate_sets(obs, 3, traj_begin=5)
    # t = 5 + j; set = t mod 3: set 2 <- j = 0, 3, 6, 9; set 0 <- j = 1, 4, 7, 10; set 1 <- 2, 5, 8, 11
    assert np.allclose(mean[:, 0], [5.5, 6.5, 4.5])
    assert np.allclose(se[:, 0], np.std([0, 3, 6, 9], ddof=1) / 2)
