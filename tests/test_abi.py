"""CPU tests of the C ABI: library loads, exports every declared symbol, and
its host-side logic (validation, canonicalization, lower bounds, planner)
behaves; no device work (no GPU here)."""
import os
import re

import numpy as np
import pytest

import oracle
import workloads
from workloads import channels, gates
from paper_2111_02396_b200 import build as B
from paper_2111_02396_b200 import qtraj

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def built():
    B.build()
    qtraj.lib()


def declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "qtraj.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"\b(qt_[a-z0-9_]+)\s*\(", hdr)))


def test_exports_every_declared_symbol():
    syms = declared_symbols()
    assert len(syms) >= 20
    L = qtraj.lib()
    for s in syms:
        assert hasattr(L, s), s


def test_no_device_means_ecuda_not_fallback():
    import ctypes
    h = ctypes.c_void_p()
    st = qtraj.lib().qt_ctx_create(0, None, ctypes.byref(h))
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if not has_gpu:
        assert st == -7  # QT_ECUDA: no CPU fallback


def test_validation_errors():
    c = qtraj.Circuit(3)
    with pytest.raises(qtraj.QtError) as e:
        c.add_gate(0, [0], np.array([[1, 1], [0, 1]]))
    assert e.value.status == -4
    with pytest.raises(qtraj.QtError) as e:
        c.add_channel(0, [0], [np.eye(2) * 0.9])
    assert e.value.status == -5
    c.add_gate(0, [0, 1], gates.CNOT())
    with pytest.raises(qtraj.QtError) as e:
        c.add_gate(0, [1], gates.X())  # qubit 1 used twice in moment 0
    assert e.value.status == -2
    with pytest.raises(qtraj.QtError) as e:
        c.add_gate(1, [3], gates.X())
    assert e.value.status == -2
    with pytest.raises(qtraj.QtError) as e:
        qtraj.Plan(c, max_fused=7)
    assert e.value.status == -3


@pytest.mark.parametrize("d", [2, 4, 8])
def test_lower_bound_matches_numpy_svd(d):
    rng = np.random.default_rng(d)
    for _ in range(5):
        K = rng.standard_normal((d, d)) + 1j * rng.standard_normal((d, d))
        ref = np.linalg.svd(K, compute_uv=False).min() ** 2
        assert abs(qtraj.kraus_lower_bound(K) - ref) < 1e-10 * max(1, ref)
    assert abs(qtraj.kraus_lower_bound(np.sqrt(0.9) * np.eye(2)) - 0.9) < 1e-14
    assert abs(qtraj.kraus_lower_bound(np.diag([1, np.sqrt(1 - 0.19)])) - 0.81) < 1e-14


def test_plan_info_deferral_counts_match_oracle_branches():
    # host planner's Alg. 2 first loop vs the oracle's: same deferred/conventional split
    c = workloads.random_circuit(6, depth=6, seed=4, noise="both", p=0.05, t1_ns=300.0, tphi_ns=600.0)
    plan = qtraj.Plan(qtraj.Circuit.from_description(c), max_fused=4)
    r = oracle.run_trajectories(c, seed=99, traj_count=30, shots=0)
    for t in range(30):
        info = plan.info(99, t)
        assert info["deferred"] == int((r["branch"][t] == 0).sum())
        assert info["conventional"] == int((r["branch"][t] == 1).sum())
        assert info["events"] == info["conventional"]


def test_plan_info_unitary_mixture_never_reduces():
    c = workloads.ghz4_depolarized(0.3)
    plan = qtraj.Plan(qtraj.Circuit.from_description(c), max_fused=4)
    for t in range(200):
        info = plan.info(7, t)
        assert info["conventional"] == 0 and info["events"] == 0  # s == 1


def test_fusion_reduces_passes_and_respects_f():
    c = workloads.sycamore_grid_qcs(config=2)
    circ = qtraj.Circuit.from_description(c)
    seen = {}
    for f in (2, 3, 4):
        plan = qtraj.Plan(circ, max_fused=f, one_gate_per_pass=True)
        info = plan.info(workloads.trajectory_seed(2), 0)
        seen[f] = info["fused_gates"]
        assert info["passes"] >= info["fused_gates"]
    assert seen[2] >= seen[3] >= seen[4]
    tiled = qtraj.Plan(circ, max_fused=4).info(workloads.trajectory_seed(2), 0)
    assert tiled["passes"] < seen[4]


def test_readout_flips_match_oracle():
    """qt_readout_flips (host, the distributed driver's readout) applied to the
    oracle's raw samples gives the oracle's recorded samples (R14)."""
    c = workloads.random_circuit(9, depth=4, seed=12, noise="depol", p=0.02, readout=True)
    c.p00 = np.full(9, 0.2)
    c.p11 = np.full(9, 0.3)
    r = oracle.run_trajectories(c, seed=41, traj_count=20, shots=5)
    assert (r["bits"] != r["bits_raw"]).any()
    for t in range(20):
        got = qtraj.readout_flips(r["bits_raw"][t], 9, c.p00, c.p11, 41, t)
        assert np.array_equal(got, r["bits"][t])
