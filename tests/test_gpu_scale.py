"""GPU parity at the benchmark's sizes (VERDICT r1 "Next round" 1(i)/(ii)), through the
C ABI against the CPU oracle: C2 (20 qubits, the bench workload and launch
configuration) on trajectory indices spread over [0, 10^4), and a 26-qubit (C3-size)
low-noise grid at f = 4 and f = 6 against the oracle's range-parallel mode (ii).
The full 256-index C2 report is tools/parity_at_scale.py (profiles/r2_parity_c2.json)."""
import numpy as np
import pytest

import oracle
import workloads

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2111_02396_b200 import qtraj  # noqa: E402
from test_gpu_parity import compare  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2111_02396_b200 import build as B
    B.build()
    return qtraj.Context(0)


def _gpu(ctx, c, seed, begin, stride, count, f, tile_bits=0, batch=None):
    plan = qtraj.Plan(qtraj.Circuit.from_description(c), max_fused=f, tile_bits=tile_bits)
    batch = batch or count
    state = torch.zeros(batch << c.n_qubits, dtype=torch.complex64, device="cuda")
    out = ctx.run_trajectories(plan, state, seed=seed, traj_count=count, traj_begin=begin, traj_stride=stride,
                               shots=1, batch=batch, observables=c.observables)
    torch.cuda.synchronize()
    return out, state


@pytest.mark.parametrize("tile_bits", [12, 13])
def test_c2_bench_workload_spread_indices(ctx, tile_bits):
    """C2 at full size: 32 trajectory indices 17 + 311 j over [0, 10^4), f = 4 tensor cores
    (tile 12: per-tile kernel; tile 13: persistent TMEM kernel): identical Kraus choices
    and samples (explained marginal decisions excepted), states within 1e-5, observables
    within 1e-4."""
    c = workloads.sycamore_grid_qcs(config=2)
    seed = workloads.trajectory_seed(2)
    ref = oracle.run_trajectories(c, seed=seed, traj_begin=17, stride=311, traj_count=32, shots=1,
                                  want_states=True)
    assert ref["rc"] == 0
    out, state = _gpu(ctx, c, seed, 17, 311, 32, 4, tile_bits=tile_bits)
    assert compare(ref, out, state) == 0


@pytest.mark.parametrize("f", [4, 6])
def test_c3_size_26_qubits(ctx, f):
    """26 qubits (C3's 2 x 13 low-noise grid, one cycle), 2 trajectories, against the
    oracle's range-parallel mode (ii); f = 4 (4-qubit tensor-core gates) and f = 6
    (5- / 6-qubit tensor-core gates)."""
    c = workloads.low_noise_grid(rows=2, cols=13, cycles=1, gamma_pd=2e-2)
    seed = workloads.trajectory_seed(3)
    ref = _c3_ref(c, seed)
    out, state = _gpu(ctx, c, seed, 0, 1, 2, f)
    assert compare(ref, out, state) == 0


_C3 = {}


def _c3_ref(c, seed):
    if "ref" not in _C3:
        _C3["ref"] = oracle.run_trajectories(c, seed=seed, traj_count=2, shots=1, want_states=True,
                                             range_parallel=True)
        assert _C3["ref"]["rc"] == 0
    return _C3["ref"]
