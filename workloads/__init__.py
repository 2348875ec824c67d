"""Seeded synthetic input generators shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no gate application, no Kraus
sampling, no lower bounds, no fusion, no sampling).  It only builds the
*inputs*: circuits as ordered moments of operations, each operation carrying
its explicit matrix (gates) or Kraus list (channels), plus readout error
tables and observable lists.  Both `oracle/` and `paper_2111_02396_b200/`
consume what is built here; neither imports the other.

Conventions:
  * qubit q <-> amplitude index bit q (R1);
  * every matrix is given in Kronecker order of the listed qubits, i.e.
    qubits[0] is the most significant matrix-index bit (R2);
  * canonical linear op order = moments in order, ops in listed order (R5).

Recipes follow SURVEY.md 8(d); seeds: circuit/calibration seed 0x211102396 + c,
trajectory seed 0x023962111 + c for config c (1-based).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import gates
from . import channels

__all__ = [
    "Gate", "Channel", "Circuit", "flatten", "gates", "channels",
    "ghz4_depolarized", "sycamore_grid_qcs", "low_noise_grid", "random_circuit",
    "circuit_seed", "trajectory_seed", "haar_unitary", "measurement", "circuit_to_json", "circuit_from_json",
    "SweepGate", "n_sets", "resolve_set", "qaoa_grid_sweep",
]


def circuit_seed(config: int) -> int:
    return 0x211102396 + config


def trajectory_seed(config: int) -> int:
    return 0x023962111 + config


@dataclass
class Gate:
    qubits: tuple
    matrix: np.ndarray  # (2^q, 2^q) complex128, Kronecker order of qubits
    name: str = "U"


@dataclass
class SweepGate:
    """Parametrized gate ("parametrized circuits for many different choices of
    parameters"): matrices[s] is the unitary of parameter set s; trajectory t of a
    run uses set t mod len(matrices)."""
    qubits: tuple
    matrices: List[np.ndarray]  # each (2^q, 2^q) complex128, Kronecker order
    name: str = "U(theta)"


@dataclass
class Channel:
    qubits: tuple
    kraus: List[np.ndarray]  # list of (2^q, 2^q) complex128, Kronecker order
    name: str = "kraus"
    record: bool = True


@dataclass
class Circuit:
    n_qubits: int
    moments: List[list] = field(default_factory=list)
    p00: Optional[np.ndarray] = None  # readout: |0> read as 1
    p11: Optional[np.ndarray] = None  # readout: |1> read as 0
    observables: List[str] = field(default_factory=list)  # 'IXYZ' strings, char q = qubit q

    def ops(self):
        for m in self.moments:
            for op in m:
                yield op

    @property
    def n_channels(self) -> int:
        return sum(isinstance(op, Channel) for op in self.ops())

    @property
    def n_gates(self) -> int:
        return sum(isinstance(op, Gate) for op in self.ops())


def flatten(c: Circuit):
    """Serialize a circuit into flat arrays in canonical order (no arithmetic).

    Returns dict with kind (0 gate / 1 channel), nq, qubits (n_ops x 6, -1 pad),
    n_kraus, record, mat_off (complex offsets), mats (interleaved float64).
    """
    kind, nq, qubits, n_kraus, record, mat_off = [], [], [], [], [], []
    blobs = []
    off = 0
    for op in c.ops():
        q = list(op.qubits)
        qubits.append(q + [-1] * (6 - len(q)))
        nq.append(len(q))
        mat_off.append(off)
        if isinstance(op, Gate):
            kind.append(0)
            n_kraus.append(0)
            record.append(0)
            m = np.ascontiguousarray(op.matrix, dtype=np.complex128)
            blobs.append(m.reshape(-1))
            off += m.size
        else:
            kind.append(1)
            n_kraus.append(len(op.kraus))
            record.append(1 if op.record else 0)
            for k in op.kraus:
                m = np.ascontiguousarray(k, dtype=np.complex128)
                blobs.append(m.reshape(-1))
                off += m.size
    mats = np.concatenate(blobs) if blobs else np.zeros(0, np.complex128)
    return dict(
        n=c.n_qubits,
        kind=np.asarray(kind, np.int32),
        nq=np.asarray(nq, np.int32),
        qubits=np.asarray(qubits, np.int32).reshape(-1, 6),
        n_kraus=np.asarray(n_kraus, np.int32),
        record=np.asarray(record, np.int32),
        mat_off=np.asarray(mat_off, np.int64),
        mats=np.ascontiguousarray(mats.view(np.float64)),
    )


def n_sets(c: Circuit) -> int:
    """Parameter sets of a circuit's sweep gates (1 without sweep gates)."""
    ns = {len(op.matrices) for op in c.ops() if isinstance(op, SweepGate)}
    if len(ns) > 1:
        raise ValueError("sweep gates with different numbers of parameter sets")
    return ns.pop() if ns else 1


def resolve_set(c: Circuit, s: int) -> Circuit:
    """The plain circuit of parameter set s (each SweepGate -> Gate(matrices[s]));
    no arithmetic, the matrices are copied as given."""
    moms = [[Gate(op.qubits, op.matrices[s], op.name) if isinstance(op, SweepGate) else op for op in m]
            for m in c.moments]
    return Circuit(n_qubits=c.n_qubits, moments=moms, p00=c.p00, p11=c.p11, observables=list(c.observables))


def measurement(qubit: int) -> Channel:
    """Mid-circuit computational-basis measurement of one qubit as a keyed channel
    (projectors; the record is the outcome, the state collapses, A12)."""
    from .channels import measure
    return Channel((int(qubit),), measure(), name="measure", record=True)


def _mat_to_json(m):
    m = np.asarray(m, dtype=np.complex128)
    return {"re": m.real.tolist(), "im": m.imag.tolist()}


def _mat_from_json(d):
    return np.asarray(d["re"], dtype=np.float64) + 1j * np.asarray(d["im"], dtype=np.float64)


def circuit_to_json(c: Circuit) -> str:
    """Circuit file format (JSON): moments of gates ({"gate": name, "qubits", "matrix"}),
    sweep gates ({"sweep": name, "qubits", "matrices": [...]}) and channels ({"channel": name, "qubits", "kraus": [...], "record"}), matrices in
    Kronecker order of the listed qubits as {"re": rows, "im": rows}; optional
    readout p00 / p11 and observables (Pauli strings, char q = qubit q)."""
    import json
    moms = []
    for m in c.moments:
        ops = []
        for op in m:
            if isinstance(op, Gate):
                ops.append({"gate": op.name, "qubits": [int(q) for q in op.qubits], "matrix": _mat_to_json(op.matrix)})
            elif isinstance(op, SweepGate):
                ops.append({"sweep": op.name, "qubits": [int(q) for q in op.qubits],
                            "matrices": [_mat_to_json(u) for u in op.matrices]})
            else:
                ops.append({"channel": op.name, "qubits": [int(q) for q in op.qubits],
                            "kraus": [_mat_to_json(k) for k in op.kraus], "record": bool(op.record)})
        moms.append(ops)
    d = {"format": "qtraj-circuit-1", "n_qubits": int(c.n_qubits), "moments": moms,
         "observables": list(c.observables)}
    if c.p00 is not None:
        d["p00"] = np.asarray(c.p00, np.float64).tolist()
    if c.p11 is not None:
        d["p11"] = np.asarray(c.p11, np.float64).tolist()
    return json.dumps(d)


def circuit_from_json(text: str) -> Circuit:
    import json
    d = json.loads(text)
    if d.get("format") != "qtraj-circuit-1":
        raise ValueError("not a qtraj-circuit-1 document")
    moms = []
    for m in d["moments"]:
        ops = []
        for op in m:
            if "gate" in op:
                ops.append(Gate(tuple(op["qubits"]), _mat_from_json(op["matrix"]), name=op["gate"]))
            elif "sweep" in op:
                ops.append(SweepGate(tuple(op["qubits"]), [_mat_from_json(u) for u in op["matrices"]], name=op["sweep"]))
            else:
                ops.append(Channel(tuple(op["qubits"]), [_mat_from_json(k) for k in op["kraus"]],
                                   name=op["channel"], record=bool(op.get("record", True))))
        moms.append(ops)
    return Circuit(n_qubits=int(d["n_qubits"]), moments=moms,
                   p00=np.asarray(d["p00"]) if "p00" in d else None,
                   p11=np.asarray(d["p11"]) if "p11" in d else None,
                   observables=list(d.get("observables", [])))


def haar_unitary(rng: np.random.Generator, d: int) -> np.ndarray:
    z = (rng.standard_normal((d, d)) + 1j * rng.standard_normal((d, d))) / np.sqrt(2)
    q, r = np.linalg.qr(z)
    ph = np.diag(r) / np.abs(np.diag(r))
    return q * ph[None, :]


# ---------------------------------------------------------------------------
# C1: GHZ-4 + depolarize(0.01) after each gate on each touched qubit.
# ---------------------------------------------------------------------------
def ghz4_depolarized(p: float = 0.01) -> Circuit:
    c = Circuit(4)
    H = gates.H()
    CX = gates.CNOT()
    seq = [(H, (0,)), (CX, (0, 1)), (CX, (1, 2)), (CX, (2, 3))]
    for m, qs in seq:
        c.moments.append([Gate(qs, m, "H" if len(qs) == 1 else "CX")])
        c.moments.append([Channel((q,), channels.depolarize(p), "depolarize") for q in qs])
    c.observables = ["ZIII", "IZII", "IIZI", "IIIZ", "ZZZZ", "XXXX"]
    return c


# ---------------------------------------------------------------------------
# Sycamore-style grid circuits.
# ---------------------------------------------------------------------------
def _grid_couplers(rows: int, cols: int):
    """Coupler patterns A/B/C/D on a rows x cols grid (qubit = r*cols + c).

    A/B: horizontal pairs starting at even/odd columns; C/D: vertical pairs
    starting at even/odd rows.  (Public Sycamore-like convention; external to
    the paper, which only gives fSim.)"""
    pat = {"A": [], "B": [], "C": [], "D": []}
    for r in range(rows):
        for c0 in range(cols - 1):
            (pat["A"] if c0 % 2 == 0 else pat["B"]).append((r * cols + c0, r * cols + c0 + 1))
    for r0 in range(rows - 1):
        for c in range(cols):
            (pat["C"] if r0 % 2 == 0 else pat["D"]).append((r0 * cols + c, (r0 + 1) * cols + c))
    return pat


def sycamore_grid_qcs(rows: int = 4, cols: int = 5, cycles: int = 14,
                      config: int = 2, noise: bool = True,
                      depol_1q: float = 1e-3, depol_2q: float = 5e-3,
                      t1q_ns: float = 25.0, t2q_ns: float = 32.0) -> Circuit:
    """C2: Sycamore-style random circuit with the approximate QCS noise model.

    Per cycle: 1q layer {sqrtX, sqrtY, sqrtW} (never repeating on a qubit),
    depolarizing(r=1e-3) after each 1q gate, decay/dephasing triple on every
    qubit (t = 25 ns); fSim(pi/2, pi/6) on pattern ABCDCDAB, coherent error
    fSim(dtheta, dphi) after it, 2q depolarizing (r=5e-3), decay triple on every
    qubit (t = 32 ns).  Calibration: T1 ~ U[12,20] us, Tphi ~ U[20,40] us,
    p00 ~ U[0.005,0.015], p11 ~ U[0.03,0.06], dtheta,dphi ~ N(0, 0.02) per pair.
    These are synthetic typical-order values, not the paper's.
    """
    rng = np.random.default_rng(circuit_seed(config))
    n = rows * cols
    c = Circuit(n)
    T1 = rng.uniform(12e3, 20e3, n)      # ns
    Tphi = rng.uniform(20e3, 40e3, n)    # ns
    c.p00 = rng.uniform(0.005, 0.015, n) if noise else None
    c.p11 = rng.uniform(0.03, 0.06, n) if noise else None
    pats = _grid_couplers(rows, cols)
    pair_err = {}
    for name in "ABCD":
        for pr in pats[name]:
            pair_err[pr] = (rng.normal(0, 0.02), rng.normal(0, 0.02))
    one_q = [gates.sqrt_x(), gates.sqrt_y(), gates.sqrt_w()]
    prev = [-1] * n
    order = "ABCDCDAB"
    fsim = gates.fsim(np.pi / 2, np.pi / 6)
    for cyc in range(cycles):
        m1 = []
        for q in range(n):
            choices = [i for i in range(3) if i != prev[q]]
            k = choices[rng.integers(len(choices))]
            prev[q] = k
            m1.append(Gate((q,), one_q[k], ["sqrtX", "sqrtY", "sqrtW"][k]))
        c.moments.append(m1)
        if noise:
            c.moments.append([Channel((q,), channels.depolarize(depol_1q), "depolarize") for q in range(n)])
            c.moments.append([Channel((q,), channels.decay_dephase(t1q_ns, T1[q], Tphi[q]), "decay")
                              for q in range(n)])
        pairs = pats[order[cyc % len(order)]]
        c.moments.append([Gate(pr, fsim, "fSim") for pr in pairs])
        if noise:
            c.moments.append([Gate(pr, gates.fsim(*pair_err[pr]), "fSim_err") for pr in pairs])
            c.moments.append([Channel(pr, channels.depolarize2(depol_2q), "depolarize2") for pr in pairs])
            c.moments.append([Channel((q,), channels.decay_dephase(t2q_ns, T1[q], Tphi[q]), "decay")
                              for q in range(n)])
    c.observables = ["I" * q + "Z" + "I" * (n - q - 1) for q in range(n)]
    return c


def low_noise_grid(rows: int = 2, cols: int = 13, cycles: int = 20, config: int = 3,
                   depol: float = 1e-3, gamma_pd: float = 1e-4, damping: str = "phase") -> Circuit:
    """C3: depolarize(1e-3) after every gate (unitary mixture, always deferred)
    plus phase_damp(gamma) on every qubit per moment.
    damping="amplitude": amplitude_damp(gamma) instead (C4 (ii): 4 x 8 grid,
    depolarize 1e-3, gamma = 1e-4)."""
    damp = channels.phase_damp if damping == "phase" else channels.amplitude_damp
    rng = np.random.default_rng(circuit_seed(config))
    n = rows * cols
    c = Circuit(n)
    pats = _grid_couplers(rows, cols)
    one_q = [gates.sqrt_x(), gates.sqrt_y(), gates.sqrt_w()]
    prev = [-1] * n
    order = "ABCDCDAB"
    fsim = gates.fsim(np.pi / 2, np.pi / 6)
    for cyc in range(cycles):
        m1 = []
        for q in range(n):
            choices = [i for i in range(3) if i != prev[q]]
            k = choices[rng.integers(len(choices))]
            prev[q] = k
            m1.append(Gate((q,), one_q[k]))
        c.moments.append(m1)
        if depol > 0:
            c.moments.append([Channel((q,), channels.depolarize(depol)) for q in range(n)])
        c.moments.append([Channel((q,), damp(gamma_pd)) for q in range(n)])
        pairs = pats[order[cyc % len(order)]]
        c.moments.append([Gate(pr, fsim, "fSim") for pr in pairs])
        if depol > 0:
            c.moments.append([Channel(pr, channels.depolarize2(depol)) for pr in pairs])
        c.moments.append([Channel((q,), damp(gamma_pd)) for q in range(n)])
    c.observables = ["I" * q + "Z" + "I" * (n - q - 1) for q in range(n)]
    return c


def random_circuit(n: int, depth: int, seed: int, max_arity: int = 2,
                   noise: Optional[str] = None, p: float = 0.01,
                   t1_ns: float = 3000.0, tphi_ns: float = 6000.0,
                   t_ns: float = 32.0, readout: bool = False) -> Circuit:
    """Haar-random 1q/2q (up to max_arity) gates on random disjoint qubits.

    noise: None | 'depol' | 'decay' | 'both' | 'ad' (amplitude damping p) |
    'pd' (phase damping p) -- channels after every gate on its qubits."""
    rng = np.random.default_rng(seed)
    c = Circuit(n)
    for _ in range(depth):
        perm = list(rng.permutation(n))
        moment, nmoment = [], []
        while perm:
            k = int(rng.integers(1, max_arity + 1))
            k = min(k, len(perm))
            qs = tuple(int(x) for x in perm[:k])
            perm = perm[k:]
            moment.append(Gate(qs, haar_unitary(rng, 2 ** k)))
            if noise is not None:
                for q in qs:
                    if noise in ("depol", "both"):
                        nmoment.append(Channel((q,), channels.depolarize(p)))
                    if noise in ("decay", "both"):
                        nmoment.append(Channel((q,), channels.decay_dephase(t_ns, t1_ns, tphi_ns)))
                    if noise == "ad":
                        nmoment.append(Channel((q,), channels.amplitude_damp(p)))
                    if noise == "pd":
                        nmoment.append(Channel((q,), channels.phase_damp(p)))
        c.moments.append(moment)
        if nmoment:
            # channels on the same qubit would collide inside one moment;
            # split into as many moments as needed (order preserved)
            while nmoment:
                used, cur, rest = set(), [], []
                for ch in nmoment:
                    if used.isdisjoint(ch.qubits):
                        cur.append(ch)
                        used.update(ch.qubits)
                    else:
                        rest.append(ch)
                c.moments.append(cur)
                nmoment = rest
    if readout:
        c.p00 = rng.uniform(0.005, 0.015, n)
        c.p11 = rng.uniform(0.03, 0.06, n)
    c.observables = ["I" * q + "Z" + "I" * (n - q - 1) for q in range(n)]
    return c


# ---------------------------------------------------------------------------
# NEXT-4: parameter sweeps.  QAOA-style grid circuit (the paper's
# "Hardware Grid" QAOA, as a circuit family only): |+>^n, then p
# layers of exp(-i gamma Z Z) on every grid coupler (patterns A, B, C, D as
# disjoint moments) and exp(-i beta X) mixers; (gamma_s, beta_s) per set s.
# ---------------------------------------------------------------------------
def zz_phase(gamma: float) -> np.ndarray:
    """exp(-i gamma Z(x)Z) (diagonal)."""
    return np.diag(np.exp(-1j * gamma * np.array([1.0, -1.0, -1.0, 1.0]))).astype(np.complex128)


def x_mixer(beta: float) -> np.ndarray:
    """exp(-i beta X)."""
    c, s = np.cos(beta), np.sin(beta)
    return np.array([[c, -1j * s], [-1j * s, c]], dtype=np.complex128)


def qaoa_grid_sweep(rows: int, cols: int, layers: int, gammas: Sequence[Sequence[float]],
                    betas: Sequence[Sequence[float]], depol: float = 1e-3, amp_damp: float = 0.0) -> Circuit:
    """gammas[s][l], betas[s][l]: angles of layer l in parameter set s.  Noise:
    depolarize(depol) after every 1q gate and on both qubits after every ZZ phase
    (unitary mixtures), optional amplitude damping on every qubit per layer.
    Observables: Z_a Z_b on every coupler."""
    n = rows * cols
    S = len(gammas)
    assert len(betas) == S and all(len(g) == layers and len(b) == layers for g, b in zip(gammas, betas))
    pat = _grid_couplers(rows, cols)
    c = Circuit(n)
    c.moments.append([Gate((q,), gates.H(), "H") for q in range(n)])
    if depol > 0:
        c.moments.append([Channel((q,), channels.depolarize(depol), "depolarize") for q in range(n)])
    for l in range(layers):
        for key in "ABCD":
            if not pat[key]:
                continue
            c.moments.append([SweepGate((a, b), [zz_phase(gammas[s][l]) for s in range(S)], "ZZ(gamma)")
                              for a, b in pat[key]])
            if depol > 0:
                c.moments.append([Channel((q,), channels.depolarize(depol), "depolarize")
                                  for a, b in pat[key] for q in (a, b)])
        c.moments.append([SweepGate((q,), [x_mixer(betas[s][l]) for s in range(S)], "X(beta)") for q in range(n)])
        if depol > 0:
            c.moments.append([Channel((q,), channels.depolarize(depol), "depolarize") for q in range(n)])
        if amp_damp > 0:
            c.moments.append([Channel((q,), channels.amplitude_damp(amp_damp), "amplitude_damp")
                              for q in range(n)])
    edges = [e for key in "ABCD" for e in pat[key]]
    c.observables = ["".join("Z" if q in e else "I" for q in range(n)) for e in edges]
    return c
