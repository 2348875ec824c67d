"""NEXT-2: calibrated QCS approximate noise model and the Z2-gauge
fiducial channels (Eq. 1 / Eq. 2).  Host-side circuit construction
only (inputs to both the oracle and the CUDA path; no method arithmetic).

Calibration -> channels, following P:393-439 step by step:
  * dephasing time from the incoherent error (to leading order)
        eps_inc = t/(3 T1) + t/(3 T_phi)   =>   T_phi = t / (3 eps_inc - t/T1)
  * decay + dephasing channel E with 1/T2 = 1/(2 T1) + 1/T_phi,
    applied on every qubit after every moment (gate or idle time) with the
    moment's duration (reading A16; K2 as reading R3)
  * readout: parallel_p00_error / parallel_p11_error
  * fSim coherent errors: Z phases e^{i phi Z} on both qubits
    before and after, then fSim(d_theta, d_phi) after each fSim
  * depolarizing error sized so the total Pauli error matches the
    calibration: two-qubit gates r_dep = r_p^tot - r_inc^0 - r_inc^1 - r_ent
    (P:436-439); one-qubit gates r_dep = r_p^tot(RB) - r_inc.

Readings (the paper points to Ref. 2019 for the error-rate conversions and is
silent on the rest; DESIGN.md lists them):
  N1 Pauli (process) error of a channel = 1 - F_pro, F_pro = sum_i |Tr K_i|^2 / D^2;
     average error r_avg = D/(D+1) * r_p.  (With these, the paper's eps_inc is the
     average error of the decay channel to first order in t -- pinned in tests.)
  N2 one-qubit RB reports an average error: r_p^tot = (D+1)/D * rb = 3/2 rb.
  N3 r_inc^q = Pauli error of the decay channel of qubit q over the gate time.
  N4 r_ent = Pauli error of the whole coherent error unitary (Z phases and
     fSim(d_theta, d_phi)), i.e. 1 - |Tr U|^2 / 16.
  N5 r_dep is clamped at 0 when the explicit errors exceed the calibrated total.
"""
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

import numpy as np

from . import Channel, Circuit, Gate, channels, gates


# ---------------------------------------------------------------------------
# Conversions
# ---------------------------------------------------------------------------
def t_phi_from_eps_inc(eps_inc: float, t: float, T1: float) -> float:
    """P:369 solved for T_phi (leading order); inf when eps_inc <= t/(3 T1)."""
    d = 3.0 * eps_inc - t / T1
    return float("inf") if d <= 0 else t / d


def pauli_error(kraus: List[np.ndarray]) -> float:
    """N1: 1 - sum_i |Tr K_i|^2 / D^2."""
    D = kraus[0].shape[0]
    return float(1.0 - sum(abs(np.trace(K)) ** 2 for K in kraus) / D ** 2)


def average_error(kraus: List[np.ndarray]) -> float:
    D = kraus[0].shape[0]
    return D / (D + 1) * pauli_error(kraus)


def decay_channel(t: float, T1: float, Tphi: float) -> List[np.ndarray]:
    """P:397-409 (K2 read as diag(0, .), R3); T_phi = inf means pure decay."""
    if np.isinf(Tphi):
        Tphi = 1e300
    return channels.decay_dephase(t, T1, Tphi)


def z_phase(phi: float) -> np.ndarray:
    """e^{i phi Z}."""
    return np.diag([np.exp(1j * phi), np.exp(-1j * phi)]).astype(np.complex128)


def depolarize_n(eps: float, n: int) -> List[np.ndarray]:
    """Eq. 1: D_n[eps](rho) = (1 - eps) rho + eps I / 2^n as Kraus
    operators: sqrt(1 - eps + eps/4^n) I and sqrt(eps/4^n) P for the 4^n - 1
    non-identity Pauli strings (lexicographic, I X Y Z per qubit)."""
    P = gates.paulis()
    D2 = 4 ** n
    ops = []
    for idx in range(D2):
        m = np.array([[1.0 + 0j]])
        for a in range(n):
            m = np.kron(m, P[(idx >> (2 * (n - 1 - a))) & 3])
        w = (1.0 - eps + eps / D2) if idx == 0 else eps / D2
        ops.append(np.sqrt(w) * m)
    return ops


def u_zz(zeta: float, T: float) -> np.ndarray:
    """Eq. 2: exp(-i 2 pi zeta T |11><11|)."""
    return np.diag([1, 1, 1, np.exp(-2j * np.pi * zeta * T)]).astype(np.complex128)


# ---------------------------------------------------------------------------
# Calibration data and the noisy-circuit builder
# ---------------------------------------------------------------------------
@dataclass
class QubitCal:
    T1: float              # ns
    eps_inc: float         # one-qubit incoherent (purity-benchmarking) error per 1q gate
    rb_1q: float           # isolated one-qubit RB average error
    p00: float = 0.0       # parallel_p00_error
    p11: float = 0.0       # parallel_p11_error


@dataclass
class PairCal:
    xeb_pauli: float                     # total parallel-XEB Pauli error r_p^tot of the 2q gate
    d_theta: float = 0.0                 # fSim angle deviations
    d_phi: float = 0.0
    z_before: Tuple[float, float] = (0.0, 0.0)   # Z phase errors on (q0, q1) before / after
    z_after: Tuple[float, float] = (0.0, 0.0)


@dataclass
class QCSNoiseModel:
    qubits: Dict[int, QubitCal]
    pairs: Dict[Tuple[int, int], PairCal] = field(default_factory=dict)
    t_1q: float = 25.0     # ns
    t_2q: float = 32.0     # ns

    def t_phi(self, q: int) -> float:
        c = self.qubits[q]
        return t_phi_from_eps_inc(c.eps_inc, self.t_1q, c.T1)

    def decay(self, q: int, t: float) -> List[np.ndarray]:
        return decay_channel(t, self.qubits[q].T1, self.t_phi(q))

    def r_inc(self, q: int, t: float) -> float:
        return pauli_error(self.decay(q, t))

    def coherent_2q(self, pair: Tuple[int, int], G: Optional[np.ndarray] = None) -> np.ndarray:
        """The coherent error E inserted AFTER the ideal gate G of the pair, so that
        E G = Z_after fSim(d_theta, d_phi) G Z_before: Z phase errors before and after
        the gate and the fSim angle deviations (fSim gates compose
        additively).  E = Z_after fSim(d) G Z_before G^dagger (Kronecker order of pair);
        G = None means identity (no Z_before / G reordering)."""
        pc = self.pairs.get(pair, PairCal(0.0))
        zb = np.kron(z_phase(pc.z_before[0]), z_phase(pc.z_before[1]))
        za = np.kron(z_phase(pc.z_after[0]), z_phase(pc.z_after[1]))
        if G is None:
            return za @ gates.fsim(pc.d_theta, pc.d_phi) @ zb
        return za @ gates.fsim(pc.d_theta, pc.d_phi) @ G @ zb @ G.conj().T

    def r_ent(self, pair: Tuple[int, int], G: Optional[np.ndarray] = None) -> float:
        return pauli_error([self.coherent_2q(pair, G)])

    def r_dep_2q(self, pair: Tuple[int, int], G: Optional[np.ndarray] = None) -> float:
        pc = self.pairs.get(pair, PairCal(0.0))
        r = pc.xeb_pauli - self.r_inc(pair[0], self.t_2q) - self.r_inc(pair[1], self.t_2q) - self.r_ent(pair, G)
        return max(0.0, r)

    def r_dep_1q(self, q: int) -> float:
        return max(0.0, 1.5 * self.qubits[q].rb_1q - self.r_inc(q, self.t_1q))

    def noisy(self, c: Circuit) -> Circuit:
        """Insert the approximate QCS noise into a noiseless circuit whose
        moments hold 1q gates and 2q fSim-family gates: per gate the coherent
        errors (2q) and the depolarizing remainder, then the decay channel on
        every qubit for the moment's duration; readout errors per qubit."""
        out = Circuit(n_qubits=c.n_qubits, observables=list(c.observables))
        for mom in c.moments:
            coherent, depol = [], []
            two_q = any(len(op.qubits) == 2 for op in mom)
            for op in mom:
                if not isinstance(op, Gate):
                    continue
                qs = tuple(op.qubits)
                if len(qs) == 2:
                    coherent.append(Gate(qs, self.coherent_2q(qs, op.matrix), "coherent_err"))
                    r = self.r_dep_2q(qs, op.matrix)
                    if r > 0:
                        depol.append(Channel(qs, channels.depolarize2(r), "depolarize2"))
                elif len(qs) == 1:
                    r = self.r_dep_1q(qs[0])
                    if r > 0:
                        depol.append(Channel(qs, channels.depolarize(r), "depolarize"))
            # each moment keeps its qubits disjoint
            out.moments.append(list(mom))
            for extra in (coherent, depol):
                if extra:
                    out.moments.append(extra)
            t = self.t_2q if two_q else self.t_1q
            out.moments.append([Channel((q,), self.decay(q, t), "decay") for q in range(c.n_qubits)])
        out.p00 = np.array([self.qubits[q].p00 for q in range(c.n_qubits)])
        out.p11 = np.array([self.qubits[q].p11 for q in range(c.n_qubits)])
        return out


def synthetic_calibration(n: int, pairs: List[Tuple[int, int]], seed: int) -> QCSNoiseModel:
    """Seeded synthetic calibration with Sycamore-like magnitudes (the paper gives
    no values; P:409 points to a datasheet): T1 ~ U[12, 20] us, eps_inc ~
    U[5e-4, 1.2e-3], RB ~ U[1e-3, 2e-3], p00 ~ U[.005, .015], p11 ~ U[.03, .06],
    XEB Pauli ~ U[5e-3, 9e-3], fSim deviations ~ N(0, 0.02), Z phases ~ N(0, 0.01)."""
    rng = np.random.default_rng(seed)
    qc = {q: QubitCal(T1=float(rng.uniform(12e3, 20e3)), eps_inc=float(rng.uniform(5e-4, 1.2e-3)),
                      rb_1q=float(rng.uniform(1e-3, 2e-3)), p00=float(rng.uniform(0.005, 0.015)),
                      p11=float(rng.uniform(0.03, 0.06))) for q in range(n)}
    pc = {}
    for p in pairs:
        pc[tuple(p)] = PairCal(xeb_pauli=float(rng.uniform(5e-3, 9e-3)), d_theta=float(rng.normal(0, 0.02)),
                               d_phi=float(rng.normal(0, 0.02)),
                               z_before=(float(rng.normal(0, 0.01)), float(rng.normal(0, 0.01))),
                               z_after=(float(rng.normal(0, 0.01)), float(rng.normal(0, 0.01))))
    return QCSNoiseModel(qubits=qc, pairs=pc)
