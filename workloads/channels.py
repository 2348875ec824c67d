"""Kraus lists of the channels used by the workloads (inputs only).

The Kraus list ORDER is data: both sides read the same uploaded list
(SURVEY 8(c) A19).
  depolarize(p):   {sqrt(1-p) I, sqrt(p/3) X, sqrt(p/3) Y, sqrt(p/3) Z}
                   i.e. E_dep of P:432 with D=2 and r_dep = p.
  depolarize2(r):  E_dep of P:432 with D=4: sqrt(1-r) I(x)I, then
                   sqrt(r/15) P_a (x) P_b for the 15 non-identity pairs in
                   lexicographic (I,X,Y,Z) order.
  decay_dephase(t, T1, Tphi): the three-operator channel of P:397-409 with
                   1/T2 = 1/(2 T1) + 1/Tphi, K2 read as diag(0, sqrt(e^{-t/T1}
                   - e^{-2t/T2})) (reading R3: the printed K2 with a 1 in the
                   top-left corner is not trace preserving).
  amplitude_damp(g): {diag(1, sqrt(1-g)), [[0, sqrt g],[0,0]]}
  phase_damp(g):     {diag(1, sqrt(1-g)), diag(0, sqrt g)}
  bit_flip(p):       {sqrt(1-p) I, sqrt(p) X}
  measure():         {|0><0|, |1><1|}: a computational-basis measurement as a
                   channel (P:102 keyed channels): sigma_min of
                   a projector is 0, so s = 0 and Alg. 2 always takes the
                   conventional branch -- p_i = <psi|P_i|psi>, collapse
                   psi <- P_i psi / sqrt(p_i), the record is the outcome i.
"""
import numpy as np

from .gates import paulis


def depolarize(p):
    I, X, Y, Z = paulis()
    return [np.sqrt(1 - p) * I, np.sqrt(p / 3) * X, np.sqrt(p / 3) * Y, np.sqrt(p / 3) * Z]


def depolarize2(r):
    P = paulis()
    ops = []
    for a in range(4):
        for b in range(4):
            if a == 0 and b == 0:
                ops.append(np.sqrt(1 - r) * np.kron(P[0], P[0]))
            else:
                ops.append(np.sqrt(r / 15) * np.kron(P[a], P[b]))
    return ops


def decay_dephase(t, T1, Tphi):
    T2 = 1.0 / (1.0 / (2.0 * T1) + 1.0 / Tphi)
    e1 = np.exp(-t / T1)
    e2 = np.exp(-t / T2)
    K0 = np.array([[1, 0], [0, e2]], dtype=np.complex128)
    K1 = np.array([[0, np.sqrt(1 - e1)], [0, 0]], dtype=np.complex128)
    K2 = np.array([[0, 0], [0, np.sqrt(max(e1 - e2 * e2, 0.0))]], dtype=np.complex128)
    return [K0, K1, K2]


def amplitude_damp(g):
    return [np.array([[1, 0], [0, np.sqrt(1 - g)]], dtype=np.complex128),
            np.array([[0, np.sqrt(g)], [0, 0]], dtype=np.complex128)]


def phase_damp(g):
    return [np.array([[1, 0], [0, np.sqrt(1 - g)]], dtype=np.complex128),
            np.array([[0, 0], [0, np.sqrt(g)]], dtype=np.complex128)]


def bit_flip(p):
    I, X, _, _ = paulis()
    return [np.sqrt(1 - p) * I, np.sqrt(p) * X]


def measure():
    return [np.array([[1, 0], [0, 0]], dtype=np.complex128), np.array([[0, 0], [0, 1]], dtype=np.complex128)]
