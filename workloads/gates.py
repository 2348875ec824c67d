"""Gate matrices (inputs only; Kronecker order of the listed qubits).

fSim(theta, phi) as printed at P:416-421.  sqrt(P) = ((1+i) I + (1-i) P)/2
for P^2 = I (the Sycamore single-qubit set {sqrtX, sqrtY, sqrtW}).
"""
import numpy as np

_I = np.eye(2, dtype=np.complex128)
_X = np.array([[0, 1], [1, 0]], dtype=np.complex128)
_Y = np.array([[0, -1j], [1j, 0]], dtype=np.complex128)
_Z = np.array([[1, 0], [0, -1]], dtype=np.complex128)


def I():
    return _I.copy()


def X():
    return _X.copy()


def Y():
    return _Y.copy()


def Z():
    return _Z.copy()


def H():
    return np.array([[1, 1], [1, -1]], dtype=np.complex128) / np.sqrt(2)


def CNOT():
    """Control = first listed qubit (most significant matrix bit)."""
    m = np.eye(4, dtype=np.complex128)
    m[2:, 2:] = _X
    return m


def CZ():
    return np.diag([1, 1, 1, -1]).astype(np.complex128)


def _sqrt_pauli(P):
    return ((1 + 1j) * _I + (1 - 1j) * P) / 2


def sqrt_x():
    return _sqrt_pauli(_X)


def sqrt_y():
    return _sqrt_pauli(_Y)


def sqrt_w():
    W = (_X + _Y) / np.sqrt(2)
    return _sqrt_pauli(W)


def rz(phi):
    return np.diag([np.exp(-0.5j * phi), np.exp(0.5j * phi)])


def fsim(theta, phi):
    """fSim(theta, phi)."""
    c, s = np.cos(theta), np.sin(theta)
    return np.array([[1, 0, 0, 0],
                     [0, c, -1j * s, 0],
                     [0, -1j * s, c, 0],
                     [0, 0, 0, np.exp(-1j * phi)]], dtype=np.complex128)


def paulis():
    return [_I.copy(), _X.copy(), _Y.copy(), _Z.copy()]
