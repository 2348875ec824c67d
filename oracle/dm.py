"""Brute-force density-matrix oracle O2 (TEST INFRASTRUCTURE ONLY; n <= 10).

rho <- U rho U^dag for gates, rho <- sum_i K_i rho K_i^dag for channels: the
exact ensemble the trajectories sample (p_i = <Psi|K_i^dag K_i|Psi>).
Each operator is embedded densely into 2^n x 2^n by explicit index mapping
(qubit q <-> index bit q; matrix in Kronecker order of the listed qubits).
Readout acts on the diagonal as a per-qubit confusion matrix.
"""
import numpy as np


def embed(U: np.ndarray, qubits, n: int) -> np.ndarray:
    """Dense 2^n x 2^n operator equal to U on `qubits` (Kronecker order), I elsewhere."""
    k = len(qubits)
    dim = 2 ** n
    E = np.zeros((dim, dim), np.complex128)
    for col in range(dim):
        # matrix column index of this basis state: qubits[0] is the MSB
        j = 0
        for m, q in enumerate(qubits):
            j |= ((col >> q) & 1) << (k - 1 - m)
        rest = col
        for q in qubits:
            rest &= ~(1 << q)
        for i in range(2 ** k):
            row = rest
            for m, q in enumerate(qubits):
                if (i >> (k - 1 - m)) & 1:
                    row |= 1 << q
            E[row, col] += U[i, j]
    return E


def evolve(circuit) -> np.ndarray:
    """Final density matrix of `circuit` (workloads.Circuit) from |0..0>."""
    from workloads import Gate  # input types only
    n = circuit.n_qubits
    dim = 2 ** n
    rho = np.zeros((dim, dim), np.complex128)
    rho[0, 0] = 1.0
    for op in circuit.ops():
        if isinstance(op, Gate):
            E = embed(op.matrix, op.qubits, n)
            rho = E @ rho @ E.conj().T
        else:
            new = np.zeros_like(rho)
            for K in op.kraus:
                E = embed(K, op.qubits, n)
                new += E @ rho @ E.conj().T
            rho = new
    return rho


def pauli_matrix(paulis: str) -> np.ndarray:
    P1 = {"I": np.eye(2), "X": np.array([[0, 1], [1, 0]]),
          "Y": np.array([[0, -1j], [1j, 0]]), "Z": np.diag([1.0, -1.0])}
    n = len(paulis)
    M = np.eye(1, dtype=np.complex128)
    # char q acts on qubit q; qubit n-1 is the most significant index bit
    for q in reversed(range(n)):
        M = np.kron(M, P1[paulis[q]])
    return M


def expectation(rho: np.ndarray, paulis: str) -> float:
    return float(np.real(np.trace(pauli_matrix(paulis) @ rho)))


def outcome_probabilities(rho: np.ndarray, p00=None, p11=None) -> np.ndarray:
    """Distribution of recorded bitstrings (index = bitstring, bit q = qubit q)."""
    probs = np.real(np.diag(rho)).copy()
    n = int(np.log2(len(probs)))
    for q in range(n):
        e0 = 0.0 if p00 is None else p00[q]
        e1 = 0.0 if p11 is None else p11[q]
        new = np.zeros_like(probs)
        for x in range(len(probs)):
            b = (x >> q) & 1
            y = x ^ (1 << q)
            if b == 0:
                new[x] += (1 - e0) * probs[x]
                new[y] += e0 * probs[x]
            else:
                new[x] += (1 - e1) * probs[x]
                new[y] += e1 * probs[x]
        probs = new
    return probs
