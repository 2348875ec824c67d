"""CPU oracle for the noisy-trajectory hot path (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` legs may import this package.  It shares no code with
paper_2111_02396_b200/ (the product path): `oracle.c` is a plain fp64
implementation of Alg. 1 / Alg. 2 of arXiv 2111.02396 with its own Philox,
and `dm.py` is a brute-force numpy density-matrix simulator.

Every function cites the passage it follows (see oracle.c's header).
"""
import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.c")

PURPOSE_CHANNEL, PURPOSE_SAMPLE, PURPOSE_READOUT = 1, 2, 3


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (plain -O2, no vector intrinsics)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-pthread",
                               "-o", _SO, _SRC, "-lm"])
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        P = ctypes.POINTER
        u32p = P(ctypes.c_uint32)
        L.orc_philox4x32_10.argtypes = [u32p, u32p, u32p]
        L.orc_philox4x32_10.restype = None
        L.orc_u53.argtypes = [ctypes.c_uint32, ctypes.c_uint32]
        L.orc_u53.restype = ctypes.c_double
        L.orc_uniform.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32,
                                  ctypes.c_uint64, ctypes.c_int]
        L.orc_uniform.restype = ctypes.c_double
        L.orc_apply_gate.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_void_p, ctypes.c_void_p]
        L.orc_apply_gate.restype = ctypes.c_int
        L.orc_sigma_min_sq.argtypes = [ctypes.c_int, ctypes.c_void_p]
        L.orc_sigma_min_sq.restype = ctypes.c_double
        L.orc_is_unitary_mixture.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
        L.orc_is_unitary_mixture.restype = ctypes.c_int
        L.orc_sample_state.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_uint64,
                                       ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p,
                                       ctypes.c_void_p]
        L.orc_sample_state.restype = ctypes.c_int
        L.orc_pauli_expectation.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_char_p]
        L.orc_pauli_expectation.restype = ctypes.c_double
        vp = ctypes.c_void_p
        L.orc_run_trajectories.argtypes = (
            [ctypes.c_int, ctypes.c_int, vp, vp, vp, vp, vp, vp, vp, vp, ctypes.c_int, vp,
             ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int64,
             ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int] + [vp] * 9)
        L.orc_run_trajectories.restype = ctypes.c_int
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data


def philox(ctr, key):
    c = (ctypes.c_uint32 * 4)(*ctr)
    k = (ctypes.c_uint32 * 2)(*key)
    o = (ctypes.c_uint32 * 4)()
    lib().orc_philox4x32_10(c, k, o)
    return list(o)


def u53(a, b):
    return lib().orc_u53(a, b)


def uniform(seed, ordinal, purpose, traj, half=0):
    return lib().orc_uniform(seed, ordinal, purpose, traj, half)


def apply_gate(psi: np.ndarray, qubits, U: np.ndarray) -> np.ndarray:
    """Alg. 1 on a complex128 state, in place; returns psi."""
    assert psi.dtype == np.complex128 and psi.flags.c_contiguous
    n = int(np.log2(psi.size))
    qs = np.asarray(qubits, np.int32)
    U = np.ascontiguousarray(U, np.complex128)
    st = lib().orc_apply_gate(psi.ctypes.data, n, len(qs), qs.ctypes.data, U.ctypes.data)
    if st != 0:
        raise ValueError(f"orc_apply_gate status {st}")
    return psi


def sigma_min_sq(K: np.ndarray) -> float:
    """p-bar = smallest singular value squared, via Jacobi on K^dag K."""
    K = np.ascontiguousarray(K, np.complex128)
    return lib().orc_sigma_min_sq(K.shape[0], K.ctypes.data)


def is_unitary_mixture(kraus) -> bool:
    Ks = np.ascontiguousarray(np.stack(kraus), np.complex128)
    return bool(lib().orc_is_unitary_mixture(Ks.shape[1], Ks.shape[0], Ks.ctypes.data))


def sample_state(psi: np.ndarray, seed: int, traj: int, shots: int):
    n = int(np.log2(psi.size))
    psi = np.ascontiguousarray(psi, np.complex128)
    bits = np.zeros(shots, np.uint64)
    mg = np.zeros(shots, np.float64)
    lib().orc_sample_state(psi.ctypes.data, n, seed, traj, shots, bits.ctypes.data, mg.ctypes.data)
    return bits, mg


def pauli_expectation(psi: np.ndarray, paulis: str) -> float:
    n = int(np.log2(psi.size))
    assert len(paulis) == n
    psi = np.ascontiguousarray(psi, np.complex128)
    return lib().orc_pauli_expectation(psi.ctypes.data, n, paulis.encode())


class TrajectoryResult(dict):
    pass


def run_trajectories(circuit, seed: int, traj_begin: int = 0, traj_count: int = 1,
                     stride: int = 1, shots: int = 1, threads: int = None,
                     want_states: bool = False, mode: int = 0, range_parallel: bool = False) -> TrajectoryResult:
    """Alg. 2 trajectories t = traj_begin + stride*j, j < traj_count.

    mode 0 = delayed inner products (Alg. 2); mode 1 = the conventional
    trajectory algorithm (every channel computes its p_i).
    range_parallel: parallel mode (ii) (for n >= 24): one
    trajectory at a time, the Alg. 1 outer loop of every pass split into 64 fixed
    index ranges over `threads` threads; results are identical to mode (i).
    `circuit` is a workloads.Circuit.  Returns numpy arrays keyed by name."""
    from workloads import flatten  # input serialization only
    f = flatten(circuit)
    n = f["n"]
    n_ops = len(f["kind"])
    n_ch = int((f["kind"] == 1).sum())
    n_obs = len(circuit.observables)
    obs = "".join(circuit.observables).encode() if n_obs else None
    obs_buf = ctypes.create_string_buffer(obs) if obs else None
    p00 = None if circuit.p00 is None else np.ascontiguousarray(circuit.p00, np.float64)
    p11 = None if circuit.p11 is None else np.ascontiguousarray(circuit.p11, np.float64)
    T = traj_count
    out = TrajectoryResult(
        kraus=np.zeros((T, n_ch), np.int32), branch=np.zeros((T, n_ch), np.int8),
        kraus_margin=np.zeros((T, n_ch), np.float64),
        bits=np.zeros((T, shots), np.uint64), bits_raw=np.zeros((T, shots), np.uint64),
        sample_margin=np.zeros((T, shots), np.float64),
        obs=np.zeros((T, n_obs), np.float64), status=np.zeros(T, np.int32))
    states = np.zeros((T, 2 ** n), np.complex128) if want_states else None
    if threads is None:
        threads = os.cpu_count() or 1
    qubits = np.ascontiguousarray(f["qubits"].reshape(-1), np.int32)
    st = lib().orc_run_trajectories(
        n, n_ops, _ptr(f["kind"]), _ptr(f["nq"]), _ptr(qubits), _ptr(f["n_kraus"]),
        _ptr(f["mat_off"]), _ptr(f["mats"]), _ptr(p00), _ptr(p11), n_obs,
        ctypes.addressof(obs_buf) if obs_buf is not None else None,
        seed, traj_begin, stride, T, shots, 1 if range_parallel else threads, mode,
        threads if range_parallel else 0,
        _ptr(states), _ptr(out["kraus"]), _ptr(out["branch"]), _ptr(out["kraus_margin"]),
        _ptr(out["bits"]), _ptr(out["bits_raw"]), _ptr(out["sample_margin"]),
        _ptr(out["obs"]), _ptr(out["status"]))
    out["rc"] = st
    out["threads"] = threads
    if want_states:
        out["states"] = states
    return out
