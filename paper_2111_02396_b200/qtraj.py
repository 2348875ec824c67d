"""ctypes binding of libqtraj (include/qtraj.h): argument marshalling only.

Every step of the hot path runs in the library's sm_100a kernels; this module
converts Python/numpy/torch arguments into the C ABI's plain pointers and
sizes.  There is no CPU fallback: if libqtraj.so is missing or no CUDA device
is present, the calls raise.
"""
from __future__ import annotations

import ctypes
import os
from typing import Iterable, List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("QT_LIB_PATH") or os.path.join(_HERE, "libqtraj.so")  # QT_LIB_PATH: experiment builds

STATUS = {0: "QT_OK", -1: "QT_EINVAL", -2: "QT_EQUBIT", -3: "QT_EARITY", -4: "QT_ENONUNITARY",
          -5: "QT_ENONCPTP", -6: "QT_EOOM", -7: "QT_ECUDA", -8: "QT_ENCCL", -9: "QT_ELEAK",
          -10: "QT_ESTATE"}


class QtError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class Stats(ctypes.Structure):
    _fields_ = [("trajectories", ctypes.c_uint64), ("passes", ctypes.c_uint64),
                ("fused_gates", ctypes.c_uint64), ("reductions", ctypes.c_uint64),
                ("channels_deferred", ctypes.c_uint64), ("channels_conventional", ctypes.c_uint64),
                ("launches", ctypes.c_uint64), ("alg_bytes", ctypes.c_double),
                ("alg_flops", ctypes.c_double), ("plan_ms", ctypes.c_double),
                ("device_ms", ctypes.c_double), ("pass_kernel_ms", ctypes.c_double),
                ("pass_launches", ctypes.c_uint64), ("h2d_bytes", ctypes.c_uint64),
                ("d2h_bytes", ctypes.c_uint64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class FuseOpts(ctypes.Structure):
    _fields_ = [("max_fused", ctypes.c_int), ("tile_bits", ctypes.c_int),
                ("low_bits", ctypes.c_int), ("one_gate_per_pass", ctypes.c_int),
                ("tensor_cores", ctypes.c_int)]


class RunOpts(ctypes.Structure):
    _fields_ = [("seed", ctypes.c_uint64), ("traj_begin", ctypes.c_uint64),
                ("traj_stride", ctypes.c_uint64), ("traj_count", ctypes.c_uint64),
                ("shots_per_traj", ctypes.c_int), ("batch", ctypes.c_int), ("mode", ctypes.c_int),
                ("profile", ctypes.c_int), ("host_threads", ctypes.c_int)]


class Pauli(ctypes.Structure):
    _fields_ = [("nq", ctypes.c_int), ("qubits", ctypes.POINTER(ctypes.c_int)),
                ("paulis", ctypes.c_char_p)]


_lib = None


def lib() -> ctypes.CDLL:
    """Load libqtraj.so (built by __graft_entry__.build()); raises if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not found: run __graft_entry__.build() (no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    vp, ip, dp = ctypes.c_void_p, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_double)
    sig = {
        "qt_ctx_create": ([ctypes.c_int, vp, ctypes.POINTER(vp)], ctypes.c_int),
        "qt_ctx_destroy": ([vp], None),
        "qt_ctx_set_stream": ([vp, vp], ctypes.c_int),
        "qt_circuit_create": ([ctypes.c_int, ctypes.POINTER(vp)], ctypes.c_int),
        "qt_circuit_destroy": ([vp], None),
        "qt_add_gate": ([vp, ctypes.c_int, ctypes.c_int, ip, dp], ctypes.c_int),
        "qt_add_channel": ([vp, ctypes.c_int, ctypes.c_int, ip, ctypes.c_int, dp, ctypes.c_int], ctypes.c_int),
        "qt_set_readout": ([vp, dp, dp], ctypes.c_int),
        "qt_circuit_num_recorded": ([vp], ctypes.c_int),
        "qt_add_gate_sweep": ([vp, ctypes.c_int, ctypes.c_int, ip, ctypes.c_int, dp], ctypes.c_int),
        "qt_readout_flips": ([ctypes.c_int, dp, dp, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, ip,
                              ctypes.POINTER(ctypes.c_uint64)], ctypes.c_int),
        "qt_circuit_num_sets": ([vp], ctypes.c_int),
        "qt_rank_sample": ([ctypes.c_int, dp, ctypes.c_int, ctypes.c_int, ip, ctypes.c_uint64, ctypes.c_uint64,
                            ctypes.c_int, ip, ctypes.POINTER(ctypes.c_uint64), ip], ctypes.c_int),
        "qt_restrict_diagonal": ([ctypes.c_int, dp, ip, dp, ip], ctypes.c_int),
        "qt_embed_rho_diagonal": ([ctypes.c_int, ip, ctypes.c_int, dp, dp], ctypes.c_int),
        "qt_channel_operator": ([ctypes.c_int, ctypes.c_int, dp, ctypes.c_int, ctypes.c_double, dp], ctypes.c_int),
        "qt_circuit_num_channels": ([vp], ctypes.c_int),
        "qt_fuse": ([vp, ctypes.c_int, ctypes.POINTER(vp)], ctypes.c_int),
        "qt_fuse_ex": ([vp, ctypes.POINTER(FuseOpts), ctypes.POINTER(vp)], ctypes.c_int),
        "qt_plan_destroy": ([vp], None),
        "qt_run_trajectories": ([vp, vp, ctypes.POINTER(RunOpts), ctypes.c_int, ctypes.POINTER(Pauli),
                                 vp, ctypes.c_size_t, vp, vp, vp, ctypes.POINTER(Stats)], ctypes.c_int),
        "qt_apply_gate": ([vp, vp, ctypes.c_int, ctypes.c_int, ip, dp], ctypes.c_int),
        "qt_apply_gate_ex": ([vp, vp, ctypes.c_int, ctypes.c_int, ip, dp, ctypes.c_int, dp], ctypes.c_int),
        "qt_sample_bitstrings": ([vp, vp, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, vp],
                                 ctypes.c_int),
        "qt_expectation_value": ([vp, vp, ctypes.c_int, ctypes.c_int, ctypes.POINTER(Pauli), dp], ctypes.c_int),
        "qt_kraus_lower_bound": ([ctypes.c_int, dp], ctypes.c_double),
        "qt_add_matrix": ([vp, ctypes.c_int, ctypes.c_int, ip, dp], ctypes.c_int),
        "qt_permute_qubits": ([vp, vp, vp, ctypes.c_int, ip], ctypes.c_int),
        "qt_draw": ([ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int],
                    ctypes.c_double),
        "qt_channel_first_loop": ([ctypes.c_int, ctypes.c_int, dp, ctypes.c_double, ctypes.c_int, ip, dp, dp],
                                  ctypes.c_int),
        "qt_channel_choose": ([ctypes.c_int, ctypes.c_int, dp, ip, dp, ctypes.c_double, ctypes.c_int, ip, dp],
                              ctypes.c_int),
        "qt_apply_plan": ([vp, vp, vp, ctypes.c_size_t], ctypes.c_int),
        "qt_reduce_rho": ([vp, vp, ctypes.c_int, ctypes.c_int, ip, dp], ctypes.c_int),
        "qt_sample_local": ([vp, vp, ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int,
                             vp, vp], ctypes.c_int),
        "qt_expectation_partials": ([vp, vp, ctypes.c_int, ctypes.c_int, ctypes.POINTER(Pauli), dp, dp],
                                    ctypes.c_int),
        "qt_plan_info": ([vp, ctypes.c_uint64, ctypes.c_uint64, ctypes.POINTER(ctypes.c_int64)], ctypes.c_int),
        "qt_last_error": ([], ctypes.c_char_p),
        "qt_version": ([], ctypes.c_char_p),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _lib = L
    return L


def _check(st: int):
    if st != 0:
        raise QtError(st, lib().qt_last_error().decode())


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _iptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int))


def _cplx(m) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(m, dtype=np.complex128)).view(np.float64).reshape(-1)


class Circuit:
    """Owning handle of a qt_circuit."""

    def __init__(self, n_qubits: int):
        h = ctypes.c_void_p()
        _check(lib().qt_circuit_create(n_qubits, ctypes.byref(h)))
        self.h = h
        self.n = n_qubits

    def add_gate(self, moment: int, qubits: Sequence[int], U) -> None:
        q = np.asarray(qubits, np.int32)
        m = _cplx(U)
        _check(lib().qt_add_gate(self.h, moment, len(q), _iptr(q), _dptr(m)))

    def add_gate_sweep(self, moment: int, qubits: Sequence[int], Us: Iterable) -> None:
        """Parametrized gate: one unitary per parameter set; trajectory t
        applies Us[t mod n_sets]."""
        q = np.asarray(qubits, np.int32)
        ms = list(Us)
        m = np.concatenate([_cplx(u) for u in ms])
        _check(lib().qt_add_gate_sweep(self.h, moment, len(q), _iptr(q), len(ms), _dptr(m)))

    def add_matrix(self, moment: int, qubits: Sequence[int], M) -> None:
        """A general (e.g. non-unitary Kraus) operator; no unitarity check."""
        q = np.asarray(qubits, np.int32)
        m = _cplx(M)
        _check(lib().qt_add_matrix(self.h, moment, len(q), _iptr(q), _dptr(m)))

    def add_measurement(self, moment: int, qubits: Sequence[int]) -> None:
        """Mid-circuit computational-basis measurement (one keyed projector channel per
        qubit: always the conventional branch of Alg. 2; records = outcomes)."""
        P0 = np.array([[1, 0], [0, 0]], dtype=np.complex128)
        P1 = np.array([[0, 0], [0, 1]], dtype=np.complex128)
        for q in qubits:
            self.add_channel(moment, [q], [P0, P1], True)

    def add_channel(self, moment: int, qubits: Sequence[int], kraus: Iterable, record: bool = True) -> None:
        q = np.asarray(qubits, np.int32)
        ks = list(kraus)
        m = np.concatenate([_cplx(k) for k in ks])
        _check(lib().qt_add_channel(self.h, moment, len(q), _iptr(q), len(ks), _dptr(m), int(bool(record))))

    def set_readout(self, p00=None, p11=None) -> None:
        a = None if p00 is None else np.ascontiguousarray(p00, np.float64)
        b = None if p11 is None else np.ascontiguousarray(p11, np.float64)
        _check(lib().qt_set_readout(self.h, None if a is None else _dptr(a), None if b is None else _dptr(b)))
        self._keep = (a, b)

    @property
    def num_recorded(self) -> int:
        return lib().qt_circuit_num_recorded(self.h)

    @property
    def num_channels(self) -> int:
        return lib().qt_circuit_num_channels(self.h)

    @property
    def num_sets(self) -> int:
        return lib().qt_circuit_num_sets(self.h)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.qt_circuit_destroy(self.h)
            self.h = None

    @classmethod
    def from_description(cls, desc) -> "Circuit":
        """Upload any object with n_qubits, moments (ops with .qubits and .matrix or
        .kraus [.record]), optional p00/p11 (e.g. workloads.Circuit)."""
        c = cls(desc.n_qubits)
        for mi, moment in enumerate(desc.moments):
            for op in moment:
                if hasattr(op, "kraus"):
                    c.add_channel(mi, op.qubits, op.kraus, getattr(op, "record", True))
                elif hasattr(op, "matrices"):
                    c.add_gate_sweep(mi, op.qubits, op.matrices)
                else:
                    c.add_gate(mi, op.qubits, op.matrix)
        if getattr(desc, "p00", None) is not None or getattr(desc, "p11", None) is not None:
            c.set_readout(desc.p00, desc.p11)
        return c


class Plan:
    """Owning handle of a qt_plan (the paper's fuser, Sec. III.B)."""

    def __init__(self, circuit: Circuit, max_fused: int = 4, tile_bits: int = 0, low_bits: int = 0,
                 one_gate_per_pass: bool = False, tensor_cores: int = 0):
        h = ctypes.c_void_p()
        o = FuseOpts(max_fused, tile_bits, low_bits, int(one_gate_per_pass), int(tensor_cores))
        _check(lib().qt_fuse_ex(circuit.h, ctypes.byref(o), ctypes.byref(h)))
        self.h = h
        self.n = circuit.n
        self.num_recorded = circuit.num_recorded
        self.num_channels = circuit.num_channels

    def info(self, seed: int, traj: int) -> dict:
        """Host-only planning of one trajectory: pass / gate / event counts."""
        out = (ctypes.c_int64 * 10)()
        _check(lib().qt_plan_info(self.h, seed, traj, out))
        keys = ["passes", "fused_gates", "events", "deferred", "conventional", "pool", "alg_bytes", "constituents",
                "tile_bits", "kernel"]
        return dict(zip(keys, list(out)))

    def plan_seconds(self, seed: int, traj0: int, count: int) -> float:
        """Host planning cost (diagnostic qt_plan_bench): seconds to plan trajectories
        traj0 .. traj0 + count - 1 on one thread into one reused program."""
        sec = ctypes.c_double()
        _check(lib().qt_plan_bench(self.h, ctypes.c_uint64(seed), ctypes.c_uint64(traj0), int(count),
                                   ctypes.byref(sec)))
        return sec.value

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.qt_plan_destroy(self.h)
            self.h = None


def _pauli_array(observables: Sequence[str]):
    """'IXYZ' strings, char q acting on qubit q."""
    arr = (Pauli * max(len(observables), 1))()
    keep = []
    for k, s in enumerate(observables):
        qs = [q for q, ch in enumerate(s) if ch != "I"]
        ps = "".join(s[q] for q in qs).encode()
        qa = np.asarray(qs, np.int32)
        keep.append((qa, ps))
        arr[k].nq = len(qs)
        arr[k].qubits = _iptr(qa)
        arr[k].paulis = ps
    return arr, keep


class Context:
    """Owning handle of a qt_ctx bound to a CUDA device and stream."""

    def __init__(self, device: int = 0, stream=None):
        import torch
        if stream is None:
            stream = torch.cuda.current_stream(device)
        h = ctypes.c_void_p()
        _check(lib().qt_ctx_create(device, ctypes.c_void_p(stream.cuda_stream), ctypes.byref(h)))
        self.h = h
        self.device = device
        self.stream = stream

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.qt_ctx_destroy(self.h)
            self.h = None

    # ---- Alg. 2 trajectories ------------------------------------------------
    def run_trajectories(self, plan: Plan, state, seed: int, traj_count: int, traj_begin: int = 0,
                         traj_stride: int = 1, shots: int = 1, batch: int = 0,
                         observables: Sequence[str] = (), profile: bool = False,
                         host_threads: int = 0, want_kraus: bool = True, mode: int = 0) -> dict:
        """state: torch complex64 CUDA tensor with >= 2^n elements per slot."""
        import torch
        assert state.is_cuda and state.dtype == torch.complex64 and state.is_contiguous()
        o = RunOpts(seed, traj_begin, traj_stride, traj_count, shots, batch, mode, int(profile), host_threads)
        bits = np.zeros((traj_count, max(shots, 0)), np.uint64)
        kraus = np.zeros((traj_count, plan.num_recorded), np.int32) if want_kraus else None
        obs = np.zeros((traj_count, len(observables)), np.float64)
        parr, keep = _pauli_array(observables)
        st = Stats()
        _check(lib().qt_run_trajectories(
            self.h, plan.h, ctypes.byref(o), len(observables), parr,
            ctypes.c_void_p(state.data_ptr()), state.numel() * 8,
            bits.ctypes.data if shots > 0 else None,
            kraus.ctypes.data if (kraus is not None and kraus.size) else None,
            obs.ctypes.data if len(observables) else None, ctypes.byref(st)))
        del keep
        return {"bits": bits, "kraus": kraus, "obs": obs, "stats": st.as_dict()}

    # ---- stand-alone state operations ---------------------------------------
    def apply_gate(self, state, qubits: Sequence[int], U, repeats: int = 1) -> Optional[float]:
        n = int(np.log2(state.numel()))
        q = np.asarray(qubits, np.int32)
        m = _cplx(U)
        ms = ctypes.c_double(0.0)
        _check(lib().qt_apply_gate_ex(self.h, ctypes.c_void_p(state.data_ptr()), n, len(q), _iptr(q), _dptr(m),
                                      repeats, ctypes.byref(ms)))
        return ms.value

    def sample_bitstrings(self, state, seed: int, traj: int, shots: int) -> np.ndarray:
        n = int(np.log2(state.numel()))
        out = np.zeros(shots, np.uint64)
        _check(lib().qt_sample_bitstrings(self.h, ctypes.c_void_p(state.data_ptr()), n, seed, traj, shots,
                                          out.ctypes.data))
        return out

    # ---- distributed-state building blocks ------------------------------------
    def permute_qubits(self, src, dst, perm: Sequence[int]) -> None:
        """dst[pi(i)] = src[i], bit b of i moved to bit perm[b]."""
        n = int(np.log2(src.numel()))
        p = np.asarray(perm, np.int32)
        _check(lib().qt_permute_qubits(self.h, ctypes.c_void_p(src.data_ptr()), ctypes.c_void_p(dst.data_ptr()), n,
                                       _iptr(p)))

    def apply_plan(self, plan: Plan, state) -> None:
        _check(lib().qt_apply_plan(self.h, plan.h, ctypes.c_void_p(state.data_ptr()), state.numel() * 8))

    def reduce_rho(self, state, qubits: Sequence[int]) -> np.ndarray:
        """rho_Q in internal order (bit m <-> m-th lowest listed qubit), fp64."""
        n = int(np.log2(state.numel()))
        q = np.asarray(qubits, np.int32)
        d = 1 << len(q)
        out = np.zeros(2 * d * d, np.float64)
        _check(lib().qt_reduce_rho(self.h, ctypes.c_void_p(state.data_ptr()), n, len(q), _iptr(q), _dptr(out)))
        return out.view(np.complex128).reshape(d, d)

    def sample_local(self, state, n_total: int, seed: int, traj: int, shot_ids: Sequence[int]) -> np.ndarray:
        n = int(np.log2(state.numel()))
        ids = np.ascontiguousarray(shot_ids, np.int32)
        out = np.zeros(len(ids), np.uint64)
        _check(lib().qt_sample_local(self.h, ctypes.c_void_p(state.data_ptr()), n, n_total, seed, traj, len(ids),
                                     ids.ctypes.data if len(ids) else None, out.ctypes.data if len(ids) else None))
        return out

    def expectation_partials(self, state, observables: Sequence[str]):
        n = int(np.log2(state.numel()))
        out = np.zeros(max(len(observables), 1), np.float64)
        norm = np.zeros(1, np.float64)
        parr, keep = _pauli_array(observables)
        _check(lib().qt_expectation_partials(self.h, ctypes.c_void_p(state.data_ptr()), n, len(observables), parr,
                                             _dptr(out), _dptr(norm)))
        del keep
        return out[: len(observables)], float(norm[0])

    def expectation_value(self, state, observables: Sequence[str]) -> np.ndarray:
        n = int(np.log2(state.numel()))
        out = np.zeros(len(observables), np.float64)
        parr, keep = _pauli_array(observables)
        _check(lib().qt_expectation_value(self.h, ctypes.c_void_p(state.data_ptr()), n, len(observables), parr,
                                          _dptr(out)))
        del keep
        return out


PURPOSE_CHANNEL, PURPOSE_SAMPLE, PURPOSE_READOUT = 1, 2, 3


def draw(seed: int, ordinal: int, purpose: int, traj: int, half: int = 0) -> float:
    """The RNG contract's uniform (Philox4x32-10, qtraj.h)."""
    return lib().qt_draw(seed, ordinal, purpose, traj, half)


def readout_flips(bits: np.ndarray, n: int, p00, p11, seed: int, traj: int, shot_ids=None) -> np.ndarray:
    """Readout error on recorded bitstrings (qt_readout_flips); returns a copy."""
    out = np.ascontiguousarray(bits, dtype=np.uint64).copy()
    ids = np.arange(len(out), dtype=np.int32) if shot_ids is None else np.ascontiguousarray(shot_ids, np.int32)
    a = None if p00 is None else np.ascontiguousarray(p00, np.float64)
    b = None if p11 is None else np.ascontiguousarray(p11, np.float64)
    _check(lib().qt_readout_flips(n, None if a is None else _dptr(a), None if b is None else _dptr(b), seed, traj,
                                  len(out), _iptr(ids), out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))))
    return out


def rank_sample(rank_mass, n_total: int, n_local: int, level_rank_bit, seed: int, traj: int, shot_ids):
    """Chain rule over the rank bits (qt_rank_sample): (prefix bits, owner rank) per shot."""
    m = np.ascontiguousarray(rank_mass, np.float64)
    lv = np.ascontiguousarray(level_rank_bit, np.int32)
    ids = np.ascontiguousarray(shot_ids, np.int32)
    pre = np.zeros(len(ids), np.uint64)
    own = np.zeros(len(ids), np.int32)
    _check(lib().qt_rank_sample(len(m), _dptr(m), n_total, n_local, _iptr(lv), seed, traj, len(ids), _iptr(ids),
                                pre.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), _iptr(own)))
    return pre, own


def restrict_diagonal(diag, fixed):
    """Diagonal operator restricted to one rank's global-qubit values (qt_restrict_diagonal):
    the diagonal over the local listed qubits (empty shape () -> a scalar)."""
    d = np.ascontiguousarray(np.asarray(diag, np.complex128)).view(np.float64)
    fx = np.ascontiguousarray(fixed, np.int32)
    out = np.zeros(2 * len(d) // 2, np.float64)
    k = ctypes.c_int(0)
    _check(lib().qt_restrict_diagonal(len(fx), _dptr(d), _iptr(fx), _dptr(out), ctypes.byref(k)))
    return out.view(np.complex128)[: 1 << k.value], k.value


def embed_rho_diagonal(global_bit, diag_local):
    """rho_Q of a diagonal-K^dag K channel from a rank's local diagonal (qt_embed_rho_diagonal)."""
    gb = np.ascontiguousarray(global_bit, np.int32)
    dl = np.ascontiguousarray(np.real(np.asarray(diag_local)), np.float64).reshape(-1)
    nq = len(gb)
    out = np.zeros(2 << (2 * nq), np.float64)
    _check(lib().qt_embed_rho_diagonal(nq, _iptr(gb), int((gb < 0).sum()), _dptr(dl), _dptr(out)))
    d = 1 << nq
    return out.view(np.complex128).reshape(d, d)


def channel_operator(kraus, pick: int, scale: float) -> np.ndarray:
    """K_pick * scale (qt_channel_operator)."""
    ks = list(kraus)
    nq = int(np.log2(np.asarray(ks[0]).shape[0]))
    m = np.concatenate([_cplx(k) for k in ks])
    out = np.zeros(2 << (2 * nq), np.float64)
    _check(lib().qt_channel_operator(nq, len(ks), _dptr(m), pick, scale, _dptr(out)))
    d = 1 << nq
    return out.view(np.complex128).reshape(d, d)


def channel_first_loop(kraus, u: float, mode: int = 0):
    """Alg. 2 lines 2-11: (pick or -1, remaining r, deferred scale)."""
    ks = list(kraus)
    nq = int(np.log2(np.asarray(ks[0]).shape[0]))
    m = np.concatenate([_cplx(k) for k in ks])
    pick = ctypes.c_int(-1)
    r = ctypes.c_double(0.0)
    sc = ctypes.c_double(1.0)
    _check(lib().qt_channel_first_loop(nq, len(ks), _dptr(m), u, mode, ctypes.byref(pick), ctypes.byref(r),
                                       ctypes.byref(sc)))
    return pick.value, r.value, sc.value


def channel_choose(kraus, positions: Sequence[int], rho: np.ndarray, r: float, mode: int = 0):
    """Alg. 2 lines 13-21 from rho over the channel's qubit positions:
    (pick, 1/sqrt(raw p_pick))."""
    ks = list(kraus)
    nq = len(positions)
    m = np.concatenate([_cplx(k) for k in ks])
    q = np.asarray(positions, np.int32)
    rr = np.ascontiguousarray(np.asarray(rho, np.complex128)).view(np.float64).reshape(-1)
    pick = ctypes.c_int(-1)
    sc = ctypes.c_double(1.0)
    _check(lib().qt_channel_choose(nq, len(ks), _dptr(m), _iptr(q), _dptr(rr), r, mode, ctypes.byref(pick),
                                   ctypes.byref(sc)))
    return pick.value, sc.value


def kraus_lower_bound(K) -> float:
    K = np.asarray(K, np.complex128)
    m = _cplx(K)
    return lib().qt_kraus_lower_bound(K.shape[0], _dptr(m))
