"""Distributed-state mode (second mode of the north star): one
trajectory of an n-qubit register whose state vector is split over G = 2^g
ranks (global index = rank << n_local | local index), for registers above one
GPU's capacity (config 5: 36 qubits on 8 x B200).

Mechanics (not in the paper, which has no distributed state; P:336 only mentions
36-qubit TPU runs):
  * a qubit map places every logical qubit either in a local slot (amplitude
    index bit < n_local) or a global slot (a rank bit);
  * consecutive operations on local qubits are buffered and applied by one
    fused plan (the library's fuser + K1 tile passes) on every rank;
  * an operation that touches global qubits first swaps them with local
    "victim" qubits: a local bit permutation (qt_permute_qubits) moves the
    victims to the top local bits, then an all-to-all (NCCL over NVLink, or
    gloo in the CPU tests) exchanges the 2^s chunks -- the classic global-qubit
    swap; victims are the local qubits used farthest in the future (Belady);
  * channels follow Alg. 2 exactly as in the single-GPU path: the first loop
    (qt_channel_first_loop) defers picks into the buffered operations; a
    conventional channel flushes, reduces rho_Q on every rank (qt_reduce_rho),
    all-reduces it (fp64) and walks lines 13-21 (qt_channel_choose) on identical
    data on every rank, so every rank takes the same branch;
  * terminal sampling: chain rule over the rank bits from all-gathered rank
    masses, then the owning rank samples the local levels (qt_sample_local,
    RNG ordinals of the whole register); Z-type observables from per-rank
    partial sums.
Results are identical to the single-state simulation (same draws, same
decisions) up to fp32 rounding; tests compare against the CPU oracle.

All per-rank arithmetic runs in libqtraj (the `GpuBackend`); this module only
orchestrates.  The collective layer is a `Fabric`: `TorchFabric` (one rank per
process, torch.distributed) or `EmulatedFabric` (all ranks in one process, for
single-GPU tests; NCCL cannot place two ranks on one GPU).
"""
from __future__ import annotations

from typing import Dict, List, Optional, Sequence

import os

import numpy as np

from . import qtraj

PURPOSE_CHANNEL, PURPOSE_SAMPLE = 1, 2


# ---------------------------------------------------------------------------
# Backends: per-rank state storage + device operations
# ---------------------------------------------------------------------------
class GpuBackend:
    """Per-rank states as complex64 CUDA tensors; all operations in libqtraj."""

    def __init__(self, ctx: "qtraj.Context", device, max_fused: int = 4):
        import torch
        self.torch = torch
        self.ctx = ctx
        self.device = device
        self.max_fused = max_fused

    def new_state(self, n_local: int, rank: int):
        s = self.torch.zeros(1 << n_local, dtype=self.torch.complex64, device=self.device)
        if rank == 0:
            s[0] = 1.0
        return s

    def apply_ops(self, state, n_local: int, ops):
        # the chunks of one exchange share their operation list: one plan for all of them
        key = (id(ops), n_local)
        if getattr(self, "_plan_key", None) != key:
            c = qtraj.Circuit(n_local)
            for i, (pos, M) in enumerate(ops):
                c.add_matrix(i, pos, M)
            self._plan = qtraj.Plan(c, max_fused=max(self.max_fused, max(len(p) for p, _ in ops)))
            self._plan_key = key
            self._plan_ops = ops  # keeps id(ops) from being reused while cached
        self.ctx.apply_plan(self._plan, state)

    def permute(self, state, perm):
        # ping-pong with one spare buffer per size: a 33-qubit slice (64 GiB)
        # and its spare fit in one B200's 180 GB
        spare = getattr(self, "_spare", None)
        out = spare if (spare is not None and spare.numel() == state.numel()) else self.torch.empty_like(state)
        self.ctx.permute_qubits(state, out, perm)
        self._spare = state
        return out

    def take_spare(self, like):
        spare = getattr(self, "_spare", None)
        if spare is not None and spare.numel() == like.numel():
            self._spare = None
            return spare
        return self.torch.empty_like(like)

    def give_spare(self, t):
        self._spare = t

    def reduce_rho(self, state, positions):
        return self.ctx.reduce_rho(state, positions)

    def expect(self, state, observables: Sequence[str]):
        return self.ctx.expectation_partials(state, observables)

    def sample_local(self, state, n_total, seed, traj, shot_ids):
        return self.ctx.sample_local(state, n_total, seed, traj, shot_ids)


# ---------------------------------------------------------------------------
# Fabrics: the collectives over the rank slices of one register
# ---------------------------------------------------------------------------
def _dest(rank: int, gbits: Sequence[int], c: int) -> int:
    r = rank
    for j, b in enumerate(gbits):
        r = (r & ~(1 << b)) | (((c >> j) & 1) << b)
    return r


def _src_chunk(rank: int, gbits: Sequence[int]) -> int:
    return sum(((rank >> b) & 1) << j for j, b in enumerate(gbits))


class EmulatedFabric:
    """All G ranks in one process (single-GPU tests); exchanges are device copies."""

    def __init__(self, world: int):
        self.world = world
        self.local_ranks = list(range(world))

    def exchange_top(self, states: Dict[int, object], gbits: Sequence[int], s: int, pool=None, on_chunk=None):
        """Swap the top s local bits with global bits gbits (top local bit
        n_local - s + j <-> rank bit gbits[j]).  on_chunk(rank, view), if given, is
        called once per received chunk (a contiguous 2^(n_local - s) block)."""
        out = {}
        size = states[0].numel()
        chunk = size >> s
        for r in range(self.world):
            out[r] = states[r].clone()
        for r in range(self.world):
            for c in range(1 << s):
                d = _dest(r, gbits, c)
                cp = _src_chunk(r, gbits)
                out[d][cp * chunk:(cp + 1) * chunk].copy_(states[r][c * chunk:(c + 1) * chunk])
                if on_chunk is not None:
                    on_chunk(d, out[d][cp * chunk:(cp + 1) * chunk])
        return out

    def allreduce(self, per_rank: Dict[int, np.ndarray]) -> np.ndarray:
        tot = None
        for r in self.local_ranks:
            tot = per_rank[r].copy() if tot is None else tot + per_rank[r]
        return tot

    def allgather(self, per_rank: Dict[int, float]) -> np.ndarray:
        return np.array([per_rank[r] for r in range(self.world)], np.float64)

    def broadcast_u64(self, arr: np.ndarray, owner: int) -> np.ndarray:
        return arr


class TorchFabric:
    """One rank per process over a torch.distributed process group (NCCL on
    NVLink for CUDA tensors, gloo for CPU tensors)."""

    def __init__(self, group=None, device=None):
        import torch
        import torch.distributed as dist
        self.torch = torch
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.local_ranks = [self.rank]
        self.device = device
        # gloo moves CPU tensors only: CUDA states are staged through the host (the
        # 2-process single-GPU test; NCCL moves device memory directly over NVLink)
        self.stage_host = dist.get_backend(group) == "gloo"

    def exchange_top(self, states, gbits, s, pool=None, on_chunk=None):
        # chunk c goes to rank _dest(c) and arrives at chunk _src_chunk(source):
        # both are increasing in rank order only for ascending gbits
        assert all(gbits[j] < gbits[j + 1] for j in range(len(gbits) - 1)), "gbits must ascend"
        if on_chunk is not None:
            return self._exchange_p2p(states, gbits, s, pool, on_chunk)
        x = states[self.rank]
        chunk = x.numel() >> s
        in_split = [0] * self.world
        out_split = [0] * self.world
        for c in range(1 << s):
            in_split[_dest(self.rank, gbits, c)] = chunk
        # the sources of this rank are the ranks that differ from it only in gbits
        for c in range(1 << s):
            out_split[_dest(self.rank, gbits, c)] = chunk
        # receive into the backend's spare buffer; the sent buffer becomes the spare
        y = pool.take_spare(x) if hasattr(pool, "take_spare") else self.torch.empty_like(x)
        if self.stage_host and x.is_cuda:
            xc = x.contiguous().cpu()
            yc = self.torch.empty_like(xc)
            self.dist.all_to_all_single(yc, xc, out_split, in_split, group=self.group)
            y.copy_(yc)
        else:
            self.dist.all_to_all_single(y, x.contiguous(), out_split, in_split, group=self.group)
        if hasattr(pool, "give_spare"):
            pool.give_spare(x)
        return {self.rank: y}

    def _exchange_p2p(self, states, gbits, s, pool, on_chunk):
        """The exchange as 2^s - 1 pairwise rounds (round k: the peer whose global-bit
        value is this rank's XOR k, so partners agree round by round; each round one
        grouped send + receive), the chunk of round k handed to on_chunk (the deferred
        local operations) while round k + 1 is in flight; the rank's own chunk first,
        without communication."""
        x = states[self.rank].contiguous()
        chunk = x.numel() >> s
        y = pool.take_spare(x) if hasattr(pool, "take_spare") else self.torch.empty_like(x)
        staged = self.stage_host and x.is_cuda
        xs = x.cpu() if staged else x
        ys = self.torch.empty_like(xs) if staged else y
        own = _src_chunk(self.rank, gbits)

        def hand(cp):
            if staged:
                y[cp * chunk:(cp + 1) * chunk].copy_(ys[cp * chunk:(cp + 1) * chunk])
            on_chunk(self.rank, y[cp * chunk:(cp + 1) * chunk])

        ys[own * chunk:(own + 1) * chunk].copy_(xs[own * chunk:(own + 1) * chunk])
        prev = None
        for k in range(1, 1 << s):
            c = own ^ k                       # the chunk that goes to this round's peer
            peer = _dest(self.rank, gbits, c)
            cp = _src_chunk(peer, gbits)      # where the peer's chunk lands (= c)
            works = self.dist.batch_isend_irecv([
                self.dist.P2POp(self.dist.isend, xs[c * chunk:(c + 1) * chunk], peer, self.group),
                self.dist.P2POp(self.dist.irecv, ys[cp * chunk:(cp + 1) * chunk], peer, self.group)])
            if prev is None:
                hand(own)  # overlaps the first round
            else:
                for w in prev[0]:
                    w.wait()
                hand(prev[1])
            prev = (works, cp)
        if prev is None:
            hand(own)
        else:
            for w in prev[0]:
                w.wait()
            hand(prev[1])
        if hasattr(pool, "give_spare"):
            pool.give_spare(x)
        return {self.rank: y}

    def _dev(self):
        return self.device if self.device is not None else "cpu"

    def allreduce(self, per_rank):
        a = np.ascontiguousarray(per_rank[self.rank])
        cplx = np.iscomplexobj(a)
        t = self.torch.from_numpy(a.view(np.float64) if cplx else a.astype(np.float64)).to(self._dev())
        self.dist.all_reduce(t, group=self.group)
        out = t.cpu().numpy()
        return out.view(np.complex128).reshape(a.shape) if cplx else out.reshape(a.shape)

    def allgather(self, per_rank):
        t = self.torch.tensor([float(per_rank[self.rank])], dtype=self.torch.float64, device=self._dev())
        bufs = [self.torch.zeros_like(t) for _ in range(self.world)]
        self.dist.all_gather(bufs, t, group=self.group)
        return np.array([b.item() for b in bufs], np.float64)

    def broadcast_u64(self, arr: np.ndarray, owner: int) -> np.ndarray:
        t = self.torch.from_numpy(np.ascontiguousarray(arr).view(np.int64)).to(self._dev())
        self.dist.broadcast(t, src=owner, group=self.group)
        return t.cpu().numpy().view(np.uint64)


# ---------------------------------------------------------------------------
# The distributed trajectory
# ---------------------------------------------------------------------------
def _is_identity(M) -> bool:
    M = np.asarray(M)
    return np.max(np.abs(M - np.eye(M.shape[0]))) < 1e-15


def _is_diag(M) -> bool:
    M = np.asarray(M)
    return not np.any(M - np.diag(np.diag(M)))


class DistributedTrajectory:
    def __init__(self, backend, fabric, n_total: int, mode: int = 0):
        world = fabric.world
        g = world.bit_length() - 1
        if (1 << g) != world:
            raise ValueError("world size must be a power of two")
        if n_total - g < 6:
            raise ValueError("need at least 6 local qubits per rank")
        self.b = backend
        self.f = fabric
        self.n = n_total
        self.g = g
        self.nl = n_total - g
        self.mode = mode
        self.slot = list(range(n_total))          # logical qubit -> physical slot
        self.states = {r: backend.new_state(self.nl, r) for r in fabric.local_ranks}
        self.pending: List = []        # shared local operations (since the last flush)
        self.pending_all: List = []    # (rank or -1 = every rank, positions, matrix), program order
        self.rank_ops = {r: [] for r in fabric.local_ranks}
        self.swaps = 0
        self.exchanged_bytes = 0
        # pending local operations that commute with a swap run per received chunk
        self.overlap = os.environ.get("QT_DIST_OVERLAP", "1") != "0"
        self.deferred_ops = 0

    # -- helpers ------------------------------------------------------------
    def _flush(self):
        if not self.pending and not any(self.rank_ops.values()):
            return
        for r in self.f.local_ranks:
            # shared ops and this rank's diagonal restrictions, in program order
            ops = [o for o in self.pending_all if o[0] == -1 or o[0] == r]
            if ops:
                self.b.apply_ops(self.states[r], self.nl, [(p, M) for _, p, M in ops])
        self.pending = []
        self.pending_all = []
        self.rank_ops = {r: [] for r in self.f.local_ranks}

    def _split_pending(self, vslots: set) -> List:
        """Remove from the pending lists the shared operations that can follow the
        exchange and return them (positions, matrix) in program order: an operation must
        stay before it if it touches a victim slot, is rank-specific (its rank-independent
        marker keeps its slots), or shares a slot with a later operation that stays
        (reverse scan); the decision uses only state shared by every rank, because the
        deferred operations are applied to chunks that arrive from other ranks."""
        keep = [False] * len(self.pending_all)
        need = set(vslots)
        for i in range(len(self.pending_all) - 1, -1, -1):
            tag, pos, _ = self.pending_all[i]
            if tag >= 0:
                keep[i] = True  # rank-specific: decided by its marker, identically on every rank
            elif tag == -2 or any(p in need for p in pos):
                keep[i] = True
                need.update(pos)
        after = [(pos, M) for (tag, pos, M), k in zip(self.pending_all, keep) if not k]
        if after:
            self.pending_all = [o for o, k in zip(self.pending_all, keep) if k]
            self.pending = [(pos, M) for tag, pos, M in self.pending_all if tag == -1]
        return after

    def _push(self, pos, M):
        self.pending.append((pos, M))
        self.pending_all.append((-1, pos, M))

    def _push_diag_global(self, qubits, M):
        """A diagonal operator touching global qubits, applied without a swap:
        on rank r it is the diagonal restricted to r's values of the global
        qubits, i.e. an operator on the local qubits only (or a scalar)
        (qt_restrict_diagonal)."""
        d = np.diag(np.asarray(M, np.complex128))
        loc = [m for m, q in enumerate(qubits) if self.slot[q] < self.nl]
        # rank-independent marker (every rank records it): the slots a later exchange must
        # not defer past; the per-rank entries below differ between ranks
        self.pending_all.append((-2, [self.slot[qubits[m]] for m in loc], None))
        for r in self.f.local_ranks:
            fixed = [(r >> (self.slot[q] - self.nl)) & 1 if self.slot[q] >= self.nl else -1 for q in qubits]
            dd, k = qtraj.restrict_diagonal(d, fixed)
            if k == 0:  # a scalar on this rank
                if dd[0] != 1.0:
                    self.pending_all.append((r, [0], np.diag([dd[0], dd[0]])))
            elif not np.all(dd == 1.0):
                self.pending_all.append((r, [self.slot[qubits[m]] for m in loc], np.diag(dd)))
            self.rank_ops[r].append(1)

    def _apply_local_perm(self, perm_slot: Dict[int, int]):
        """Move local slot a -> perm_slot[a] (others fixed)."""
        perm = list(range(self.nl))
        for a, b in perm_slot.items():
            perm[a] = b
        if perm == list(range(self.nl)):
            return
        for r in self.f.local_ranks:
            self.states[r] = self.b.permute(self.states[r], perm)
        inv = {a: b for a, b in perm_slot.items()}
        for q in range(self.n):
            if self.slot[q] < self.nl:
                self.slot[q] = inv.get(self.slot[q], self.slot[q])

    def _choose_victims(self, s: int, keep: set, upcoming: List[set]) -> List[int]:
        """s local logical qubits not in `keep`, used farthest in the future (Belady)."""
        local_q = [q for q in range(self.n) if self.slot[q] < self.nl and q not in keep]

        def next_use(q):
            for i, ops in enumerate(upcoming):
                if q in ops:
                    return i
            return 1 << 30
        local_q.sort(key=lambda q: (-next_use(q), -self.slot[q]))
        return local_q[:s]

    def _swap_in(self, glob: List[int], victims: List[int]):
        """Exchange logical qubits `glob` (global) with `victims` (local)."""
        s = len(glob)
        assert len(victims) == s
        # pair j <-> rank bit gbits[j] in ascending order: the all-to-all then sends
        # chunk c to ranks in increasing order and receives chunks in source-rank
        # order (TorchFabric relies on it)
        pairs = sorted(zip(glob, victims), key=lambda gv: self.slot[gv[0]])
        glob = [g for g, _ in pairs]
        victims = [v for _, v in pairs]
        # pending operations that touch no victim (and precede no operation that must be
        # applied first) commute with the exchange: they are applied to every received
        # chunk, overlapping the transfers of the others; the rest is flushed now
        after = self._split_pending({self.slot[v] for v in victims}) if self.overlap else []
        self._flush()
        # local permutation: victim j -> top slot nl - s + j (swapping with the occupant)
        top = [self.nl - s + j for j in range(s)]
        occupant = {self.slot[q]: q for q in range(self.n) if self.slot[q] < self.nl}
        cur = {q: self.slot[q] for q in range(self.n)}
        for j, v in enumerate(victims):
            a, b = cur[v], top[j]
            if a == b:
                continue
            w = occupant[b]
            occupant[a], occupant[b] = w, v
            cur[v], cur[w] = b, a
        moved = {self.slot[q]: cur[q] for q in range(self.n) if self.slot[q] < self.nl and cur[q] != self.slot[q]}
        self._apply_local_perm(moved)
        gbits = [self.slot[q] - self.nl for q in glob]
        if after:
            # positions through the local permutation; none is a top (victim) slot
            ops = [([moved.get(p, p) for p in pos], M) for pos, M in after]
            assert all(p < self.nl - s for pos, _ in ops for p in pos)
            self.deferred_ops += len(ops)
            self.states = self.f.exchange_top(self.states, gbits, s, pool=self.b,
                                              on_chunk=lambda r, view: self.b.apply_ops(view, self.nl - s, ops))
        else:
            self.states = self.f.exchange_top(self.states, gbits, s, pool=self.b)
        self.swaps += 1
        self.exchanged_bytes += (1 - 2.0 ** -s) * 8 * (1 << self.nl) * len(self.f.local_ranks)
        for j, q in enumerate(glob):
            v = victims[j]
            self.slot[v] = self.nl + gbits[j]
            self.slot[q] = top[j]

    def _rho_diag_global(self, qubits: Sequence[int]):
        """Diagonal of rho_Q over qubits some of which are global: rank r holds
        the entries whose global bits equal r's (qt_embed_rho_diagonal).  Returns
        per-rank matrices in the internal order of the sorted slot positions, and
        those positions."""
        pos = [self.slot[q] for q in qubits]
        order = sorted(pos)
        loc = [p for p in order if p < self.nl]
        out = {}
        for rk in self.f.local_ranks:
            if loc:
                diag_l = np.real(np.diag(self.b.reduce_rho(self.states[rk], loc)))
            else:
                _, norm = self.b.expect(self.states[rk], [])
                diag_l = np.array([norm])
            gbits = [(rk >> (p - self.nl)) & 1 if p >= self.nl else -1 for p in order]
            out[rk] = qtraj.embed_rho_diagonal(gbits, diag_l)
        return out, pos

    def _pauli_values(self, strings: Sequence[str]) -> np.ndarray:
        """<P>/<psi|psi> of Pauli strings (char q = logical qubit q) whose X / Y
        qubits are all local in the current layout."""
        zvals = {}
        for rk in self.f.local_ranks:
            loc = []
            for s_ in strings:
                ls = ["I"] * self.nl
                for q in range(self.n):
                    if self.slot[q] < self.nl:
                        ls[self.slot[q]] = s_[q]
                    else:
                        assert s_[q] in "IZ", "X / Y qubits must be local"
                loc.append("".join(ls))
            vals, norm = self.b.expect(self.states[rk], loc)
            if not norm > 0.0:  # an empty slice (e.g. after amplitude damping): 0/0 partials
                vals = np.zeros(len(loc))
                norm = 0.0
            sg = []
            for s_ in strings:
                par = 0
                for q in range(self.n):
                    if self.slot[q] >= self.nl and s_[q] == "Z":
                        par ^= (rk >> (self.slot[q] - self.nl)) & 1
                sg.append(-1.0 if par else 1.0)
            zvals[rk] = np.asarray([sgn * v * norm for sgn, v in zip(sg, vals)] + [norm], np.float64)
        tot = self.f.allreduce(zvals)
        return tot[:-1] / tot[-1]

    def _ensure_local(self, qubits: Sequence[int], upcoming: List[set]):
        """Make `qubits` local.  The all-to-all of an s-qubit swap moves (1 - 2^-s) of
        the state, so other global qubits ride along when they are used (within the
        lookahead) before the local victim that would replace them (Belady): one
        3-qubit exchange (7/8 of the state) instead of three 1-qubit ones (3/2)."""
        glob = [q for q in qubits if self.slot[q] >= self.nl]
        if not glob:
            return

        def next_use(q):
            for i, ops in enumerate(upcoming):
                if q in ops:
                    return i
            return 1 << 30
        others = sorted((q for q in range(self.n) if self.slot[q] >= self.nl and q not in glob), key=next_use)
        victims = self._choose_victims(len(glob) + len(others), set(qubits), upcoming)
        take, vict = list(glob), victims[:len(glob)]
        for j, x in enumerate(others):
            k = len(glob) + j
            if k >= len(victims) or not next_use(x) < min(next_use(victims[k]), len(upcoming)):
                break
            take.append(x)
            vict.append(victims[k])
        self._swap_in(take, vict)

    # -- Alg. 2 over a distributed register ---------------------------------
    def run(self, circuit, seed: int, traj: int, shots: int = 1, observables: Sequence[str] = (),
            lookahead: int = 64):
        ops = list(circuit.ops())
        uses = [set(op.qubits) for op in ops]
        kraus_rec = []
        ch = 0
        for i, op in enumerate(ops):
            upcoming = uses[i + 1:i + 1 + lookahead]
            touches_global = any(self.slot[q] >= self.nl for q in op.qubits)
            if not hasattr(op, "kraus"):
                # sweep gates: parameter set traj mod n_sets, as in qt_run_trajectories
                mats = getattr(op, "matrices", None)
                M = np.asarray(mats[traj % len(mats)] if mats is not None else op.matrix, np.complex128)
                if touches_global and _is_diag(M):
                    self._push_diag_global(op.qubits, M)
                else:
                    self._ensure_local(op.qubits, upcoming)
                    self._push([self.slot[q] for q in op.qubits], M)
                continue
            u = qtraj.draw(seed, ch, PURPOSE_CHANNEL, traj, 0)
            pick, r, sc = qtraj.channel_first_loop(op.kraus, u, self.mode)
            if pick < 0:
                # conventional: Alg. 2 lines 13-21 on rho_Q of the unnormalized state
                self._flush()
                if touches_global and all(_is_diag(np.conj(np.asarray(K)).T @ np.asarray(K)) for K in op.kraus):
                    # every K_i^dag K_i diagonal: only the diagonal of rho_Q is needed,
                    # which each rank holds for its own global-bit values (no swap)
                    rho, pos = self._rho_diag_global(op.qubits)
                else:
                    self._ensure_local(op.qubits, upcoming)
                    pos = [self.slot[q] for q in op.qubits]
                    rho = {rk: self.b.reduce_rho(self.states[rk], pos) for rk in self.f.local_ranks}
                tot = self.f.allreduce(rho)
                pick, sc = qtraj.channel_choose(op.kraus, pos, tot, r, self.mode)
            M = qtraj.channel_operator(op.kraus, pick, sc)
            if not _is_identity(M):
                if any(self.slot[q] >= self.nl for q in op.qubits) and _is_diag(M):
                    self._push_diag_global(op.qubits, M)
                else:
                    self._ensure_local(op.qubits, upcoming)
                    self._push([self.slot[q] for q in op.qubits], M)
            if getattr(op, "record", True):  # keyed channels only, as qt_run_trajectories records them
                kraus_rec.append(pick)
            ch += 1
        self._flush()
        out = {"kraus": np.array(kraus_rec, np.int32)}
        # Pauli expectations: a string's X / Y qubits must be local (the operator is
        # then block-diagonal over the ranks; its global Z bits give a sign per
        # rank).  Strings that need no swap are evaluated together; the others
        # swap their X / Y qubits in first (one string at a time).
        if observables:
            vals = np.zeros(len(observables))
            ready = [i for i, s_ in enumerate(observables)
                     if all(self.slot[q] < self.nl for q in range(self.n) if s_[q] in "XY")]
            later = [i for i in range(len(observables)) if i not in ready]
            if ready:
                vals[ready] = self._pauli_values([observables[i] for i in ready])
            for i in later:
                xy = [q for q in range(self.n) if observables[i][q] in "XY"]
                if len(xy) > self.nl:
                    raise ValueError(f"distributed mode: a Pauli string needs at most {self.nl} X / Y qubits")
                self._ensure_local(xy, [])
                vals[i] = self._pauli_values([observables[i]])[0]
            out["obs"] = vals
        # layout for sampling: logical qubits >= nl global, local slot i = logical i
        high_local = [q for q in range(self.nl, self.n) if self.slot[q] < self.nl]
        low_global = [q for q in range(self.nl) if self.slot[q] >= self.nl]
        if low_global:
            self._swap_in(low_global, high_local)
        self._apply_local_perm({self.slot[q]: q for q in range(self.nl) if self.slot[q] != q})
        assert all(self.slot[q] == q for q in range(self.nl))
        out["swaps"] = self.swaps
        # rank masses for the chain rule over the rank bits
        masses = {}
        for rk in self.f.local_ranks:
            _, norm = self.b.expect(self.states[rk], [])
            masses[rk] = norm if norm > 0.0 else 0.0
        M = self.f.allgather(masses)
        # chain rule over the rank bits (levels n-1 .. nl; qt_rank_sample), then the
        # local levels on the owner
        level_bit = [self.slot[lvl] - self.nl for lvl in range(self.nl, self.n)]
        bits, owners = qtraj.rank_sample([M[r] for r in range(self.f.world)], self.n, self.nl, level_bit, seed, traj,
                                         np.arange(shots, dtype=np.int32))
        bits = bits.astype(np.uint64)
        for rk in self.f.local_ranks:
            ids = [sh for sh in range(shots) if owners[sh] == rk]
            if ids:
                low = self.b.sample_local(self.states[rk], self.n, seed, traj, ids)
                for sh, lb in zip(ids, low):
                    bits[sh] |= np.uint64(lb)
        for sh in range(shots):  # every rank ends with every shot's bits
            bits[sh:sh + 1] = self.f.broadcast_u64(bits[sh:sh + 1], int(owners[sh]))
        out["bits_raw"] = bits.copy()
        p00, p11 = getattr(circuit, "p00", None), getattr(circuit, "p11", None)
        if shots > 0 and (p00 is not None or p11 is not None):  # readout error, same draws on every rank
            bits = qtraj.readout_flips(bits, self.n, p00, p11, seed, traj)
        out["bits"] = bits
        out["masses"] = M
        return out
