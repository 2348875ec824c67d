"""Planner statistics of the persistent TMEM kernel (v2 layouts) on C2 trajectories,
from the undeclared diagnostic qt_plan_dump: passes (items), tensor-core gates,
segments (gathers), L / X transitions, and the modelled shared-memory wavefronts
per warp access of the segment gathers (fp32 tile -> registers) and write-backs:
lanes 0..4 of a warp differ in the tile bits of the layout's 5 lane roles, the
8-byte bank pair of a tile slot is linear in its bits under the T = 13 swizzle, so
a 32 x 8 B access is served per half-warp and takes 2 x 2^(4 - rank) wavefronts,
rank over lanes 0..3 (2 when those span all 16 bank pairs).  usage: python tools/v2_plan_stats.py [--traj 64]"""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads  # noqa: E402
from paper_2111_02396_b200 import qtraj  # noqa: E402

kGateTC, kGateRunStart, kGateV2, kGateRunEnd, kGateXNext, kGatePair0 = 0x100, 0x200, 0x800, 0x1000, 0x2000, 0x4000


def rank(vs):
    basis = []
    for v in vs:
        for b in basis:
            v = min(v, v ^ b)
        if v:
            basis.append(v)
    return len(basis)


def units_of(words):
    u = []
    for w in words:
        w &= (1 << 64) - 1
        for j in range(4):
            u.append((w >> (16 * j)) & 0xFFFF)
    return u


def dump(plan, seed, traj):
    cap = 1 << 16
    out = (ctypes.c_int64 * cap)()
    qtraj._check(qtraj.lib().qt_plan_dump(plan.h, ctypes.c_uint64(seed), ctypes.c_uint64(traj), out, ctypes.c_int64(cap)))
    v = list(out)
    i = 1
    passes = []
    for _ in range(v[0]):
        tm, fl, gc = v[i], v[i + 1], v[i + 2]
        i += 3
        gates = []
        for _g in range(gc):
            gates.append((v[i], v[i + 1], units_of(v[i + 2:i + 7])))
            i += 7
        passes.append((tm, fl, gates))
    return passes


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--traj", type=int, default=64)
    ap.add_argument("--fuse", type=int, default=4)
    a = ap.parse_args()
    c = workloads.sycamore_grid_qcs(config=2)
    plan = qtraj.Plan(qtraj.Circuit.from_description(c), max_fused=a.fuse)
    seed = workloads.trajectory_seed(2)
    st = dict(items=0, tc=0, cc=0, seg=0, L=0, X=0, gwf=0, wwf=0, seg_len=[])
    hist_g, hist_w = {}, {}
    for t in range(a.traj):
        for tm, fl, gates in dump(plan, seed, t):
            st["items"] += 1
            run = 0
            for m, k, u in gates:
                if not (k & kGateTC):
                    st["cc"] += 1
                    continue
                st["tc"] += 1
                run += 1
                # 8-byte accesses are served per half-warp: lanes 0..3 must span the 16 bank
                # pairs; 16-byte pair accesses (kGatePair0) per quarter warp: lanes 0..2 the
                # 8 chunks (wavefronts per 8 bytes)
                if k & kGatePair0:
                    wf = 2 * 2 ** (3 - rank([(x >> 4) & 7 for x in u[6:9]]))
                else:
                    wf = 2 * 2 ** (4 - rank([(x >> 3) & 15 for x in u[6:10]]))
                if k & kGateRunStart:
                    st["seg"] += 1
                    st["gwf"] += wf
                    hist_g[wf] = hist_g.get(wf, 0) + 1
                if k & kGateRunEnd:
                    st["wwf"] += wf
                    hist_w[wf] = hist_w.get(wf, 0) + 1
                    st["seg_len"].append(run)
                    run = 0
                elif k & kGateXNext:
                    st["X"] += 1
                else:
                    st["L"] += 1
    it = max(st["items"], 1)
    print(f"trajectories {a.traj}: items/traj {st['items'] / a.traj:.2f}  TC gates/item {st['tc'] / it:.2f}  "
          f"CUDA-core gates/item {st['cc'] / it:.3f}  segments/item {st['seg'] / it:.2f}  "
          f"L/item {st['L'] / it:.2f}  X/item {st['X'] / it:.2f}")
    print(f"gather wavefronts per LDS.64 {st['gwf'] / max(st['seg'], 1):.2f} {dict(sorted(hist_g.items()))}; "
          f"write-back {st['wwf'] / max(st['seg'], 1):.2f} {dict(sorted(hist_w.items()))}")
    sl = st["seg_len"]
    print("segment length histogram", {n: sl.count(n) for n in sorted(set(sl))})


if __name__ == "__main__":
    main()
