"""Modelled shared-memory wavefronts of the persistent kernel's segment gathers (C2 plans) under its
own swizzle vs the TMA SWIZZLE_128B image, with the planner's current lane choices (tools/v2_plan_stats.py model)."""
import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, 'tools'))
import v2_plan_stats as S
import workloads
from paper_2111_02396_b200 import qtraj
c = workloads.sycamore_grid_qcs(config=2)
plan = qtraj.Plan(qtraj.Circuit.from_description(c), max_fused=4)
seed = workloads.trajectory_seed(2)
def tb(x):  # tile bit of a v2 unit (top bit - 3)
    return x.bit_length() - 1 - 3
def tma(b):
    x = 8 << b
    return x ^ (((x >> 7) & 7) << 4)
tot = {"v2": 0, "tma": 0}; n = 0
for t in range(32):
    for tm, fl, gates in S.dump(plan, seed, t):
        for m, k, u in gates:
            if not (k & S.kGateTC) or not (k & S.kGateRunStart):
                continue
            n += 1
            lanes = [tb(x) for x in u[6:11]]
            if k & S.kGatePair0:
                v2 = 2 * 2 ** (3 - S.rank([(x >> 4) & 7 for x in u[6:9]]))
                tw = 2 * 2 ** (3 - S.rank([(tma(b) >> 4) & 7 for b in lanes[:3]]))
            else:
                v2 = 2 * 2 ** (4 - S.rank([(x >> 3) & 15 for x in u[6:10]]))
                tw = 2 * 2 ** (4 - S.rank([(tma(b) >> 3) & 15 for b in lanes[:4]]))
            tot["v2"] += v2; tot["tma"] += tw
print("gathers", n, "mean wavefronts per 8B: v2 swizzle %.2f, TMA swizzle (same lanes) %.2f" % (tot["v2"] / n, tot["tma"] / n))
