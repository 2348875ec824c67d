"""Generator of tests/golden/rng_contract.txt: the RNG-contract golden vectors of
reading R6 computed by a THIRD implementation of
Philox4x32-10 (Salmon et al. 2011) in plain Python integers, independent of
oracle/ (C) and of the CUDA path (csrc/philox.hpp).  Test infrastructure only.

Contract: key = (seed_lo32, seed_hi32), counter = (ordinal, purpose, traj_lo32,
traj_hi32), purpose 1 CHANNEL, 2 SAMPLE, 3 READOUT, 4 MEASURE; each block gives
u53(x0, x1) (half 0) and u53(x2, x3) (half 1), u53(a, b) = ((a >> 5) 2^26 +
(b >> 6)) 2^-53.  CHANNEL: ordinal = channel ordinal, half 0.  SAMPLE / READOUT:
ordinal = shot * ceil(n / 2) + level // 2 (qubit // 2), half = level % 2.

usage: python tools/gen_rng_golden.py [--check]   (writes / compares the file)"""
import math
import os
import sys

M0, M1 = 0xD2511F53, 0xCD9E8D57
W0, W1 = 0x9E3779B9, 0xBB67AE85
MASK = 0xFFFFFFFF
PATH = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                    "rng_contract.txt")


def philox(ctr, key):
    c0, c1, c2, c3 = ctr
    k0, k1 = key
    for _ in range(10):
        p0, p1 = M0 * c0, M1 * c2
        hi0, lo0 = p0 >> 32, p0 & MASK
        hi1, lo1 = p1 >> 32, p1 & MASK
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
        k0, k1 = (k0 + W0) & MASK, (k1 + W1) & MASK
    return [c0, c1, c2, c3]


def u53(a, b):
    return ((a >> 5) * 67108864 + (b >> 6)) * (1.0 / 9007199254740992.0)


def draw(seed, ordinal, purpose, traj, half=0):
    x = philox([ordinal & MASK, purpose, traj & MASK, (traj >> 32) & MASK], [seed & MASK, (seed >> 32) & MASK])
    return u53(x[0], x[1]) if half == 0 else u53(x[2], x[3])


def ghz4_histogram(seed, p=0.01, trajectories=1000):
    """Config 1 (GHZ-4, depolarize(p) on every touched qubit after every gate: 7
    channels): Alg. 2 first loop on lower bounds pbar = (1 - p, p/3,
    p/3, p/3) = squared scales of the Kraus list (I, X, Y, Z); a unitary mixture,
    so s = 1 and the fall-through picks the last operator."""
    pbar = [math.sqrt(1 - p) ** 2] + [math.sqrt(p / 3) ** 2] * 3
    hist = [0, 0, 0, 0]
    for t in range(trajectories):
        for c in range(7):
            r = draw(seed, c, 1, t)
            pick = 3
            for i, pb in enumerate(pbar):
                if r < pb:
                    pick = i
                    break
                r -= pb
            hist[pick] += 1
    return hist


def lines():
    seed = 0x23962112
    n = 4
    half_n = (n + 1) // 2
    out = ["# RNG-contract golden vectors (reading R6: key=(seed_lo,seed_hi),",
           "# ctr=(ordinal, purpose, traj_lo, traj_hi), u53(a,b)=((a>>5)*2^26+(b>>6))*2^-53).",
           "# Written by tools/gen_rng_golden.py: a third Philox4x32-10 in plain Python",
           "# integers, independent of oracle/ and of the CUDA path.",
           "# seed 0x23962112 (config 1 trajectory seed); n = 4 for the SAMPLE / READOUT ordinals."]
    out.append("block 0 1 0 0 -> " + " ".join(f"{w:08x}" for w in philox([0, 1, 0, 0], [seed, 0])))
    for t in (0, 1):
        out.append(f"channel traj={t} ordinals 0,1,2 -> " + " ".join(repr(draw(seed, c, 1, t)) for c in range(3)))
    for t, shot in ((0, 0), (0, 1), (0, 2), (5, 3)):
        vals = [draw(seed, shot * half_n + lvl // 2, 2, t, lvl % 2) for lvl in (3, 2, 1, 0)]
        out.append(f"sample traj={t} shot={shot} levels 3,2,1,0 -> " + " ".join(repr(v) for v in vals))
    for t, shot in ((0, 0), (0, 1), (7, 2)):
        vals = [draw(seed, shot * half_n + q // 2, 3, t, q % 2) for q in range(n)]
        out.append(f"readout traj={t} shot={shot} qubits 0,1,2,3 -> " + " ".join(repr(v) for v in vals))
    # a far trajectory index (traj_hi32 != 0)
    out.append("channel traj=4294967297 ordinal 9 -> " + repr(draw(seed, 9, 1, (1 << 32) + 1)))
    out.append("# config 1 (GHZ-4 + depolarize(0.01), 7 channels x 1000 trajectories) pick histogram I X Y Z")
    out.append("ghz4_hist " + " ".join(str(h) for h in ghz4_histogram(seed)))
    return out


if __name__ == "__main__":
    text = "\n".join(lines()) + "\n"
    if "--check" in sys.argv:
        sys.exit(0 if open(PATH).read() == text else 1)
    with open(PATH, "w") as f:
        f.write(text)
    print(text)
