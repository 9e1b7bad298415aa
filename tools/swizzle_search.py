"""Search GF(2)-linear tile swizzles swz(l) = l ^ sum_{i>=3, bit i of l} v_i
(v_i in GF(2)^3, bits 0-2 identity) for the fused kernel's shared-memory
access patterns (see run_slots in gf_engine.cu):
  gate / grp loops: LDS.128, quarter-warp = tuples {t, t+1} x amps {0,lo,hi,lo+hi}
      -> wavefronts per quarter = 2^(3 - rank(v_b0, v_lo, v_hi))
  hole loop: LDS.64, half-warp = tuples 4q+{0..3} x amps {0, lo} x re/im
      -> wavefronts per half   = 2^(3 - rank(v_b0, v_b1, v_lo))
b0, b1 = lowest local bits outside {lo, hi}.  Cost per slot = gate + hole
excess, weighted over all target pairs (lo < hi) of an m-bit tile."""
import itertools
import random
import sys

M = int(sys.argv[1]) if len(sys.argv) > 1 else 11


def rank(vs):
    basis = []
    for v in vs:
        for b in basis:
            v = min(v, v ^ b)
        if v:
            basis.append(v)
    return len(basis)


def vec(V, i):
    return 1 << i if i < 3 else V[i - 3]


def cost(V, pairs):
    tot = 0.0
    for lo, hi in pairs:
        free = [b for b in range(M) if b not in (lo, hi)]
        b0, b1 = free[0], free[1]
        g = 2 ** (3 - rank([vec(V, b0), vec(V, lo), vec(V, hi)]))
        h = 2 ** (3 - rank([vec(V, b0), vec(V, b1), vec(V, lo)]))
        # REV slot: 1 gate (psi) + 3 grp-pattern vectors, 3 hole operands
        tot += 4 * (g - 1) + 3 * (h - 1)
    return tot / len(pairs)


pairs = [(a, b) for b in range(1, M) for a in range(b)]
if len(sys.argv) > 2:  # weight by the dense slots of a GF_DUMP_PLAN dump (reverse passes)
    pairs = []
    for line in open(sys.argv[2]):
        if line.startswith("rev"):
            for tok in line.split("slots:")[1].split():
                mode, rest = tok.split(":")
                lo, hi = map(int, rest.split(","))
                if mode == "0":
                    pairs.append((lo, hi))
cur = [1, 2, 5, 2, 5, 2, 5, 2][: M - 3]  # the fold (l>>3)^(l>>5)^(l>>7)^(l>>9)
cur = []
for i in range(3, M):
    v = 0
    for s in (3, 5, 7, 9):
        if 0 <= i - s < 3:
            v ^= 1 << (i - s)
    cur.append(v)
print("current fold", cur, "cost", round(cost(cur, pairs), 3))
best, bc = None, 1e9
rng = random.Random(0)
for restart in range(200):
    V = [rng.randrange(8) for _ in range(M - 3)]
    c = cost(V, pairs)
    improved = True
    while improved:
        improved = False
        for i in range(M - 3):
            for v in range(8):
                if v == V[i]:
                    continue
                W = V[:]
                W[i] = v
                cw = cost(W, pairs)
                if cw < c - 1e-12:
                    V, c, improved = W, cw, True
    if c < bc:
        best, bc = V, c
print("best", best, "cost", round(bc, 3))
