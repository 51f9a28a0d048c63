"""Why the warp tiles keep the lane-per-cell candidate walk: a Monte Carlo of
c4's 32-cell tiles comparing the walk's passes with the passes of warp-level claim rounds
(as k_collide_heavy runs them).

Per cell: N ~ Poisson(10) particles (the equilibrium box), M = floor(N(N-1)/2 * c + u) candidates
with c chosen so that E[M] = 3.13 (the measured 3.13 per cell), candidate pairs uniform over the
cell's particle pairs.  Lane-per-cell walk: one pass per candidate of the tile's largest cell.
Claim rounds: in each round every undone candidate whose particles no earlier undone candidate
of its cell touches runs; the runnable ones are compacted onto the 32 lanes, ceil(ready / 32)
passes per round.  usage: python analysis/claim_rounds_model.py [TILES]"""
import sys

import numpy as np


def tile_passes(rng, c):
    walk = 0
    claims = []                                   # per cell: list of (i, j) in k order
    for _ in range(32):
        n = rng.poisson(10.0)
        if n < 2:
            claims.append([])
            continue
        m = int(np.floor(n * (n - 1) / 2 * c + rng.random()))
        walk = max(walk, m)
        pairs = []
        for _ in range(m):
            i = rng.integers(n)
            j = rng.integers(n - 1)
            j += j >= i
            pairs.append((i, j))
        claims.append(pairs)
    rounds, passes = 0, 0
    undone = [list(range(len(p))) for p in claims]
    while any(undone):
        ready = 0
        nxt = []
        for cell, u in zip(claims, undone):
            touched, keep = set(), []
            for k in u:
                i, j = cell[k]
                if i in touched or j in touched:
                    keep.append(k)
                else:
                    ready += 1
                touched.add(i)
                touched.add(j)
            nxt.append(keep)
        undone = nxt
        rounds += 1
        passes += -(-ready // 32)
    return walk, rounds, passes


def main():
    tiles = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
    rng = np.random.Generator(np.random.PCG64(7))
    n = rng.poisson(10.0, 200000)
    c = 3.13 / np.mean(n * (n - 1) / 2)
    w, r, p = np.array([tile_passes(rng, c) for _ in range(tiles)]).T
    print(f"tiles {tiles}: lane-per-cell walk passes {w.mean():.2f}; claim rounds {r.mean():.2f} "
          f"({p.mean():.2f} compacted 32-lane passes)")


if __name__ == "__main__":
    main()
