#!/usr/bin/env python
"""Offline search for the lane order of k_gen's warp-local face pass B (development tool; kernel_gen.cuh c_passb*).

Pass B runs one t2-line per lane: lane offsets FSD fo + l (+ 5 b) in the face-slot arrays, FSD = TSEL mod 16. Under
the lane order of passes A / C (lane = N fo + l) each half-warp of 8-byte accesses has 2-way bank conflicts. Any
permutation of the warp's (fo, l) tasks is valid (the passes are separated by __syncwarp); this picks one whose first
half-warp has distinct residues (FSD fo + l) mod 16 and whose second has the fewest repeats.

    python tools/passb_perm.py
"""
import collections
import random

TSEL = {3: 9, 4: 3, 5: 9}


def search(N, iters=20000, seed=1):
    rng = random.Random(seed)
    fpw = 32 // N
    tasks = [(fo, l) for fo in range(fpw) for l in range(N)]
    res = lambda t: (TSEL[N] * t[0] + t[1]) % 16
    cost = lambda h: max(collections.Counter(map(res, h)).values()) if h else 0
    best = None
    for _ in range(iters):
        rng.shuffle(tasks)
        h0, seen, rest = [], set(), []
        for t in tasks:
            if len(h0) < 16 and res(t) not in seen:
                h0.append(t)
                seen.add(res(t))
            else:
                rest.append(t)
        if len(rest) > 16:
            continue
        c = cost(h0) + cost(rest)
        if best is None or c < best[0]:
            best = (c, list(h0), list(rest))
    c, h0, h1 = best
    order = h0 + [None] * (16 - len(h0)) + h1
    order += [None] * (32 - len(order))
    ident = [(L // N, L % N) if L < fpw * N else None for L in range(32)]
    ic = sum(cost([t for t in ident[h * 16:(h + 1) * 16] if t]) for h in range(2))
    return c, ic, [-1 if t is None else t[0] * N + t[1] for t in order]


if __name__ == "__main__":
    for N in (3, 4, 5):
        c, ic, order = search(N)
        print(f"N={N}: wavefronts per pass-B access {c} (lane order of passes A/C: {ic})")
        print("  {" + ", ".join(map(str, order)) + "}")
