"""Randomized soak of ONE long-lived context (development tool): a random mix of the public calls
-- front door (both kernels, both round modes, level caps), batch front door, device-resident
loops, one code split across several contexts (exchange group), single rounds (whole, bounded, split into task ranges), witnesses, histograms (whole and
split across ranks), brute force -- on random codes, every result against the C oracle. Meant to
be run with MDG_SLOTS small as well (the scratch ring then wraps every few launches).
Usage: python tools/soak.py ITERATIONS SEED"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_08963_b200 as mdg  # noqa: E402
from oracle import port  # noqa: E402

iters, seed = int(sys.argv[1]), int(sys.argv[2])
rng = np.random.default_rng(seed)
dev = mdg.Device(0)
group = [mdg.Device(0) for _ in range(3)]  # long-lived members of the in-process exchange group
bad = []


def rand_code(kmax=20, full_rank=True):
    while True:
        k = int(rng.integers(2, kmax))
        n = int(rng.integers(k + 1, 4 * k + 24))
        if rng.random() < 0.15:  # a wide code: every row width of the kernels (up to 32 words)
            k = int(rng.integers(2, min(kmax, 9)))
            n = int(rng.integers(100, 1025))
        dens = float(rng.choice([0.08, 0.25, 0.5]))
        dense = (rng.random((k, n)) < dens).astype(np.uint64)
        rows = np.zeros((k, (n + 63) // 64), dtype=np.uint64)
        for c in range(n):
            rows[:, c // 64] |= dense[:, c] << np.uint64(c % 64)
        r = port.rank(rows, n)
        if r == 0 or (full_rank and r != k):
            continue
        return rows, n, k


def expect_rounds(ref, n, k, exact):
    U, want = n - k + 1, []
    for c, j, w, u in ref.rounds:
        want.append([c, j, w if exact else min(w, U), u])
        U = u
    return want


def weight(rows, idx):
    acc = np.zeros(rows.shape[1], dtype=np.uint64)
    for r in idx:
        acc ^= rows[r]
    return sum(bin(int(x)).count("1") for x in acc)


def check(ok, what):
    if not ok:
        bad.append(what)
        print("MISMATCH", what, flush=True)


for it in range(iters):
    op = int(rng.integers(0, 9))
    try:
        if op == 0:  # front door
            rows, n, k = rand_code()
            s, kernel, exact = int(rng.integers(0, 1000)), int(rng.integers(0, 2)), bool(rng.integers(0, 2))
            cap = int(rng.integers(0, 4))
            ref = port.min_weight(rows, n, 10, s, level_cap=cap)
            r = mdg.min_weight(rows, n, 10, s, level_cap=cap, kernel=kernel, device=dev, exact_rounds=exact)
            want = expect_rounds(ref, n, k, exact)
            check(r.d == ref.d and r.rounds == want[:len(r.rounds)] and len(r.rounds) == len(want) and
                  r.levels == ref.levels and (r.capped or r.witness_ok), ("min_weight", it, n, k, s, kernel, exact, cap))
        elif op == 1:  # batch front door
            codes = [rand_code(14) for _ in range(int(rng.integers(2, 7)))]
            same = codes
            seeds = [int(rng.integers(0, 1000)) for _ in same]
            runs = mdg.min_weight_batch([c[0] for c in same], [c[1] for c in same], trials=10, seed=seeds,
                                        device=dev, streams=int(rng.integers(1, 5)))
            for (rows, n, k), s, r in zip(same, seeds, runs):
                ref = port.min_weight(rows, n, 10, s)
                check(r.d == ref.d and r.rounds == expect_rounds(ref, n, k, False) and r.witness_ok,
                      ("batch", it, n, k, s))
        elif op == 2:  # device-resident loop over a loaded Gamma set, twice
            rows, n, k = rand_code()
            s = int(rng.integers(0, 1000))
            gs = mdg.GammaSet.build(rows, n, 10, s)
            dev.load_gset(gs)
            ref = port.min_weight(rows, n, 10, s)
            for kernel in (int(rng.integers(0, 2)), int(rng.integers(0, 2))):
                r = dev.bz_loop(gs, kernel=kernel)
                check(r.d == ref.d and r.rounds == expect_rounds(ref, n, k, False) and r.witness_ok,
                      ("bz_loop", it, n, k, s, kernel))
        elif op in (3, 4):  # single rounds on a raw matrix: whole, bounded, split; witness
            rows, n, k = rand_code(18, full_rank=False)
            dev.load_gammas(rows, n, ranks=None)
            dev.set_kernel(int(rng.integers(0, 2)))
            c = int(rng.integers(1, min(k, 6) + 1))
            w, _ = port.round_min(rows, n, c)
            o = dev.round(0, c)
            check(o.min_weight == w, ("round", it, n, k, c))
            idx = dev.round_witness(0, c, o)
            check(len(idx) == c and weight(rows, idx) == w, ("witness", it, n, k, c))
            cut = int(rng.integers(max(1, w - 2), w + 4))
            ob = dev.round_bounded(0, c, cut)
            check(ob.min_weight == min(w, cut) and bool(ob.bounded) == (w >= cut), ("bounded", it, n, k, c, cut))
            world = int(rng.integers(2, 5))
            best = 1 << 30
            for rnk in range(world):
                lo, hi = dev.split_range(0, c, rnk, world)
                if hi > lo:
                    best = min(best, dev.round_range(0, c, lo, hi).min_weight)
            check(best == w, ("split", it, n, k, c, world))
            dev.set_kernel(0)
        elif op == 5:  # histograms, whole and split
            rows, n, k = rand_code(14, full_rank=False)
            dev.load_gammas(rows, n, ranks=None)
            c = int(rng.integers(1, min(k, 5) + 1))
            w, h = port.round_hist(rows, n, c)
            o, hist = dev.round_hist(0, c, n)
            check(hist.tolist() == h.tolist() and o.min_weight == w, ("hist", it, n, k, c))
            world = int(rng.integers(2, 5))
            tot = np.zeros(n + 1, dtype=np.uint64)
            for rnk in range(world):
                tot += dev.round_hist_dist(0, c, n, rnk, world)[1]
            check(tot.tolist() == h.tolist(), ("hist split", it, n, k, c, world))
        elif op == 6:  # brute force
            rows, n, k = rand_code(14)
            r = mdg.brute_force(rows, n, device=dev)
            check(r.d == port.brute(rows, n) and r.witness_ok, ("brute", it, n, k))
        elif op == 8:  # one code split across 2-3 contexts (exchange group), every round or some
            rows, n, k = rand_code()
            s = int(rng.integers(0, 1000))
            world = int(rng.integers(2, 4))
            split_min = int(rng.choice([1, 200, 5000]))
            ref = port.min_weight(rows, n, 10, s)
            runs = mdg.min_weight_multi(rows, n, group[:world], trials=10, seed=s, split_min=split_min,
                                        kernel=int(rng.integers(0, 2)))
            for r in runs:
                check(r.d == ref.d and r.rounds == expect_rounds(ref, n, k, False) and r.levels == ref.levels and
                      r.witness_ok, ("multi", it, n, k, s, world, split_min))
        else:  # rank-deficient input through the front door
            rows, n, k = rand_code(12, full_rank=False)
            extra = rows[rng.integers(0, k, size=3)]
            rows2 = np.vstack([rows, extra[0:1] ^ extra[1:2], extra[2:3]])
            s = int(rng.integers(0, 1000))
            ref = port.min_weight(rows2, n, 10, s)
            r = mdg.min_weight(rows2, n, 10, s, device=dev)
            check(r.d == ref.d and r.levels == ref.levels and r.witness_ok, ("deficient", it, n, k, s))
    except Exception as e:  # an unexpected error is a failure too
        bad.append(("exception", it, op, str(e)[:200]))
        print("EXCEPTION", it, op, str(e)[:300], flush=True)
print(f"soak seed {seed}: {iters} operations, {len(bad)} failures (MDG_SLOTS={os.environ.get('MDG_SLOTS')})", flush=True)
sys.exit(1 if bad else 0)
