"""Randomized parity sweep (development tool): full BZ runs of random codes with every stage-1
variant forced on every tile bound (MDG_FORCE_FOLD, set per subprocess), both kernels and round
modes, against the C oracle. Usage: python tools/forced_sweep.py CODE COUNT SEED"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_08963_b200 as mdg  # noqa: E402
from oracle import port  # noqa: E402

code, count, seed = (int(a) for a in sys.argv[1:4])
os.environ["MDG_FORCE_FOLD"] = str(code)
rng = np.random.default_rng(seed)
dev = mdg.Device(0)
checked = bad = 0
while checked < count:
    k = int(rng.integers(4, 28))
    n = int(rng.integers(k + 1, 4 * k + 20))
    dens = float(rng.choice([0.1, 0.25, 0.5]))
    dense = (rng.random((k, n)) < dens).astype(np.uint64)
    rows = np.zeros((k, (n + 63) // 64), dtype=np.uint64)
    for c in range(n):
        rows[:, c // 64] |= dense[:, c] << np.uint64(c % 64)
    if port.rank(rows, n) != k:
        continue
    s = int(rng.integers(0, 1000))
    ref = port.min_weight(rows, n, 10, s)
    for kernel in (0, 1):
        for exact in (True, False):
            r = mdg.min_weight(rows, n, 10, s, kernel=kernel, device=dev, exact_rounds=exact)
            U, want = n - k + 1, []
            for c, j, w, u in ref.rounds:
                want.append([c, j, w if exact else min(w, U), u])
                U = u
            ok = (r.d == ref.d and r.levels == ref.levels and r.rounds == want and r.witness_ok)
            if not ok:
                bad += 1
                print("MISMATCH", code, n, k, dens, s, kernel, exact, r.d, ref.d, flush=True)
    checked += 1
print(f"code {code}: {checked} codes x 4 runs, {bad} mismatches", flush=True)
