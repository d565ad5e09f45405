"""Best-of-N device time of a fixed set of bounded rounds (development tool; run it under
different MDG_* tuning variables to compare tile plans)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_08963_b200 as mdg  # noqa: E402

CASES = [  # (n, k, seed, j, c, cutoff)
    (128, 64, 1, 0, 5, 16), (128, 64, 1, 0, 6, 16), (128, 64, 1, 0, 7, 15),
    (256, 32, 7, 0, 7, 76), (256, 32, 7, 0, 8, 76), (256, 32, 7, 0, 9, 76),
    (300, 200, 11, 0, 4, 28), (300, 200, 11, 0, 5, 26), (300, 200, 11, 1, 5, 26),
]
dev = mdg.Device(0)
cache = {}
out = []
total = 0.0
for (n, k, seed, j, c, cut) in CASES:
    if (n, k, seed) not in cache:
        G = mdg.gen_matrix(n, k, seed, True)
        cache[(n, k, seed)] = mdg.GammaSet.build(G, n, 10, seed)
    gs = cache[(n, k, seed)]
    dev.load_gset(gs)
    best = None
    for _ in range(4 if c < 7 or n != 300 else 2):
        o = dev.round_bounded(j, c, cut)
        best = o.device_ms if best is None else min(best, o.device_ms)
    total += best
    out.append(f"{n}/{k} c{c}j{j}={best * 1e3:.1f}us")
print(" ".join(out), f"total={total * 1e3:.1f}us", flush=True)
