"""GPU vs host permutation search time for many trials (dev tool)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_08963_b200 as mdg  # noqa: E402

dev = mdg.Device(0)
for (n, k, seed) in [(128, 64, 1), (300, 200, 11), (256, 32, 7)]:
    G = mdg.gen_matrix(n, k, seed, True)
    mdg.GammaSet.build(G, n, 10, 1, device=dev)  # warm-up
    for trials in (1000, 10000, 100000):
        t0 = time.perf_counter()
        g = mdg.GammaSet.build(G, n, trials, 1, device=dev)
        t1 = time.perf_counter()
        line = f"[{n},{k}] trials={trials} gpu={1e3 * (t1 - t0):.2f} ms (m={g.m}, k_last={g.k_last})"
        if trials <= 10000:
            t2 = time.perf_counter()
            h = mdg.GammaSet.build(G, n, trials, 1)
            t3 = time.perf_counter()
            assert h.column_perm == g.column_perm
            line += f" host={1e3 * (t3 - t2):.2f} ms (x{(t3 - t2) / (t1 - t0):.1f})"
        print(line, flush=True)
