"""Config 1 by exhaustive Gray-code brute force (2^40 - 1 codewords): device time (development tool)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_08963_b200 as mdg  # noqa: E402

dev = mdg.Device(0)
G = mdg.gen_matrix(80, 40, 1, True)
for rep in range(3):
    t0 = time.perf_counter()
    r = mdg.brute_force(G, 80, device=dev)
    dt = time.perf_counter() - t0
    print(f"d={r.d} evaluated={r.evaluated} wall_s={dt:.4f} device_s={r.device_seconds:.4f} "
          f"cw/s={r.evaluated / r.device_seconds:.4e}", flush=True)
