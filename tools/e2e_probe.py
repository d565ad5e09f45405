"""Where the front-door time of one config-2 code goes (development tool)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_08963_b200 as mdg  # noqa: E402

dev = mdg.Device(0)
Gs = [mdg.gen_matrix(128, 64, s, True) for s in range(1, 9)]
for rep in range(3):
    t = {"gamma": 0.0, "load": 0.0, "loop": 0.0, "loop_nowit": 0.0, "front": 0.0}
    for G in Gs:
        t0 = time.perf_counter()
        gs = mdg.GammaSet.build(G, 128, 10, 1)
        t1 = time.perf_counter()
        dev.load_gset(gs)
        t2 = time.perf_counter()
        dev.bz_loop(gs)
        t3 = time.perf_counter()
        dev.bz_loop(gs, witness=False)
        t4 = time.perf_counter()
        mdg.min_weight(G, 128, 10, 1, device=dev)
        t5 = time.perf_counter()
        t["gamma"] += t1 - t0
        t["load"] += t2 - t1
        t["loop"] += t3 - t2
        t["loop_nowit"] += t4 - t3
        t["front"] += t5 - t4
    print({k: f"{v / 8 * 1e3:.3f} ms" for k, v in t.items()}, flush=True)
