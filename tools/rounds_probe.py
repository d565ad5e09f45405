"""Per-round breakdown of one device-chained BZ run (development tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_08963_b200 as mdg  # noqa: E402

n, k, seed = (int(a) for a in (sys.argv[1:4] if len(sys.argv) > 3 else (128, 64, 1)))
cap = int(sys.argv[4]) if len(sys.argv) > 4 else 0
G = mdg.gen_matrix(n, k, seed, True)
gs = mdg.GammaSet.build(G, n, 10, seed)
dev = mdg.Device(0)
dev.load_gset(gs)
for rep in range(3 if not cap else 1):
    r = dev.bz_loop(gs, level_cap=cap)
print(f"d={r.d} loop_ms={r.loop_seconds*1e3:.3f} launches={r.launches}")
tot = 0.0
for (c, j, w, U), ev, ms, b in zip(r.rounds, r.round_evaluated, r.round_ms, r.round_bounded):
    tot += ms
    print(f"c={c} j={j} w={w} U={U} bounded={b} cw={ev} ms={ms:.4f} cw/s={ev / max(ms, 1e-9) * 1e3:.3e}")
print(f"sum round ms {tot:.3f}")
