import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
code, count, seed = (int(a) for a in sys.argv[1:4])
os.environ["MDG_FORCE_FOLD"] = str(code)
import paper_1911_08963_b200 as mdg
from oracle import port
rng = np.random.default_rng(seed)
dev = mdg.Device(0)
checked = 0
while checked < count:
    k = int(rng.integers(4, 28)); n = int(rng.integers(k + 1, 4 * k + 20))
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
            try:
                r = mdg.min_weight(rows, n, 10, s, kernel=kernel, device=dev, exact_rounds=exact)
            except Exception as e:
                print("FAIL", checked, n, k, dens, s, kernel, exact, str(e)[:300], flush=True)
                print("ref d", ref.d, "m", ref.m, "k_last", ref.k_last, "rounds", ref.rounds, flush=True)
                np.save(f"gpurun_out/repro_{checked}.npy", rows)
                gs = mdg.GammaSet.build(rows, n, 10, s)
                dev2 = mdg.Device(0); dev2.load_gset(gs); dev2.set_kernel(kernel)
                for (c, j, w, u) in ref.rounds:
                    o = dev2.round(j, c)
                    print("  round", c, j, "ref", w, "gpu", o.min_weight, hex(o.argmin_key), "tasks", o.task_lo, o.task_hi, flush=True)
                    try:
                        print("   witness", dev2.round_witness(j, c, o))
                    except Exception as e2:
                        print("   witness FAIL", str(e2)[:100])
                dev2.close()
    checked += 1
print("done", checked)
