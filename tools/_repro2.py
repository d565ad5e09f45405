import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_08963_b200 as mdg
from oracle import port
rows = np.load("tools/_data/repro_607.npy"); n, s = 85, 729
ref = port.min_weight(rows, n, 10, s)
dev = mdg.Device(0)
for rep in range(6):
    try:
        r = mdg.min_weight(rows, n, 10, s, kernel=0, device=dev, exact_rounds=True)
        ok = r.d == ref.d and r.rounds == [[c, j, w, u] for c, j, w, u in ref.rounds] and r.witness_ok
        print("rep", rep, "ok" if ok else "MISMATCH", r.d, r.rounds[-4:], flush=True)
    except Exception as e:
        print("rep", rep, "FAIL", str(e)[:120], flush=True)
