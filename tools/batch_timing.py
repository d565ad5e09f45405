"""Wall time of the batch front door on the bench's eight config-2 codes (development tool).
MDG_TIMING=1 adds the per-code timeline from the library."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_08963_b200 as mdg  # noqa: E402

dev = mdg.Device(0)
Gs = [mdg.gen_matrix(128, 64, s, True) for s in range(1, 9)]
for gsearch in (sys.argv[1:] or ["host", "gpu"]):
    for streams in (4,):
        ts = []
        for rep in range(6):
            t0 = time.perf_counter()
            runs = mdg.min_weight_batch(Gs, 128, trials=10, seed=list(range(1, 9)), device=dev,
                                        streams=streams, gamma_search=gsearch)
            ts.append(time.perf_counter() - t0)
        print(f"gamma_search={gsearch} streams={streams} batch ms best {min(ts[1:]) * 1e3:.3f} "
              f"median {sorted(ts[1:])[len(ts[1:]) // 2] * 1e3:.3f}", flush=True)
