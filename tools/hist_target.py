"""Profiling / timing target of the histogram kernel (config 5: 100 x 256 random matrix,
mt19937_64 seed 3, the full weight histogram of level c), run a few times.
Usage: python tools/hist_target.py [--c 5] [--reps 3]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_08963_b200 as mdg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--c", type=int, default=5)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
M = mdg.gen_matrix(256, 100, 3, identity=False)
dev = mdg.Device(0)
dev.load_gammas(M, 256, ranks=None)
for i in range(a.reps):
    o, h = dev.round_hist(0, a.c, 256)
    print(f"rep {i}: c={a.c} min={o.min_weight} evaluated={o.evaluated} ms={o.device_ms:.4f} "
          f"cw/s={o.evaluated / (o.device_ms * 1e-3):.4e} hist_sum={int(h.sum())}", flush=True)
dev.close()
