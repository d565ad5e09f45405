"""Profiling target: the dominant launch of the bench workload (config 2, seed 1,
level-7 round of Gamma_0: 621,216,192 codewords), run a few times.
Usage: python tools/ncu_target.py [--kernel tab|rd] [--c 7] [--reps 3]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_08963_b200 as mdg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--kernel", default="tab")
ap.add_argument("--c", type=int, default=7)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--n", type=int, default=128)
ap.add_argument("--k", type=int, default=64)
ap.add_argument("--seed", type=int, default=1)
ap.add_argument("--j", type=int, default=0)
ap.add_argument("--cutoff", type=int, default=0, help="bound U (0 = exact round)")
a = ap.parse_args()
G = mdg.gen_matrix(a.n, a.k, a.seed, True)
gs = mdg.GammaSet.build(G, a.n, 10, a.seed)
dev = mdg.Device(0)
dev.load_gset(gs)
dev.set_kernel(mdg.KERNEL_TAB if a.kernel == "tab" else mdg.KERNEL_RD)
for i in range(a.reps):
    o = dev.round_bounded(a.j, a.c, a.cutoff) if a.cutoff else dev.round(a.j, a.c)
    print(f"rep {i}: w={o.min_weight} evaluated={o.evaluated} ms={o.device_ms:.4f} "
          f"cw/s={o.evaluated / (o.device_ms * 1e-3):.4e}", flush=True)
dev.close()
