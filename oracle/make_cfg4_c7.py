"""TEST INFRASTRUCTURE — pin config 4 ([300,200] seed 11) to level cap 7 with the reference.

The cap-6 trace (tests/golden/configs_cap4_6.json) comes from the reference's own
level loop.  Level 7 costs 2 x C(200,7) = 4.5e12 codewords, so this script runs
its two rounds one at a time through the reference's `scheduled_round`
(proj/src/parallel.cpp:256-275, dynamic schedule, prefix p = 3, all host
threads) on the reference-built Gamma matrices (the same `best_gamma_over_
permutations` output the cap-6 trace used: the Gamma hashes are compared), and
writes each round's minimum to a checkpoint file as soon as it finishes.  The
level-7 (L, U) entry is then replayed with the reference's run_bz_loop rules
(engines.cpp:447-476): U = min(U, w) per round (no round skipped: U > L at cap 6),
L = max(L, lower_bound(m, 7, k, k_last)) (gamma.cpp:96-100).

Output: tests/golden/configs_cap4_7.json, the cap-6 record extended by level 7.
Usage: nohup python oracle/make_cfg4_c7.py [--workers N] &   (about 2 h on 8 cores)
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import ref  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")
CKPT = os.path.join(ROOT, "oracle", "_ref", "cfg4_c7_rounds.json")


def lower_bound(m, c, k, k_last):
    """gamma.cpp:96-100."""
    return (m - 1) * (c + 1) + max(0, c + 1 - k + k_last)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workers", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--c", type=int, default=7)
    a = ap.parse_args()
    with open(os.path.join(GOLD, "configs_cap4_6.json")) as f:
        base = next(r for r in json.load(f)["data"] if r["name"] == "cfg4")
    assert base["level_cap"] == a.c - 1 and base["capped"]
    n, k, seed = base["gen"]["n"], base["gen"]["k"], base["gen"]["seed"]
    text = ref.gen(n, k, seed)
    g = ref.trace(text, trials=10, seed=seed, engine="stack", level_cap=1, with_rows=True)
    assert g["gamma_hash"] == base["gamma_hash"], "Gamma set differs from the cap-6 golden"
    W = (n + 63) // 64
    done = {}
    if os.path.exists(CKPT):
        with open(CKPT) as f:
            done = {int(j): v for j, v in json.load(f).items()}
    for j, hexrows in enumerate(g["gammas"]):
        if j in done:
            continue
        rows = np.array([[int(h[16 * i:16 * i + 16], 16) for i in range(W)] for h in hexrows],
                        dtype=np.uint64)
        t0 = time.time()
        w, combos = ref.round_min(rows, n, a.c, engine="scheduled", workers=a.workers)
        done[j] = {"w": w, "combinations": combos, "seconds": time.time() - t0,
                   "engine": f"scheduled_round dynamic p=3, {a.workers} threads"}
        print(f"round (c={a.c}, j={j}): w={w} combos={combos} {done[j]['seconds']:.0f}s", flush=True)
        os.makedirs(os.path.dirname(CKPT), exist_ok=True)
        with open(CKPT, "w") as f:
            json.dump({str(x): v for x, v in done.items()}, f)
    m, k_last = base["m"], base["k_last"]
    U, L = base["U_final"], base["L_final"]
    rounds = [list(r) for r in base["rounds"]]
    for j in range(m):
        assert U > L
        U = min(U, done[j]["w"])
        rounds.append([a.c, j, done[j]["w"], U])
    L = max(L, lower_bound(m, a.c, k, k_last))
    out = dict(base)
    out.update(level_cap=a.c, rounds=rounds, levels=base["levels"] + [[a.c, L, U]],
               U_final=U, L_final=L, g_final=a.c,
               combinations=base["combinations"] + sum(v["combinations"] for v in done.values()),
               level7_rounds={str(j): v for j, v in done.items()})
    out.pop("wall_seconds", None)
    with open(os.path.join(GOLD, f"configs_cap4_{a.c}.json"), "w") as f:
        json.dump({"generator": "oracle/make_cfg4_c7.py (cap-6 reference trace + level-7 rounds by "
                                "the reference's scheduled_round via oracle/_ref/libmdref_v3.so)",
                   "data": [out]}, f, separators=(",", ":"))
        f.write("\n")
    print(f"level {a.c}: L={L} U={U}")


if __name__ == "__main__":
    main()
