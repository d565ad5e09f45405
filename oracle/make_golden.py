"""TEST INFRASTRUCTURE — regenerate tests/golden/ from the compiled reference.

Runs the UNMODIFIED reference library (oracle/_ref/libmdref_v3.so, built by
``make -C oracle ref`` from /root/reference/proj/src) through our harness and
writes the golden vectors the parity tests compare against:

  configs.json   BASELINE configs 1-4: input hash, Gamma set (m, k_last, ranks,
                 column_perm, Gamma hashes), per-round minima and per-level
                 (L, U) trace, d. Config 4 is level-capped.
  cfg5_hist.json config 5: per-level min weight and full weight histogram.
  cfg5_hist_c6.json  the same matrix at level 6 (--only cfg5_hist_c6; 1.19e9 codewords).
  kats.json      reference known-answer codes (acceptance_main.cpp:90-125,
                 test_engines.cpp:227-255): traces + brute-force d.
  seeded.json    acceptance criterion 1's 200 seeded codes
                 (acceptance_main.cpp:44-87): traces + brute-force d.
  rounds.json    single-round minima on raw matrices (test_engines.cpp:157-169
                 and wider shapes), reference round_stack.

Usage: python oracle/make_golden.py [--only NAME] [--cap4 5] [--workers 8]
Needs /root/reference (this container only); the outputs are committed.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import port, ref  # noqa: E402

GOLD = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")

CONFIGS = [
    # name, n, k, seed, engine, level_cap
    ("cfg1", 80, 40, 1, "saved", 0),
    *[(f"cfg2_s{s}", 128, 64, s, "saved", 0) for s in range(1, 9)],
    ("cfg3", 256, 32, 7, "saved", 0),
    ("cfg4", 300, 200, 11, "scheduled", 5),
]


def cyclic(poly_exps, m):
    """cyclic_generator_matrix (codeconstruct.cpp:161-174): row i = x^i f(x)."""
    deg = max(poly_exps)
    k = m - deg
    rows = []
    for i in range(k):
        r = ["0"] * m
        for e in poly_exps:
            r[e + i] = "1"
        rows.append("".join(r))
    return f"{m} {k}\n" + "\n".join(rows) + "\n"


def extend(text):
    """extend_code (codeconstruct.cpp:233-241): append the row parity."""
    lines = [ln for ln in text.splitlines() if ln.strip()]
    n, k = (int(x) for x in lines[0].split())
    rows = [r + ("1" if r.count("1") % 2 else "0") for r in lines[1:]]
    return f"{n + 1} {k}\n" + "\n".join(rows) + "\n"


def matrix_hash(text):
    rows, n = port.parse_matrix_text(text)
    return port.hash_rows(rows, n)


def do_configs(workers, cap4):
    out = []
    for name, n, k, seed, engine, cap in CONFIGS:
        if name == "cfg4":
            cap = cap4
        text = ref.gen(n, k, seed)
        t0 = time.time()
        tr = ref.trace(text, trials=10, seed=seed, engine=engine, s=5, workers=workers, level_cap=cap)
        tr.update(name=name, matrix_hash=matrix_hash(text), gen={"n": n, "k": k, "seed": seed,
                                                                   "identity": True})
        print(f"{name}: d={tr['d']} U={tr['U_final']} rounds={len(tr['rounds'])} "
              f"{time.time() - t0:.1f}s", flush=True)
        out.append(tr)
    return out


def do_hist(cmax=5):
    text = ref.gen(256, 100, 3, identity=False)
    import subprocess
    exe = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_ref", "mdref_v3")
    path = "/tmp/_cfg5.txt"
    with open(path, "w") as f:
        f.write(text)
    t0 = time.time()
    js = json.loads(subprocess.run([exe, "hist", path, "--cmax", str(cmax)], check=True,
                                   capture_output=True, text=True).stdout)
    js.update(name="cfg5", matrix_hash=matrix_hash(text),
              gen={"n": 256, "k": 100, "seed": 3, "identity": False})
    print(f"cfg5: mins={[lv['min'] for lv in js['levels']]} {time.time() - t0:.1f}s", flush=True)
    return js


def do_hist_c6():
    """Level 6 of config 5's matrix (1,192,052,400 codewords, ~3 min on one core): the histogram
    kernel's large parity case. Only the level-6 record is kept."""
    js = do_hist(6)
    return {"n": js["n"], "k": js["k"], "level": js["levels"][5], "name": "cfg5_c6",
            "matrix_hash": js["matrix_hash"], "gen": js["gen"]}


def do_kats():
    ham = cyclic([3, 1, 0], 7)
    gol = cyclic([11, 10, 6, 5, 4, 2, 0], 23)
    fx = [("hamming_7_4", ham, 3), ("ext_hamming_8_4", extend(ham), 4),
          ("golay_23_12", gol, 7), ("ext_golay_24_12", extend(gol), 8),
          ("identity_3", "3 3\n100\n010\n001\n", 1)]
    # test_engines.cpp:227-233: Hamming built from taps {0,1,3} shifted per row
    fx.append(("hamming_taps", "7 4\n" + "\n".join(
        "".join("1" if c - i in (0, 1, 3) else "0" for c in range(7)) for i in range(4)) + "\n", 3))
    # rank-deficient input (min_weight row-reduces it, test_engines.cpp:257-...)
    base = ref.random_full_rank(14, 5, 81)
    lines = base.splitlines()
    dup = "14 7\n" + "\n".join(lines[1:6] + [lines[1], lines[2]]) + "\n"
    fx.append(("rank_deficient_14_5", dup, None))
    for n in range(1, 21):
        fx.append((f"repetition_{n}", f"{n} 1\n" + "1" * n + "\n", n))
    out = []
    for name, text, d_lit in fx:
        tr = ref.trace(text, trials=10, seed=1, engine="saved", with_rows=True)
        d_brute = ref.min_weight_d(text, "brute", 10, 1)
        if d_lit is not None:
            assert tr["d"] == d_lit == d_brute, (name, tr["d"], d_lit, d_brute)
        tr.update(name=name, matrix=text, d_brute=d_brute)
        out.append(tr)
    print(f"kats: {len(out)}", flush=True)
    return out


def do_seeded():
    out = []
    for i in range(200):
        text = ref.seeded_code(1000 + i)
        tr = ref.trace(text, trials=6, seed=i, engine="saved")
        tr.update(name=f"seeded_{i}", matrix=text, d_brute=ref.min_weight_d(text, "brute", 6, i))
        assert tr["d"] == tr["d_brute"]
        out.append(tr)
    print(f"seeded: {len(out)}", flush=True)
    return out


def do_rounds():
    cases = [(21, 10, 2024, range(1, 8)), (150, 24, 5, range(1, 5)), (300, 30, 6, range(1, 4)),
             (64, 20, 7, range(1, 21)), (520, 12, 8, range(1, 13)), (33, 1, 9, [1])]
    out = []
    for n, k, seed, cs in cases:
        text = ref.random_full_rank(n, k, seed)
        rows, _ = port.parse_matrix_text(text)
        levels = []
        for c in cs:
            w, combos = ref.round_min(rows, n, c, engine="stack")
            w2, _ = ref.round_min(rows, n, c, engine="saved", s=3)
            assert w == w2
            levels.append({"c": c, "min": w, "combinations": combos})
        out.append({"n": n, "k": k, "seed": seed, "matrix": text, "levels": levels})
    print(f"rounds: {len(out)}", flush=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    ap.add_argument("--cap4", type=int, default=5)
    ap.add_argument("--workers", type=int, default=os.cpu_count() or 1)
    a = ap.parse_args()
    os.makedirs(GOLD, exist_ok=True)
    jobs = {
        "kats": lambda: do_kats(),
        "seeded": lambda: do_seeded(),
        "rounds": lambda: do_rounds(),
        "cfg5_hist": lambda: do_hist(),
        "cfg5_hist_c6": lambda: do_hist_c6(),
        "configs": lambda: do_configs(a.workers, a.cap4),
    }
    for name, fn in jobs.items():
        if (a.only and name != a.only) or (not a.only and name == "cfg5_hist_c6"):
            continue  # the level-6 histogram only on request (--only cfg5_hist_c6)
        data = fn()
        fname = name if not (name == "configs" and a.cap4 != 5) else f"configs_cap4_{a.cap4}"
        with open(os.path.join(GOLD, fname + ".json"), "w") as f:
            json.dump({"generator": "oracle/make_golden.py (reference via oracle/_ref/libmdref_v3.so)",
                       "data": data}, f, separators=(",", ":"))
            f.write("\n")


if __name__ == "__main__":
    main()
