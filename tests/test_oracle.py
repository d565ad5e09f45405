"""Pin the plain-C oracle restatement (oracle/mdoracle.c) to the reference.

The golden vectors were produced by running the compiled, unmodified
reference (oracle/_ref, see oracle/make_golden.py). Every check here is CPU
only; the GPU parity tests then compare the CUDA path against the same
vectors and against this oracle.
"""
import numpy as np
import pytest

from conftest import load_golden
from oracle import port


def test_generator_matches_reference_convention():
    for cfg in load_golden("configs"):
        g = cfg["gen"]
        rows = port.gen_matrix(g["n"], g["k"], g["seed"], g["identity"])
        assert port.hash_rows(rows, g["n"]) == cfg["matrix_hash"], cfg["name"]
    h = load_golden("cfg5_hist")
    rows = port.gen_matrix(256, 100, 3, identity=False)
    assert port.hash_rows(rows, 256) == h["matrix_hash"]


@pytest.mark.parametrize("kind", ["kats", "seeded"])
def test_traces_match_reference(kind):
    for case in load_golden(kind):
        rows, n = port.parse_matrix_text(case["matrix"])
        tr = port.min_weight(rows, n, case["trials"], case["seed"])
        assert tr.d == case["d"] == case["d_brute"], case["name"]
        assert tr.rounds == case["rounds"], case["name"]
        assert tr.levels == case["levels"], case["name"]
        assert tr.m == case["m"] and tr.k_last == case["k_last"], case["name"]
        assert tr.g_final == case["g_final"], case["name"]
        assert tr.column_perm == case["column_perm"], case["name"]
        assert tr.gamma_hash == case["gamma_hash"], case["name"]
        assert port.brute(port.row_basis(rows, n), n) == case["d_brute"], case["name"]


def test_round_minima_match_reference():
    for case in load_golden("rounds"):
        rows, n = port.parse_matrix_text(case["matrix"])
        for lv in case["levels"]:
            w, combos = port.round_min(rows, n, lv["c"])
            assert (w, combos) == (lv["min"], lv["combinations"]), (case["n"], case["k"], lv)


def test_configs_gamma_sets_and_early_levels():
    """Gamma sets of all configs; trace prefixes at a level cap small enough for the CPU suite."""
    caps = {"cfg1": 0, "cfg3": 5, "cfg4": 3}
    for cfg in load_golden("configs"):
        g = cfg["gen"]
        rows = port.gen_matrix(g["n"], g["k"], g["seed"], True)
        cap = caps.get(cfg["name"], 4)
        tr = port.min_weight(rows, g["n"], cfg["trials"], cfg["seed"], level_cap=cap)
        assert tr.m == cfg["m"] and tr.k_last == cfg["k_last"], cfg["name"]
        assert tr.column_perm == cfg["column_perm"], cfg["name"]
        assert tr.gamma_hash == cfg["gamma_hash"], cfg["name"]
        nr = len(tr.rounds)
        assert tr.rounds == cfg["rounds"][:nr], cfg["name"]
        assert tr.levels == cfg["levels"][: len(tr.levels)], cfg["name"]
        if cap == 0:
            assert tr.d == cfg["d"]


def test_cfg5_histograms():
    """The C port's histograms against the reference's at every level of config 5 (c = 1..5)
    and at level 6 of the same matrix (1,192,052,400 codewords, ~20 s)."""
    h = load_golden("cfg5_hist")
    rows = port.gen_matrix(256, 100, 3, identity=False)
    for lv in h["levels"] + [load_golden("cfg5_hist_c6")["level"]]:
        w, hist = port.round_hist(rows, 256, lv["c"])
        assert w == lv["min"]
        assert hist.tolist() == lv["hist"]
        assert int(hist.sum()) == lv["count"]


def test_lower_bound_spot_values():
    # test_gamma.cpp:121-128
    L = port.lib().mdo_lower_bound
    assert L(2, 1, 4, 3) == 3
    assert L(2, 3, 12, 12) == 8
    assert L(1, 4, 10, 4) == 0
    assert L(3, 2, 5, 5) == 9
    assert L(1, 2, 8, 8) == 3
    assert port.lib().mdo_singleton_upper(7, 4) == 4
    assert port.lib().mdo_singleton_upper(23, 12) == 12
    assert port.lib().mdo_singleton_upper(5, 5) == 1


def test_cfg4_cap7_golden_consistent():
    """configs_cap4_7.json (the reference's cap-6 trace + its level-7 rounds, oracle/
    make_cfg4_c7.py) extends configs_cap4_6.json exactly, and its level-7 (L, U) entry is the
    run_bz_loop replay (engines.cpp:447-476) with the oracle's lower_bound (gamma.cpp:96-100);
    the Gamma set is the one the oracle restatement builds from the config-4 input."""
    c6 = next(c for c in load_golden("configs_cap4_6") if c["name"] == "cfg4")
    c7 = next(c for c in load_golden("configs_cap4_7") if c["name"] == "cfg4")
    assert c7["rounds"][:len(c6["rounds"])] == c6["rounds"]
    assert c7["levels"][:len(c6["levels"])] == c6["levels"]
    assert c7["gamma_hash"] == c6["gamma_hash"] and c7["column_perm"] == c6["column_perm"]
    U, L = c6["U_final"], c6["L_final"]
    for j in range(c7["m"]):
        w = c7["level7_rounds"][str(j)]["w"]
        assert c7["level7_rounds"][str(j)]["combinations"] == 2283896214600  # C(200, 7)
        U = min(U, w)
        assert c7["rounds"][len(c6["rounds"]) + j] == [7, j, w, U]
    L = max(L, int(port.lib().mdo_lower_bound(c7["m"], 7, c7["k"], c7["k_last"])))
    assert c7["levels"][-1] == [7, L, U] and (U, L) == (c7["U_final"], c7["L_final"]) == (22, 8)
