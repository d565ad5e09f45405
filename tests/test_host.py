"""Host side of the product (lib/libmdg.so) on CPU: Gamma systematization,
permutation search, bounds, level loop, matrix I/O, generator, combinatorics.

Mirrors the reference's test_gamma.cpp / test_engines.cpp (run_bz_loop) /
test_cli.cpp (matrix grammar) / test_enumeration.cpp cases, with the golden
vectors of the compiled reference as the expected values.
"""
import itertools

import numpy as np
import pytest

from conftest import load_golden
from oracle import port


def test_generator_matches_reference(mdg):
    for cfg in load_golden("configs"):
        g = cfg["gen"]
        rows = mdg.gen_matrix(g["n"], g["k"], g["seed"], g["identity"])
        assert mdg.hash_rows(rows, g["n"]) == cfg["matrix_hash"], cfg["name"]
    rows = mdg.gen_matrix(256, 100, 3, identity=False)
    assert mdg.hash_rows(rows, 256) == load_golden("cfg5_hist")["matrix_hash"]


def test_gamma_sets_bit_identical_to_reference(mdg):
    cases = load_golden("configs") + load_golden("kats") + load_golden("seeded")
    for case in cases:
        if "matrix" in case:
            rows, n = mdg.parse_matrix(case["matrix"])
        else:
            g = case["gen"]
            rows, n = mdg.gen_matrix(g["n"], g["k"], g["seed"], True), g["n"]
        gs = mdg.GammaSet.build(rows, n, case["trials"], case["seed"])
        assert gs.m == case["m"] and gs.k_last == case["k_last"], case["name"]
        assert gs.ranks == case["ranks"], case["name"]
        assert gs.column_perm == case["column_perm"], case["name"]
        assert [gs.hash(j) for j in range(gs.m)] == case["gamma_hash"], case["name"]
        if "gammas" in case:  # full rows for the known-answer codes
            for j in range(gs.m):
                got = ["".join("%016x" % int(w) for w in row) for row in gs.gamma(j)]
                assert got == case["gammas"][j], case["name"]


def test_hamming_gamma_structure(mdg):
    # test_gamma.cpp:38-51
    text = next(c for c in load_golden("kats") if c["name"] == "hamming_taps")["matrix"]
    rows, n = mdg.parse_matrix(text)
    gs = mdg.GammaSet.compute(rows, n)
    assert (gs.m, gs.k, gs.n, gs.ranks, gs.k_last) == (2, 4, 7, [4, 3], 3)
    g0 = gs.gamma(0)
    for r in range(4):
        for c in range(4):
            assert ((int(g0[r, 0]) >> c) & 1) == (r == c)


def test_rank_deficient_rejected_by_compute(mdg):
    # test_gamma.cpp:93-98
    G = np.zeros((2, 1), dtype=np.uint64)
    G[0, 0] = G[1, 0] = 1 << 1
    with pytest.raises(mdg.InvalidArgument):
        mdg.GammaSet.compute(G, 5)


def test_permutation_search_deterministic_and_never_worse(mdg):
    # test_gamma.cpp:100-119 (random_full_rank codes from the reference's generator)
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    for rep in range(12):
        text = ref.random_full_rank(8 + rep, 3 + rep % 5, 500 + rep)
        rows, n = mdg.parse_matrix(text)
        base = mdg.GammaSet.compute(rows, n)
        best = mdg.GammaSet.build(rows, n, 8, 1234)
        assert (best.m, best.k_last) >= (base.m, base.k_last)
        again = mdg.GammaSet.build(rows, n, 8, 1234)
        assert again.column_perm == best.column_perm


def test_bounds_spot_values(mdg):
    # test_gamma.cpp:121-134
    assert mdg.lower_bound(2, 1, 4, 3) == 3
    assert mdg.lower_bound(2, 3, 12, 12) == 8
    assert mdg.lower_bound(1, 4, 10, 4) == 0
    assert mdg.lower_bound(3, 2, 5, 5) == 9
    assert mdg.lower_bound(1, 2, 8, 8) == 3
    assert mdg.singleton_upper(7, 4) == 4
    assert mdg.singleton_upper(23, 12) == 12
    assert mdg.singleton_upper(5, 5) == 1
    with pytest.raises(mdg.InvalidArgument):
        mdg.singleton_upper(3, 4)


def _oracle_round(gs):
    """RoundRunner backed by the C oracle (round_stack restated) on the product's Gammas."""
    gam = [gs.gamma(j) for j in range(gs.m)]

    def fn(j, c, stop_at):
        return port.round_min(gam[j], gs.n, c)[0]
    return fn


@pytest.mark.parametrize("kind", ["kats", "seeded"])
def test_level_loop_trace_matches_reference(mdg, kind):
    """The native run_bz_loop (driven through the RoundRunner seam) reproduces the
    reference's per-round and per-level trace, d and g_final."""
    for case in load_golden(kind):
        rows, n = mdg.parse_matrix(case["matrix"])
        gs = mdg.GammaSet.build(rows, n, case["trials"], case["seed"])
        res = mdg.run_bz_loop(gs, _oracle_round(gs))
        assert res.d == case["d"], case["name"]
        assert res.rounds == case["rounds"], case["name"]
        assert res.levels == case["levels"], case["name"]
        assert res.g_final == case["g_final"], case["name"]


def test_level_loop_known_codes(mdg):
    # test_engines.cpp:227-255: Hamming d=3, g_final=1, two rounds; n=k: 0 rounds, d=1
    kats = {c["name"]: c for c in load_golden("kats")}
    rows, n = mdg.parse_matrix(kats["hamming_taps"]["matrix"])
    gs = mdg.GammaSet.compute(rows, n)
    res = mdg.run_bz_loop(gs, _oracle_round(gs))
    assert (res.d, res.g_final, len(res.rounds)) == (3, 1, 2)
    rows, n = mdg.parse_matrix(kats["identity_3"]["matrix"])
    gs = mdg.GammaSet.compute(rows, n)
    res = mdg.run_bz_loop(gs, _oracle_round(gs))
    assert (res.d, res.g_final, len(res.rounds)) == (1, 0, 0)


def test_level_cap_trace_prefix(mdg):
    """Level cap: the loop stops before any round of level cap+1 (config 4 semantics)."""
    cfg4 = next(c for c in load_golden("configs") if c["name"] == "cfg4")
    g = cfg4["gen"]
    rows = mdg.gen_matrix(g["n"], g["k"], g["seed"], True)
    gs = mdg.GammaSet.build(rows, g["n"], 10, g["seed"])
    res = mdg.run_bz_loop(gs, _oracle_round(gs), level_cap=3)
    assert res.capped
    assert res.rounds == cfg4["rounds"][: len(res.rounds)] and len(res.rounds) == 6
    assert res.levels == cfg4["levels"][:3]


def test_matrix_grammar(mdg):
    # test_cli.cpp:70-98
    good = ("# generator\n\n  7 4 \n# mid-stream comment\n1101000\n"
            "0110100\n\n0011010\n0001101\n")
    rows, n = mdg.parse_matrix(good)
    ham = "7 4\n1101000\n0110100\n0011010\n0001101\n"
    assert mdg.serialize_matrix(rows, n) == ham
    assert mdg.serialize_matrix(*mdg.parse_matrix(ham)) == ham
    bad = [("7 4\n11x1000\n0110100\n0011010\n0001101\n", "line 2, column 3", "symbols must be 0 or 1"),
           ("7 4\n110100\n", "line 2, column 7", "exactly 7 symbols"),
           ("7 4\n1101000\n0110100\n", "line 4, column 1", "expected 4 rows, got 2"),
           ("7 4 9\n", "line 1, column 1", "exactly: n k"),
           ("0 4\n", "line 1, column 1", ">= 1"),
           ("", "line 1, column 1", "missing header")]
    for text, pos, frag in bad:
        with pytest.raises(mdg.InvalidArgument) as ei:
            mdg.parse_matrix(text)
        assert pos in str(ei.value) and frag in str(ei.value)


def test_parse_errors_match_the_compiled_reference(mdg):
    """Every malformed (and odd but legal) text gets the reference parser's verdict: the same
    "line L, column C: message" from parse_matrix (io.cpp:33-73) in oracle/_ref, or the same
    matrix. Skipped where the compiled reference is absent."""
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    import random
    rng = random.Random(7)
    ham = "7 4\n1101000\n0110100\n0011010\n0001101\n"
    texts = ["", "\n\n", "# only a comment", "7", "7 x\n", "x 4\n", "-1 4\n1\n", "7 4 \t\r\n1101000\r\n0110100\r\n0011010\r\n0001101",
             "99999999999999999999999 4\n", "1048577 1\n", "3 1048577\n", "7 4\n1101000\n0110100\n0011010\n",
             "7 4\n1101000\n0110100\n0011010\n0001101\n0001101\n", "2 2\n10\n0 1\n", "2 2\n 10 \n\t01\t\n",
             "2 2\n10 # tail\n01\n", "+2 +2\n10\n01\n", "2 2\n#\n10\n\n\n01", "2 2\n10\n012\n", "2 2\n10\n0\n", "2.0 2\n10\n01\n"]
    for _ in range(300):  # mutations of a good file: a replaced, dropped or inserted character
        t = list(ham)
        for _ in range(rng.randint(1, 3)):
            pos = rng.randrange(len(t) + 1)
            op = rng.random()
            ch = rng.choice("01 \n#x2\t\r7-")
            if op < 0.4 and pos < len(t):
                t[pos] = ch
            elif op < 0.7 and pos < len(t):
                del t[pos]
            else:
                t.insert(pos, ch)
        texts.append("".join(t))
    checked_err = checked_ok = 0
    for text in texts:
        try:
            want = ref.trace(text, trials=1, seed=1, engine="stack", with_rows=False)
            want_err = None
        except RuntimeError as e:
            want, want_err = None, str(e)
        if want_err is not None and not want_err.startswith("line "):
            continue  # parsed, then rejected later (e.g. the zero matrix): not the parser's verdict
        if want_err is not None:
            with pytest.raises(mdg.InvalidArgument) as ei:
                mdg.parse_matrix(text)
            assert want_err in str(ei.value), (text, want_err, str(ei.value))
            checked_err += 1
        else:
            rows, n = mdg.parse_matrix(text)
            assert (n, rows.shape[0]) == (want["n"], want["k_input"] if "k_input" in want else rows.shape[0])
            checked_ok += 1
    assert checked_err > 50 and checked_ok > 5


def test_binomial_and_overflow(mdg):
    # test_enumeration.cpp:73-81
    for p in range(0, 40):
        for q in range(0, p + 1):
            from math import comb
            assert mdg.binomial(p, q) == comb(p, q)
    with pytest.raises(mdg.OverflowError_):
        mdg.binomial(128, 64)


def test_revolving_door_rank_unrank_exhaustive(mdg):
    """rank/unrank invert each other; consecutive ranks differ by one swap; every
    combination appears exactly once (k <= 12, all c)."""
    for k in range(1, 13):
        for c in range(1, k + 1):
            from math import comb
            N = comb(k, c)
            seen = set()
            prev = None
            for r in range(N):
                idx = mdg.rd_unrank(c, r)
                assert idx == sorted(idx) and idx[-1] < k
                assert mdg.rd_rank(idx) == r
                s = frozenset(idx)
                seen.add(s)
                if prev is not None:
                    assert len(prev ^ s) == 2
                prev = s
            assert len(seen) == N
    assert mdg.rd_unrank(3, 0) == [0, 1, 2]


def test_zero_and_degenerate_inputs(mdg):
    """row_basis of the zero matrix throws (f2core.cpp:92-97) -> invalid argument, never a
    device call; trials 0 is rejected like gamma.cpp:79-80."""
    Z = np.zeros((3, 1), dtype=np.uint64)
    with pytest.raises(mdg.InvalidArgument):
        mdg.GammaSet.build(Z, 10, 10, 1)
    G = mdg.gen_matrix(20, 5, 1, True)
    with pytest.raises(mdg.InvalidArgument):
        mdg.GammaSet.build(G, 20, 0, 1)
    with pytest.raises(mdg.InvalidArgument):
        mdg.GammaSet.compute(np.zeros((0, 1), dtype=np.uint64), 20)


def test_round_split_balances_codewords(mdg):
    """The multi-rank split of a round (mdg_plan_split, the cut chain_loop / mdg_round_split
    use): contiguous task ranges covering every task once, their codewords summing to C(k, c),
    each rank within one tile of 1/world of the codewords -- tiles differ in size (the last
    pivots' tiles are partial), so a task-count split is not balanced (engines.cpp:508-557
    splits by combinations for the same reason)."""
    from math import comb
    for (k, c, nw, resident) in [(64, 7, 2, 592), (64, 6, 2, 592), (200, 7, 4, 592), (200, 7, 7, 296),
                                 (200, 5, 4, 296), (32, 9, 7, 296), (100, 5, 8, 592), (40, 3, 2, 592)]:
        for world in (1, 2, 3, 8):
            ranges = [mdg.plan_split(k, c, nw, resident, r, world) for r in range(world)]
            assert ranges[0][0] == 0
            for a, b in zip(ranges, ranges[1:]):
                assert a[1] == b[0]
            assert sum(x[2] for x in ranges) == comb(k, c), (k, c, world)
            T = ranges[-1][1]
            tile_max = 256 * 8 * 256  # TX x YC (YC = 256 threads x R <= 8 items)
            for lo, hi, cw in ranges:
                assert abs(cw - comb(k, c) / world) <= tile_max, (k, c, nw, world, lo, hi, cw)
            assert T > 0
    import pytest
    with pytest.raises(mdg.InvalidArgument):
        mdg.plan_split(64, 7, 2, 592, 2, 2)
