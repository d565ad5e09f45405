"""GPU parity: the CUDA round kernels and the GPU front door against the
reference golden vectors and the C oracle (bit-exact: every result here is an
integer). Run on a B200 with ``pytest -m gpu``. Everything goes through the
C ABI (lib/libmdg.so)."""
import threading
from math import comb

import numpy as np
import pytest

from conftest import load_golden
from oracle import port

pytestmark = pytest.mark.gpu

KERNELS = [0, 1]  # tab, rd


def popcount_rows(rows, idx):
    acc = np.zeros(rows.shape[1], dtype=np.uint64)
    for r in idx:
        acc ^= rows[r]
    return sum(bin(int(x)).count("1") for x in acc), acc


# ------------------------------------------------------------------ rounds
@pytest.mark.parametrize("kernel", KERNELS)
def test_round_minima_vs_reference(mdg, device, kernel):
    device.set_kernel(kernel)
    for case in load_golden("rounds"):
        rows, n = mdg.parse_matrix(case["matrix"])
        device.load_gammas(rows, n, ranks=None)
        for lv in case["levels"]:
            out = device.round(0, lv["c"])
            assert out.min_weight == lv["min"], (case["n"], case["k"], lv, kernel)
            assert out.combinations == lv["combinations"]
            assert out.evaluated == lv["combinations"]
            idx = device.round_witness(0, lv["c"], out)
            assert len(set(idx)) == lv["c"]
            assert popcount_rows(rows, idx)[0] == lv["min"]


@pytest.mark.parametrize("kernel", KERNELS)
def test_round_random_shapes_vs_oracle(mdg, device, kernel):
    """Raw matrices of many widths (every NW template 1..16) and levels vs the oracle."""
    rng = np.random.default_rng(7)
    device.set_kernel(kernel)
    for n in [5, 31, 32, 33, 64, 65, 97, 128, 160, 200, 256, 300, 384, 450, 512, 520, 700, 900, 1024]:
        k = int(rng.integers(6, 26))
        W = (n + 63) // 64
        rows = rng.integers(0, 2**63, size=(k, W), dtype=np.uint64)
        if n % 64:
            rows[:, -1] &= np.uint64((1 << (n % 64)) - 1)
        device.load_gammas(rows, n, ranks=None)
        for c in range(1, min(k, 5) + 1):
            w, combos = port.round_min(rows, n, c)
            out = device.round(0, c)
            assert (out.min_weight, out.evaluated) == (w, combos), (n, k, c, kernel)


@pytest.mark.parametrize("kernel", KERNELS)
def test_identity_elision_rounds_vs_oracle(mdg, device, kernel):
    """Gamma sets with full and partial identity blocks (compacted rows + identity count)
    give the oracle's per-round minima on the uncompacted matrices."""
    device.set_kernel(kernel)
    for (n, k, seed) in [(80, 40, 1), (300, 200, 11), (50, 30, 4), (70, 20, 5), (45, 40, 6)]:
        G = mdg.gen_matrix(n, k, seed, True)
        gs = mdg.GammaSet.build(G, n, 3, seed)
        device.load_gset(gs)
        for j in range(gs.m):
            g = gs.gamma(j)
            for c in range(1, 4):
                w, combos = port.round_min(g, n, c)
                out = device.round(j, c)
                assert (out.min_weight, out.evaluated) == (w, combos), (n, k, j, c, kernel)
                idx = device.round_witness(j, c, out)
                assert popcount_rows(g, idx)[0] == w


def test_histogram_cfg5(mdg, device):
    h = load_golden("cfg5_hist")
    rows = mdg.gen_matrix(256, 100, 3, identity=False)
    device.load_gammas(rows, 256, ranks=None)
    for lv in h["levels"]:
        out, hist = device.round_hist(0, lv["c"], 256)
        assert hist.tolist() == lv["hist"], lv["c"]
        assert out.min_weight == lv["min"]
        assert out.evaluated == lv["count"] == comb(100, lv["c"])
        full = device.round(0, lv["c"])
        assert full.min_weight == lv["min"]


def test_histogram_level6_vs_reference(mdg, device):
    """The histogram kernel at its steady-state size: level 6 of config 5's matrix, all
    C(100, 6) = 1,192,052,400 codewords, bit-exact against the reference's histogram -- whole
    and as the sum of three ranks' shares."""
    lv = load_golden("cfg5_hist_c6")["level"]
    rows = mdg.gen_matrix(256, 100, 3, identity=False)
    device.load_gammas(rows, 256, ranks=None)
    out, hist = device.round_hist(0, 6, 256)
    assert hist.tolist() == lv["hist"] and out.min_weight == lv["min"] == 81
    assert out.evaluated == lv["count"] == comb(100, 6)
    total = np.zeros(257, dtype=np.uint64)
    for r in range(3):
        o, h, reduced = device.round_hist_dist(0, 6, 256, r, 3)
        total += h
    assert total.tolist() == lv["hist"]


def test_histogram_split_across_ranks_sums_to_golden(mdg):
    """SURVEY.md 8e, config 5 at N > 1: every rank counts its contiguous share of the histogram
    kernel's tiles; the partial histograms (no communicator: the caller sums) add up to the
    reference's, the shares partition the tiles and are balanced in codewords."""
    from math import comb
    h = load_golden("cfg5_hist")
    M = mdg.gen_matrix(256, 100, 3, identity=False)
    for world in (2, 3, 8):
        devs = [mdg.Device(0) for _ in range(world)]
        try:
            for d in devs:
                d.load_gammas(M, 256, ranks=None)
            for lv in h["levels"]:
                c = lv["c"]
                total = np.zeros(257, dtype=np.uint64)
                edges, evaluated = [], []
                for r, d in enumerate(devs):
                    out, hist, reduced = d.round_hist_dist(0, c, 256, r, world)
                    assert not reduced
                    total += hist
                    edges.append((out.task_lo, out.task_hi))
                    evaluated.append(out.evaluated)
                assert total.tolist() == lv["hist"], (world, c)
                assert edges[0][0] == 0 and all(edges[i][1] == edges[i + 1][0] for i in range(world - 1))
                assert sum(evaluated) == comb(100, c)
                if c == 5:  # each share within a few tiles of 1 / world
                    assert max(evaluated) - min(evaluated) <= 0.05 * comb(100, c) / world + 4 * 1024 * 128
            out, hist, reduced = devs[0].round_hist_dist(0, 4, 256, 0, 1)
            assert not reduced and hist.tolist() == h["levels"][3]["hist"]
            with pytest.raises(Exception):
                devs[0].round_hist_dist(0, 4, 256, 2, 2)
        finally:
            for d in devs:
                d.close()


def test_histogram_with_identity_vs_oracle(mdg, device):
    G = mdg.gen_matrix(70, 20, 5, True)
    gs = mdg.GammaSet.build(G, 70, 3, 5)
    device.load_gset(gs)
    for j in range(gs.m):
        for c in (1, 2, 3, 4):
            w, hist_ref = port.round_hist(gs.gamma(j), 70, c)
            out, hist = device.round_hist(j, c, 70)
            assert hist.tolist() == hist_ref.tolist() and out.min_weight == w


@pytest.mark.parametrize("kernel", KERNELS)
def test_partition_covers_round(mdg, device, kernel):
    """Task ranges (the multi-GPU split) partition the round exactly."""
    device.set_kernel(kernel)
    G = mdg.gen_matrix(128, 64, 1, True)
    gs = mdg.GammaSet.build(G, 128, 10, 1)
    device.load_gset(gs)
    for c in (2, 3, 4):
        full = device.round(0, c)
        T = device.tasks(0, c)
        for world in (2, 3, 8):
            parts = [device.round_range(0, c, T * r // world, T * (r + 1) // world) for r in range(world)]
            assert sum(p.evaluated for p in parts) == comb(64, c)
            assert min(p.min_weight for p in parts) == full.min_weight
            assert min(p.argmin_key for p in parts) == full.argmin_key


@pytest.mark.parametrize("kernel", KERNELS)
def test_early_exit_is_exact(mdg, device, kernel):
    """stop_at: the round stops once a weight <= stop_at exists; the returned minimum is
    then <= stop_at and is a real codeword weight."""
    device.set_kernel(kernel)
    G = mdg.gen_matrix(128, 64, 1, True)
    gs = mdg.GammaSet.build(G, 128, 10, 1)
    device.load_gset(gs)
    c = 7  # large enough that not every task starts before the bound fires
    full = device.round(0, c)
    early = device.round(0, c, stop_at=full.min_weight + 3)
    assert early.min_weight <= full.min_weight + 3 and early.min_weight >= full.min_weight
    assert early.stopped_early and early.evaluated < full.evaluated
    idx = device.round_witness(0, c, early)
    g0 = gs.gamma(0)
    assert popcount_rows(g0, idx)[0] == early.min_weight


def test_kernels_agree_on_keys_weight(mdg, device):
    G = mdg.gen_matrix(256, 32, 7, True)
    gs = mdg.GammaSet.build(G, 256, 10, 7)
    device.load_gset(gs)
    for j in range(gs.m):
        for c in (3, 5):
            device.set_kernel(0)
            a = device.round(j, c)
            device.set_kernel(1)
            b = device.round(j, c)
            assert a.min_weight == b.min_weight and a.evaluated == b.evaluated
    device.set_kernel(0)


def test_round_argument_errors(mdg, device):
    rows = mdg.gen_matrix(40, 10, 2, True)
    device.load_gammas(rows, 40, ranks=None)
    with pytest.raises(mdg.InvalidArgument):
        device.round(0, 0)
    with pytest.raises(mdg.InvalidArgument):
        device.round(0, 11)
    with pytest.raises(mdg.InvalidArgument):
        device.round(1, 1)
    out = device.round(0, 10)  # c = k: the single all-rows combination
    assert out.evaluated == 1
    w = popcount_rows(rows, range(10))[0]
    assert out.min_weight == w
    with pytest.raises(mdg.InvalidArgument):  # identity block missing at the claimed rank
        device.load_gammas(np.ones((3, 1), dtype=np.uint64), 10, ranks=[3])


@pytest.mark.parametrize("kernel", KERNELS)
def test_bounded_round_vs_oracle(mdg, device, kernel):
    """Bound-pruned rounds return min(true minimum, cutoff), flag `bounded` exactly when no
    codeword lies below the cutoff, and name a witness of the returned weight otherwise."""
    device.set_kernel(kernel)
    for (n, k, seed) in [(128, 64, 1), (300, 200, 11), (256, 32, 7), (70, 20, 5)]:
        G = mdg.gen_matrix(n, k, seed, True)
        gs = mdg.GammaSet.build(G, n, 10, seed)
        device.load_gset(gs)
        for j in range(gs.m):
            g = gs.gamma(j)
            for c in (2, 3, 4):
                w, _ = port.round_min(g, n, c)
                for cutoff in (w - 3, w, w + 1, w + 5, 1, n + 1):
                    if cutoff < 1:
                        continue
                    out = device.round_bounded(j, c, cutoff)
                    assert out.min_weight == min(w, cutoff), (n, k, j, c, cutoff, kernel)
                    assert out.bounded == (w >= cutoff), (n, k, j, c, cutoff)
                    if not out.bounded:
                        idx = device.round_witness(j, c, out)
                        assert popcount_rows(g, idx)[0] == w


# -------------------------------------------------------------- front door
def _check_run(res, case, name, exact=True):
    if exact:
        assert res.rounds == case["rounds"], name
        assert not any(res.round_bounded), name
    else:
        # bounded rounds: w = min(exact w, U before the round); identical U after each round
        U = case["n"] - case["k"] + 1
        exp = []
        for c, j, w, Ua in case["rounds"]:
            exp.append([c, j, min(w, U), Ua])
            assert res.round_bounded[len(exp) - 1] == (1 if w >= U else 0), (name, c, j)
            U = Ua
        assert res.rounds == exp, name
    assert res.levels == case["levels"][: len(res.levels)] and len(res.levels) == len(case["levels"]), name
    assert res.m == case["m"] and res.k_last == case["k_last"], name
    assert res.g_final == case["g_final"], name
    assert res.column_perm == case["column_perm"], name
    assert res.gamma_hash == case["gamma_hash"], name
    assert res.witness_ok, name
    wt = sum(bin(int(x)).count("1") for x in res.witness)
    assert wt == res.d, name


@pytest.mark.parametrize("exact", [True, False])
@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("kind", ["kats", "seeded"])
def test_min_weight_small_codes(mdg, device, kind, kernel, exact):
    for case in load_golden(kind):
        rows, n = mdg.parse_matrix(case["matrix"])
        res = mdg.min_weight(rows, n, case["trials"], case["seed"], kernel=kernel, device=device,
                             exact_rounds=exact)
        assert res.d == case["d"] == case["d_brute"], case["name"]
        _check_run(res, case, case["name"], exact)


@pytest.mark.parametrize("exact", [True, False])
@pytest.mark.parametrize("name", ["cfg1", "cfg2_s1", "cfg2_s2", "cfg2_s3", "cfg2_s4", "cfg2_s5",
                                  "cfg2_s6", "cfg2_s7", "cfg2_s8", "cfg3", "cfg4"])
def test_min_weight_configs(mdg, device, name, exact):
    case = next(c for c in load_golden("configs") if c["name"] == name)
    g = case["gen"]
    rows = mdg.gen_matrix(g["n"], g["k"], g["seed"], True)
    res = mdg.min_weight(rows, g["n"], case["trials"], case["seed"], level_cap=case["level_cap"],
                         device=device, exact_rounds=exact)
    if case["capped"]:
        assert res.capped and res.d == case["U_final"]
    else:
        assert not res.capped and res.d == case["d"]
    _check_run(res, case, name, exact)
    # the witness lies in the code spanned by G (rank does not grow)
    assert port.rank(np.vstack([rows, res.witness[None, :]]), g["n"]) == port.rank(rows, g["n"])


def test_min_weight_cfg4_cap6(mdg, device):
    import os
    from conftest import GOLD
    if not os.path.exists(os.path.join(GOLD, "configs_cap4_6.json")):
        pytest.skip("cap-6 golden not generated")
    case = next(c for c in load_golden("configs_cap4_6") if c["name"] == "cfg4")
    g = case["gen"]
    rows = mdg.gen_matrix(g["n"], g["k"], g["seed"], True)
    res = mdg.min_weight(rows, g["n"], 10, g["seed"], level_cap=6, device=device)
    assert res.capped and res.d == case["U_final"]
    _check_run(res, case, "cfg4_cap6", exact=False)


def test_dist_two_ranks_threaded(mdg):
    """The multi-rank front door (rank-range split + per-round min reduction) with two
    ranks on one GPU as two host threads exchanging keys through a barrier (no kernel
    ever waits on another); results equal the single-rank run."""
    case = next(c for c in load_golden("configs") if c["name"] == "cfg2_s8")
    g = case["gen"]
    rows = mdg.gen_matrix(g["n"], g["k"], g["seed"], True)
    world = 2
    slots = [None] * world
    bar = threading.Barrier(world)
    results = [None] * world

    def reducer_for(rank):
        def red(keys):
            slots[rank] = keys.copy()
            bar.wait()
            out = np.minimum.reduce([s for s in slots])
            bar.wait()
            return out
        return red

    calls = [0] * world

    def counting(rank, red):
        def f(keys):
            calls[rank] += 1
            return red(keys)
        return f

    for split_min in (1, 0, 10**6):  # every round split / default (none here) / from level 5
        calls[:] = [0] * world

        def worker(rank):
            dev = mdg.Device(0)
            results[rank] = mdg.min_weight_dist(rows, g["n"], rank, world,
                                                counting(rank, reducer_for(rank)), trials=10,
                                                seed=g["seed"], device=dev, split_min=split_min)
            dev.close()

        ts = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        for r in range(world):
            res = results[r]
            assert res.d == case["d"]
            _check_run(res, case, f"rank{r}", exact=False)
        split_rounds = sum(1 for c, j, w, U in case["rounds"] if comb(64, c) >= max(split_min, 1)) \
            if split_min else 0
        assert calls[0] == calls[1] >= split_rounds, (split_min, calls)
        if split_min == 0:
            assert calls == [0, 0]  # cfg2 seed 8 never reaches 2e8-codeword rounds


@pytest.mark.parametrize("shared", [True, False])
@pytest.mark.parametrize("world", [2, 3])
def test_min_weight_multi_group_split(mdg, world, shared, monkeypatch):
    """The chained split path (each rank's contiguous tile range of every round of at least
    split_min codewords, the per-round key min-reduced IN STREAM before the round closes --
    the production multi-GPU path, here with the in-process exchange group instead of NCCL:
    cudaStreamWaitEvent on the members' round events, then a min kernel; no kernel waits on
    another) with `world` contexts on one GPU: d, per-round and per-level trace, Gamma set and
    witness equal the golden on every rank; the ranks' evaluated counts add up to the
    single-rank count of the split rounds; levels below split_min still run fused. `shared`:
    the members also share one round key word that every tile result goes to and every tile
    fetch polls (one rank's find prunes the others' tiles); MDG_NO_SHARED_BOUND turns it off."""
    if shared:
        monkeypatch.delenv("MDG_NO_SHARED_BOUND", raising=False)
    else:
        monkeypatch.setenv("MDG_NO_SHARED_BOUND", "1")
    devs = [mdg.Device(0) for _ in range(world)]
    cases = {c["name"]: c for c in load_golden("configs")}
    cases["cfg4_cap6"] = next(c for c in load_golden("configs_cap4_6") if c["name"] == "cfg4")
    try:
        for name in ("cfg1", "cfg2_s1", "cfg2_s8", "cfg3", "cfg4_cap6"):
            case = cases[name]
            g = case["gen"]
            cap = case["level_cap"] if case["capped"] else 0
            rows = mdg.gen_matrix(g["n"], g["k"], g["seed"], True)
            single = mdg.min_weight(rows, g["n"], 10, g["seed"], level_cap=cap, device=devs[0])
            for split_min in ((1, 0, 10**6, 1 << 62) if name != "cfg4_cap6" else (0,)):
                runs = mdg.min_weight_multi(rows, g["n"], devs, trials=10, seed=g["seed"],
                                            level_cap=cap, split_min=split_min)
                assert len(runs) == world
                for r, res in enumerate(runs):
                    assert res.d == (case["U_final"] if cap else case["d"]), (name, r)
                    assert res.capped == bool(cap)
                    _check_run(res, case, f"{name} rank{r} split_min={split_min}", exact=False)
                if split_min == 1 and name == "cfg2_s1":  # every round split: each rank
                    # evaluates about 1/world of the codewords of the single-rank run
                    assert max(r_.evaluated for r_ in runs) < 0.75 * single.evaluated, name
    finally:
        for d in devs:
            d.close()


def test_min_weight_multi_group_split_rd(mdg):
    """The split path with the revolving-door kernel's plans (rd tiles are revolving-door rank
    ranges of the prefixes; tab_split cuts them the same way): two contexts, every round split,
    golden traces on both ranks."""
    devs = [mdg.Device(0) for _ in range(2)]
    try:
        for name in ("cfg1", "cfg2_s8", "cfg3"):
            case = next(c for c in load_golden("configs") if c["name"] == name)
            g = case["gen"]
            rows = mdg.gen_matrix(g["n"], g["k"], g["seed"], True)
            runs = mdg.min_weight_multi(rows, g["n"], devs, trials=10, seed=g["seed"],
                                        kernel=mdg.KERNEL_RD, split_min=1)
            for r, res in enumerate(runs):
                _check_run(res, case, f"rd {name} rank{r}", exact=False)
    finally:
        for d in devs:
            d.close()


def test_min_weight_multi_group_stress(mdg):
    """Many short split rounds through a four-member exchange group (every round of config 1
    and config 2 seed 8 split, 12 runs): members that run ahead of the others must never make a
    slow member read the next round's slots (the barrier snapshots them); every rank's trace
    equals the golden every time."""
    devs = [mdg.Device(0) for _ in range(4)]
    try:
        for name in ("cfg1", "cfg2_s8"):
            case = next(c for c in load_golden("configs") if c["name"] == name)
            g = case["gen"]
            rows = mdg.gen_matrix(g["n"], g["k"], g["seed"], True)
            for _ in range(6):
                for r, res in enumerate(mdg.min_weight_multi(rows, g["n"], devs, trials=10,
                                                             seed=g["seed"], split_min=1)):
                    _check_run(res, case, f"stress {name} rank{r}", exact=False)
    finally:
        for d in devs:
            d.close()


def test_min_weight_multi_errors(mdg):
    """Argument checks of the single-process multi front door, and a member failure (a level
    beyond the device limit would be hit by every rank at once; here a bad context list)
    surfaces as an error on the caller instead of a hang."""
    rows = mdg.gen_matrix(80, 40, 1, True)
    d0 = mdg.Device(0)
    try:
        with pytest.raises(mdg.InvalidArgument):
            mdg.min_weight_multi(rows, 80, [d0, d0])  # the same context twice
        with pytest.raises(mdg.InvalidArgument):
            mdg.min_weight_multi(rows, 80, [])
        # the group marker is not a host reducer
        with pytest.raises(mdg.InvalidArgument):
            mdg.min_weight_dist(rows, 80, 0, 2, "group", trials=10, seed=1, device=d0)
        one = mdg.min_weight_multi(rows, 80, [d0], trials=10, seed=1)
        assert one[0].d == 9
    finally:
        d0.close()


# ------------------------------------------------------------ brute force
@pytest.mark.parametrize("kind", ["kats", "seeded"])
def test_brute_force_vs_reference(mdg, device, kind):
    """GPU Gray-code brute force (brute_force_gray, engines.cpp:480-558) == the reference's
    brute-force d on every known-answer and seeded code; the witness has weight d."""
    for case in load_golden(kind):
        rows, n = mdg.parse_matrix(case["matrix"])
        res = mdg.brute_force(rows, n, device=device)
        assert res.d == case["d_brute"], case["name"]
        assert res.witness_ok and (res.m, res.k_last, res.g_final) == (0, 0, 0), case["name"]
        assert res.combinations == (1 << case["k"]) - 1 == res.evaluated, case["name"]


def test_brute_force_cfg1_k40(mdg, device):
    """Config 1 by exhaustion: all 2^40 - 1 codewords, d = 9 (== the BZ result)."""
    G = mdg.gen_matrix(80, 40, 1, True)
    res = mdg.brute_force(G, 80, device=device)
    assert res.d == 9 and res.witness_ok
    assert res.evaluated == (1 << 40) - 1
    with pytest.raises(mdg.InvalidArgument):
        mdg.brute_force(G, 80, brute_cap=39, device=device)


def test_nccl_single_rank(mdg):
    """The in-stream NCCL allreduce(min) path of the chained loop, with one rank."""
    case = next(c for c in load_golden("configs") if c["name"] == "cfg2_s8")
    g = case["gen"]
    rows = mdg.gen_matrix(g["n"], g["k"], g["seed"], True)
    dev = mdg.Device(0)
    dev.nccl_init(mdg.nccl_unique_id(), 0, 1)
    for split_min in (1, 0):  # every round through NCCL / the default (none at this size)
        res = mdg.min_weight_dist(rows, g["n"], 0, 1, "nccl", trials=10, seed=g["seed"],
                                  device=dev, split_min=split_min)
        assert res.d == case["d"]
        _check_run(res, case, "nccl1", exact=False)
    dev.close()


def test_cli_json_record(mdg, tmp_path):
    """`mindist mindist FILE --algorithm gpu|brute` prints the reference's JSON record
    (cli.cpp:223-238) plus the new keys; exit code 0."""
    import json
    import os
    import subprocess
    from conftest import ROOT
    exe = os.path.join(ROOT, "paper_1911_08963_b200", "bin", "mindist")
    kats = {c["name"]: c for c in load_golden("kats")}
    f = tmp_path / "golay.txt"
    f.write_text(kats["golay_23_12"]["matrix"])
    for alg in ("gpu", "brute"):
        r = subprocess.run([exe, "mindist", str(f), "--algorithm", alg, "--seed", "1"],
                           capture_output=True, text=True, timeout=120)
        assert r.returncode == 0, r.stderr
        rec = json.loads(r.stdout)
        for key in ("d", "n", "k", "algorithm", "m", "k_last", "g_final", "row_additions",
                    "combinations", "wall_seconds", "seed", "workers", "witness", "witness_ok"):
            assert key in rec, key
        assert rec["d"] == 7 and rec["n"] == 23 and rec["k"] == 12 and rec["witness_ok"]
        assert rec["algorithm"] == alg
        assert rec["witness"].count("1") == 7
        if alg == "gpu":
            case = kats["golay_23_12"]
            assert rec["levels"] == case["levels"]
            assert (rec["m"], rec["k_last"], rec["g_final"]) == (case["m"], case["k_last"],
                                                                 case["g_final"])
    r = subprocess.run([exe, "mindist", str(f), "--seed", "1", "--pretty", "--exact-rounds"],
                       capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "d:             7" in r.stdout
    # result_to_text's twelve lines in the reference's order (cli.cpp:240-255)
    keys = [ln.split(":")[0] for ln in r.stdout.splitlines()]
    assert keys == ["d", "n", "k", "algorithm", "m", "k_last", "g_final", "row_additions",
                    "combinations", "wall_seconds", "seed", "workers"], keys
    # workers: --workers, else MINDIST_WORKERS, else 1 (cli.cpp:78-79), echoed in the record
    for env, args, want in [({}, [], 1), ({"MINDIST_WORKERS": "6"}, [], 6),
                            ({"MINDIST_WORKERS": "6"}, ["--workers", "3"], 3)]:
        r = subprocess.run([exe, "mindist", str(f), "--seed", "1"] + args, capture_output=True,
                           text=True, timeout=120, env=dict(os.environ, **env))
        assert r.returncode == 0 and json.loads(r.stdout)["workers"] == want, (env, args, r.stderr)
    # a reference command line with CPU-engine options runs unchanged on the GPU engine
    r = subprocess.run([exe, "mindist", str(f), "--algorithm", "saved", "--s", "5", "--unroll", "2",
                        "--workers", "8", "--schedule", "dynamic", "--prefix", "3", "--order",
                        "left_lex", "--trials", "10", "--seed", "1", "--gamma-search", "gpu"],
                       capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    rec = json.loads(r.stdout)
    assert rec["d"] == 7 and rec["levels"] == kats["golay_23_12"]["levels"]
    # several files: one record each, in order, run as one batch
    files = []
    for name in ("golay_23_12", "hamming_taps", "ext_golay_24_12", "rank_deficient_14_5", "repetition_9"):
        if name in kats:
            p = tmp_path / f"{name}.txt"
            p.write_text(kats[name]["matrix"])
            files.append((p, kats[name]))
    r = subprocess.run([exe, "mindist"] + [str(p) for p, _ in files] + ["--seed", "1"],
                       capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    recs = [json.loads(line) for line in r.stdout.splitlines()]
    assert [x["d"] for x in recs] == [c["d"] for _, c in files]


@pytest.mark.parametrize("kernel", KERNELS)
def test_cfg4_cap7_vs_reference(mdg, device, kernel):
    """Config 4 to level cap 7 (4.7e12 codewords, BASELINE.md's throughput and scaling case)
    against the REFERENCE: tests/golden/configs_cap4_7.json is the reference's own cap-6 trace
    extended by its level-7 rounds, each computed by the reference's scheduled_round on the
    reference-built Gamma matrices (oracle/make_cfg4_c7.py, ~2 h on 8 cores). Both kernels
    (tab: bound-pruned prefix-sum tiles; rd: revolving-door walk) give its bounded-round trace,
    (L, U) levels and Gamma set; the witness is verified."""
    case = next(c for c in load_golden("configs_cap4_7") if c["name"] == "cfg4")
    g = case["gen"]
    G = mdg.gen_matrix(g["n"], g["k"], g["seed"], True)
    r = mdg.min_weight(G, g["n"], 10, g["seed"], level_cap=7, kernel=kernel, device=device)
    assert r.capped and r.d == case["U_final"]
    _check_run(r, case, f"cfg4_cap7 kernel={kernel}", exact=False)


@pytest.mark.gpu
def test_graft_smoke():
    """The driver's smoke() (config 1 in exact and bounded round modes + a config-5 histogram)."""
    import __graft_entry__
    __graft_entry__.smoke()


@pytest.mark.parametrize("streams", [1, 3])
def test_min_weight_batch_equals_single(mdg, device, streams):
    """The batch front door (several codes in flight on their own streams) returns, code by
    code, the golden result: d, per-round and per-level trace, Gamma set and a witness."""
    cases = [c for c in load_golden("configs") if not c["capped"]]
    mats, ns, seeds = [], [], []
    for case in cases:
        g = case["gen"]
        mats.append(mdg.gen_matrix(g["n"], g["k"], g["seed"], True))
        ns.append(g["n"])
        seeds.append(case["seed"])
    runs = mdg.min_weight_batch(mats, ns, trials=10, seed=seeds, device=device, streams=streams)
    assert len(runs) == len(cases)
    for res, case in zip(runs, cases):
        assert not res.capped and res.d == case["d"], case["name"]
        _check_run(res, case, case["name"], exact=False)
    with pytest.raises(mdg.InvalidArgument):  # a zero matrix fails the whole batch
        mdg.min_weight_batch([mats[0], np.zeros_like(mats[0])], 80, device=device, streams=2)
    assert mdg.min_weight_batch([], 80, device=device) == []


def test_bz_loop_batch_equals_single(mdg):
    """mdg_bz_loop_device_batch: the resident loops of eight config-2 codes (and a mixed set)
    through the library's worker pool equal the per-code loops; repeated calls reuse the pool."""
    cases = {c["name"]: c for c in load_golden("configs")}
    names = [f"cfg2_s{s}" for s in range(1, 9)] + ["cfg1", "cfg3"]
    devs, gsets = [], []
    for name in names:
        g = cases[name]["gen"]
        G = mdg.gen_matrix(g["n"], g["k"], g["seed"], True)
        gs = mdg.GammaSet.build(G, g["n"], 10, g["seed"])
        d = mdg.Device(0)
        d.load_gset(gs)
        devs.append(d)
        gsets.append(gs)
    try:
        for streams in (1, 3, 4, 16):
            for kernel in KERNELS:
                runs = mdg.bz_loop_batch(devs, gsets, kernel=kernel, streams=streams)
                for name, r in zip(names, runs):
                    _check_run(r, cases[name], name, exact=False)
        single = [d.bz_loop(gs) for d, gs in zip(devs, gsets)]
        for a, b in zip(single, mdg.bz_loop_batch(devs, gsets)):
            assert (a.d, a.rounds, a.levels, a.witness_ok) == (b.d, b.rounds, b.levels, b.witness_ok)
        with pytest.raises(mdg.InvalidArgument):
            mdg.bz_loop_batch([devs[0], devs[0]], gsets[:2])
    finally:
        for d in devs:
            d.close()


def test_pruning_off_same_minima(mdg, device):
    """mdg_set_pruning(0) (every codeword's weight exact) returns the same round minima."""
    for (n, k, seed) in [(128, 64, 1), (300, 200, 11), (256, 32, 7)]:
        G = mdg.gen_matrix(n, k, seed, True)
        gs = mdg.GammaSet.build(G, n, 10, seed)
        device.load_gset(gs)
        for j in range(gs.m):
            for c in (2, 3, 4):
                a = device.round(j, c)
                device.set_pruning(False)
                b = device.round(j, c)
                device.set_pruning(True)
                assert (a.min_weight, a.evaluated) == (b.min_weight, b.evaluated), (n, k, j, c)


def test_witness_after_plan_switch(mdg, device):
    """A round's witness decodes with the tile plan the round ran on (plan_tag), even after
    the caller switches pruning or the kernel in between (the plans differ); a key from
    another Gamma set fails loudly (the decoded rows are re-weighed) instead of returning
    a wrong combination."""
    G = mdg.gen_matrix(128, 64, 1, True)
    gs = mdg.GammaSet.build(G, 128, 10, 1)
    device.load_gset(gs)
    rows = gs.gamma(0)
    try:
        for c in (3, 4, 5):
            for first, then in (((True, 0), (False, 0)), ((False, 0), (True, 1)), ((True, 1), (True, 0))):
                device.set_pruning(first[0])
                device.set_kernel(first[1])
                o = device.round(0, c)
                device.set_pruning(then[0])
                device.set_kernel(then[1])
                idx = device.round_witness(0, c, o)
                assert popcount_rows(rows, idx)[0] == o.min_weight, (c, first, then)
    finally:
        device.set_pruning(True)
        device.set_kernel(0)
    o = device.round(0, 4)
    other = mdg.GammaSet.build(mdg.gen_matrix(128, 64, 2, True), 128, 10, 2)
    device.load_gset(other)
    with pytest.raises(mdg.MdgError):
        device.round_witness(0, 4, o)


def _sparse_code(rng, k, n, density):
    """A random full-rank k x n matrix with sparse columns: column sets of size k are often
    rank-deficient, so (m, k_last) depends on the column order."""
    from oracle import port
    while True:
        dense = (rng.random((k, n)) < density).astype(np.uint64)
        W = (n + 63) // 64
        rows = np.zeros((k, W), dtype=np.uint64)
        for c in range(n):
            rows[:, c // 64] |= dense[:, c] << np.uint64(c % 64)
        if port.rank(rows, n) == k:
            return rows


def test_gpu_permutation_search_equals_host(mdg, device):
    """mdg_gset_build_gpu (one warp per trial) returns the host search's Gamma set bit for
    bit: same (m, k_last), ranks, column_perm and Gammas for every trial count."""
    rng = np.random.default_rng(5)
    cases = []
    for case in load_golden("kats") + load_golden("seeded")[:40]:
        rows, n = mdg.parse_matrix(case["matrix"])
        cases.append((rows, n))
    for (k, n, dens) in [(12, 30, 0.15), (20, 50, 0.12), (30, 70, 0.08), (40, 90, 0.06),
                         (64, 128, 0.5), (70, 150, 0.04), (100, 260, 0.03)]:
        cases.append((_sparse_code(rng, k, n, dens), n))
    cases.append((mdg.gen_matrix(300, 200, 11, True), 300))
    varied = 0
    for rows, n in cases:
        try:
            base = mdg.GammaSet.compute(rows, n)
        except mdg.InvalidArgument:  # rank-deficient input: build() takes row_basis first
            base = None
        for trials in (1, 10, 257):
            for seed in (0, 7):
                h = mdg.GammaSet.build(rows, n, trials, seed)
                g = mdg.GammaSet.build(rows, n, trials, seed, device=device)
                assert (g.m, g.k_last, g.ranks) == (h.m, h.k_last, h.ranks), (n, trials, seed)
                assert g.column_perm == h.column_perm, (n, trials, seed)
                assert [g.hash(j) for j in range(g.m)] == [h.hash(j) for j in range(h.m)]
                if base is not None and (h.m, h.k_last) != (base.m, base.k_last):
                    varied += 1
    assert varied > 0  # some cases really depend on the permutation


def test_min_weight_gpu_gamma_search(mdg, device):
    for name in ("cfg1", "cfg2_s3"):
        case = next(c for c in load_golden("configs") if c["name"] == name)
        g = case["gen"]
        rows = mdg.gen_matrix(g["n"], g["k"], g["seed"], True)
        res = mdg.min_weight(rows, g["n"], case["trials"], case["seed"], device=device,
                             gamma_search="gpu")
        assert res.d == case["d"]
        _check_run(res, case, name, exact=False)


def test_fused_levels_equal_per_round_launches(mdg):
    """Chained loops with fused levels (default) and with one launch per round
    (MDG_FUSE_MAX=0) give identical traces, d and witness weights in both round modes."""
    import os
    fused = mdg.Device(0)
    os.environ["MDG_FUSE_MAX"] = "0"
    try:
        single = mdg.Device(0)
    finally:
        del os.environ["MDG_FUSE_MAX"]
    codes = []
    for name in ("cfg1", "cfg2_s3", "cfg3"):
        case = next(c for c in load_golden("configs") if c["name"] == name)
        g = case["gen"]
        codes.append((mdg.gen_matrix(g["n"], g["k"], g["seed"], True), g["n"], case["seed"]))
    for case in load_golden("seeded")[:60]:
        rows, n = mdg.parse_matrix(case["matrix"])
        codes.append((rows, n, case["seed"]))
    for rows, n, seed in codes:
        for exact in (False, True):
            a = mdg.min_weight(rows, n, 10, seed, device=fused, exact_rounds=exact)
            b = mdg.min_weight(rows, n, 10, seed, device=single, exact_rounds=exact)
            assert (a.d, a.rounds, a.levels, a.round_bounded) == (b.d, b.rounds, b.levels, b.round_bounded)
            assert a.witness_ok and b.witness_ok
    fused.close()
    single.close()


@pytest.mark.parametrize("n,k,seed,cap", [(512, 16, 1, 0), (1024, 8, 2, 0), (100, 99, 3, 0),
                                          (64, 64, 4, 0), (300, 150, 5, 3), (301, 150, 6, 3),
                                          (200, 3, 7, 0), (40, 1, 8, 0), (96, 2, 9, 0),
                                          (1000, 40, 10, 2), (130, 64, 11, 4)])
def test_unusual_shapes_vs_oracle(mdg, device, n, k, seed, cap):
    """Shapes far from the BASELINE configs -- many Gammas (m up to 96, beyond the fused-level
    limit), one-row codes, n = k and n = k + 1, 32-word compacted rows, partial blocks --
    through the front door in both round modes, against the C oracle's trace."""
    G = mdg.gen_matrix(n, k, seed, True)
    ref = port.min_weight(port.gen_matrix(n, k, seed, True), n, 10, seed, level_cap=cap)
    for exact in (True, False):
        res = mdg.min_weight(G, n, 10, seed, level_cap=cap, device=device, exact_rounds=exact)
        assert (res.d, res.capped, res.m, res.k_last) == (ref.d, ref.capped, ref.m, ref.k_last)
        assert res.levels == ref.levels and res.gamma_hash == ref.gamma_hash
        U, want = n - k + 1, []
        for c, j, w, u_after in ref.rounds:
            want.append([c, j, w if exact else min(w, U), u_after])
            U = u_after
        assert res.rounds == want
        if not res.capped:
            assert res.witness_ok


def test_histogram_and_witness_rd_plan(mdg, device):
    """Revolving-door plans (prefixes in revolving-door order) give the same histograms and
    valid witnesses on full and partial Gammas."""
    for (n, k, seed) in [(70, 20, 5), (300, 200, 11), (256, 100, 3)]:
        G = mdg.gen_matrix(n, k, seed, True)
        gs = mdg.GammaSet.build(G, n, 3, seed)
        device.load_gset(gs)
        for j in range(gs.m):
            g = gs.gamma(j)
            for c in (2, 3):
                device.set_kernel(mdg.KERNEL_TAB)
                a, ha = device.round_hist(j, c, n)
                device.set_kernel(mdg.KERNEL_RD)
                b, hb = device.round_hist(j, c, n)
                assert ha.tolist() == hb.tolist() and a.min_weight == b.min_weight, (n, k, j, c)
                o = device.round(j, c)
                idx = device.round_witness(j, c, o)
                assert len(set(idx)) == c and popcount_rows(g, idx)[0] == o.min_weight
        device.set_kernel(mdg.KERNEL_TAB)


@pytest.mark.parametrize("kernel", KERNELS)
def test_random_sparse_codes_vs_oracle(mdg, device, kernel):
    """Random codes of random shapes and densities (sparse rows exercise the partial-word
    fold options, partial Gammas, transposed tiles and fused levels) in both round modes:
    d, trace and witness against the C oracle."""
    rng = np.random.default_rng(1234 + kernel)
    checked = 0
    while checked < 120:
        k = int(rng.integers(4, 23))
        n = int(rng.integers(k + 1, 3 * k + 12))
        dens = float(rng.choice([0.08, 0.15, 0.3, 0.5]))
        try:
            rows = _sparse_code(rng, k, n, dens)
        except Exception:
            continue
        seed = int(rng.integers(0, 1000))
        ref = port.min_weight(rows, n, 10, seed)
        for exact in (True, False):
            res = mdg.min_weight(rows, n, 10, seed, kernel=kernel, device=device, exact_rounds=exact)
            assert (res.d, res.m, res.k_last, res.levels) == (ref.d, ref.m, ref.k_last, ref.levels), (n, k, dens, seed)
            U, want = n - k + 1, []
            for c, j, w, u_after in ref.rounds:
                want.append([c, j, w if exact else min(w, U), u_after])
                U = u_after
            assert res.rounds == want, (n, k, dens, seed, exact)
            assert res.witness_ok
        checked += 1


def test_min_weight_batch_many_mixed(mdg, device):
    """Many codes of mixed shapes through the batch front door with 8 streams: each result
    equals the single-code front door's (trace, d, Gamma set)."""
    mats, ns, seeds = [], [], []
    for case in load_golden("seeded")[:48]:
        rows, n = mdg.parse_matrix(case["matrix"])
        mats.append(rows)
        ns.append(n)
        seeds.append(case["seed"])
    for (n, k, s) in [(128, 64, 3), (256, 32, 7), (80, 40, 1), (300, 200, 11)]:
        mats.append(mdg.gen_matrix(n, k, s, True))
        ns.append(n)
        seeds.append(s)
    caps = [0] * (len(mats) - 1) + [4]
    runs = mdg.min_weight_batch(mats[:-1], ns[:-1], trials=10, seed=seeds[:-1], device=device, streams=8)
    runs.append(mdg.min_weight_batch([mats[-1]], ns[-1], trials=10, seed=seeds[-1], level_cap=4,
                                     device=device)[0])
    for i, r in enumerate(runs):
        one = mdg.min_weight(mats[i], ns[i], 10, seeds[i], level_cap=caps[i], device=device)
        assert (r.d, r.rounds, r.levels, r.gamma_hash, r.capped) == \
               (one.d, one.rounds, one.levels, one.gamma_hash, one.capped), i
        assert r.witness_ok or r.capped


@pytest.mark.parametrize("code", [1, 1 | 64, 1 | 16 | 64, 1 | 32 | 64, 2 | 16, 4, 1 | 128])
def test_forced_fold_options_vs_oracle(mdg, device, code):
    """Every stage-1 variant, forced on every tile bound T (MDG_FORCE_FOLD; the plan normally
    picks them per T only for large rounds): the pair pre-filter (| 64) over one two-word
    fold group -- all of NW = 2, the first two words of NW = 3 (drop, | 16) and NW = 4 (half,
    | 32) -- and its fall-through to single folds and exact weights, on raw and systematic
    matrices of 1..8 words, bounded at cutoffs around the true minimum."""
    import os
    rng = np.random.default_rng(99 + code)
    os.environ["MDG_FORCE_FOLD"] = str(code)
    try:
        for n in (40, 64, 80, 96, 128, 150, 200, 256):
            k = int(rng.integers(10, 20))
            W = (n + 63) // 64
            rows = rng.integers(0, 2**63, size=(k, W), dtype=np.uint64)
            if n % 64:
                rows[:, -1] &= np.uint64((1 << (n % 64)) - 1)
            if rng.random() < 0.5:  # sparse rows: the bound admits more candidates
                rows &= rng.integers(0, 2**63, size=(k, W), dtype=np.uint64)
            device.load_gammas(rows, n, ranks=None)
            for c in (2, 3, 4, 5):
                w, _ = port.round_min(rows, n, c)
                assert device.round(0, c).min_weight == w, (n, k, c, code)
                for cutoff in (w, w + 1, w + 3, w + 12, n + 1):
                    out = device.round_bounded(0, c, cutoff)
                    assert out.min_weight == min(w, cutoff), (n, k, c, cutoff, code)
                    assert out.bounded == (w >= cutoff), (n, k, c, cutoff, code)
                    if not out.bounded:
                        idx = device.round_witness(0, c, out)
                        assert popcount_rows(rows, idx)[0] == w
        for name in ("cfg1", "cfg2_s1", "cfg2_s8"):
            case = next(c for c in load_golden("configs") if c["name"] == name)
            g = case["gen"]
            G = mdg.gen_matrix(g["n"], g["k"], g["seed"], True)
            res = mdg.min_weight(G, g["n"], case["trials"], case["seed"], device=device, exact_rounds=True)
            _check_run(res, case, name, True)
    finally:
        del os.environ["MDG_FORCE_FOLD"]


def test_position_keys_name_the_tab_find_witness(mdg, device):
    """Round keys carry the winner's position (kPosFlag); the witness decoded from them equals
    the one tab_find re-searches (the lowest position of the round minimum in the lowest
    tile), on raw and systematic matrices, exact and bounded rounds. The library reads
    MDG_NO_POS_KEY once, so the tab_find side runs in a subprocess."""
    import json
    import os
    import subprocess
    import sys
    script = r'''
import json, sys
import numpy as np
sys.path.insert(0, %r)
import paper_1911_08963_b200 as mdg
rng = np.random.default_rng(5)
dev = mdg.Device(0)
out = []
for n in (40, 64, 100, 128, 200, 256):
    k = int(rng.integers(12, 24))
    W = (n + 63) // 64
    rows = rng.integers(0, 2**63, size=(k, W), dtype=np.uint64)
    if n %% 64:
        rows[:, -1] &= np.uint64((1 << (n %% 64)) - 1)
    dev.load_gammas(rows, n, ranks=None)
    for c in (2, 3, 4, 5):
        for cut in (0, 3, 1000):
            o = dev.round_bounded(0, c, cut) if cut else dev.round(0, c)
            if o.bounded:
                continue
            out.append([n, c, cut, o.min_weight, sorted(dev.round_witness(0, c, o)), o.argmin_key >> 51 & 1])
print(json.dumps(out))
''' % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    runs = {}
    for mode in ("pos", "find"):
        env = dict(os.environ)
        if mode == "find":
            env["MDG_NO_POS_KEY"] = "1"
        r = subprocess.run([sys.executable, "-c", script], env=env, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        runs[mode] = json.loads(r.stdout.strip().splitlines()[-1])
    assert len(runs["pos"]) == len(runs["find"]) > 40
    assert all(x[5] == 1 for x in runs["pos"]) and all(x[5] == 0 for x in runs["find"])
    for a, b in zip(runs["pos"], runs["find"]):
        assert a[:5] == b[:5], (a, b)


def test_reference_loop_drives_gpu_round(tmp_path):
    """INTEGRATION.md §1 built literally (tests/integration/bz_gpu.cpp -> oracle/_ref/bz_gpu):
    the UNMODIFIED reference's min_weight steps and run_bz_loop (engines.cpp:447-476, linked
    from oracle/_ref) with the GPU RoundRunner calling mdg_round. Every exact round minimum,
    U, d and g_final equal the reference's own goldens."""
    import json
    import os
    import subprocess
    from conftest import ROOT
    exe = os.path.join(ROOT, "oracle", "_ref", "bz_gpu")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/bz_gpu not built (needs /root/reference at build time)")
    import paper_1911_08963_b200 as mdg
    cases = [c for c in load_golden("configs") if c["name"] in ("cfg1", "cfg2_s1", "cfg2_s8", "cfg3", "cfg4")]
    kats = {c["name"]: c for c in load_golden("kats")}
    for case in cases + [kats["hamming_7_4"], kats["golay_23_12"], kats["ext_golay_24_12"]]:
        if "gen" in case:
            g = case["gen"]
            text = mdg.serialize_matrix(mdg.gen_matrix(g["n"], g["k"], g["seed"], True), g["n"])
        else:
            text = case["matrix"]
        f = tmp_path / f"{case['name']}.txt"
        f.write_text(text)
        cmd = [exe, str(f), "--seed", str(case["seed"]), "--trials", str(case["trials"])]
        if case.get("capped"):
            cmd += ["--cap", str(case["level_cap"])]
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, (case["name"], r.stderr)
        rec = json.loads(r.stdout)
        assert rec["rounds"] == case["rounds"], case["name"]
        assert (rec["m"], rec["k_last"], rec["g_final"]) == (case["m"], case["k_last"], case["g_final"])
        assert rec["d"] == (case["U_final"] if case.get("capped") else case["d"]), case["name"]


def test_cli_devices_split(mdg, tmp_path):
    """`mindist mindist FILE --devices 0,0 --split-min 1`: one process, two contexts (here on
    the same GPU), every round split across them through the exchange group; the record has
    the golden d / trace / levels and "devices": 2."""
    import json
    import os
    import subprocess
    from conftest import ROOT
    exe = os.path.join(ROOT, "paper_1911_08963_b200", "bin", "mindist")
    case = next(c for c in load_golden("configs") if c["name"] == "cfg2_s8")
    g = case["gen"]
    f = tmp_path / "cfg2_s8.txt"
    f.write_text(mdg.serialize_matrix(mdg.gen_matrix(g["n"], g["k"], g["seed"], True), g["n"]))
    r = subprocess.run([exe, "mindist", str(f), "--seed", str(g["seed"]), "--devices", "0,0",
                        "--split-min", "1"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    rec = json.loads(r.stdout)
    assert rec["d"] == case["d"] and rec["devices"] == 2 and rec["witness_ok"]
    assert rec["levels"] == case["levels"]
    r = subprocess.run([exe, "mindist", str(f), str(f), "--devices", "0,0", "--seed", "1"],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 2 and "--devices" in r.stderr


def test_group_abi_driven_by_caller(mdg):
    """The exchange group through its own C ABI (mdg_group_create / mdg_group_attach /
    mdg_group_reduce_min): the caller drives each member from its own thread with
    mdg_min_weight_dist(..., reduce_min = mdg_group_reduce_min); every member's record equals
    the golden, and detaching restores single-context runs."""
    import ctypes as C
    import threading
    case = next(c for c in load_golden("configs") if c["name"] == "cfg2_s1")
    g = case["gen"]
    G = mdg.gen_matrix(g["n"], g["k"], g["seed"], True)
    world = 2
    devs = [mdg.Device(0) for _ in range(world)]
    grp = C.c_void_p()
    L = mdg.lib()
    assert L.mdg_group_create(world, C.byref(grp)) == 0
    try:
        for r, d in enumerate(devs):
            assert L.mdg_group_attach(d.handle, grp, r) == 0
        out = [None] * world
        errs = []

        def member(r):
            try:
                out[r] = mdg.min_weight_dist(G, g["n"], r, world, "group", trials=10, seed=g["seed"],
                                             device=devs[r], split_min=1)
            except Exception as e:  # surfaced below
                errs.append(e)

        ts = [threading.Thread(target=member, args=(r,)) for r in range(world)]
        for t in ts:
            t.start()
        for t in ts:
            t.join(timeout=300)
        assert not errs, errs
        for r in range(world):
            _check_run(out[r], case, f"group rank {r}", exact=False)
        for d in devs:
            assert L.mdg_group_attach(d.handle, None, 0) == 0
        solo = mdg.min_weight(G, g["n"], 10, g["seed"], device=devs[0])
        _check_run(solo, case, "after detach", exact=False)
    finally:
        L.mdg_group_free(grp)
        for d in devs:
            d.close()


def test_group_divergence_fails_fast(mdg):
    """Members whose level loops diverge (here: different split_min, so they enqueue different
    split rounds) fail with an error instead of hanging: a (c, j) mismatch at a barrier, or a
    member leaving the loop while another waits at a split round."""
    import ctypes as C
    import threading
    import time
    G = mdg.gen_matrix(128, 64, 1, True)
    L = mdg.lib()
    for mins in ((1, 10**6), (1, 1 << 62)):
        devs = [mdg.Device(0) for _ in range(2)]
        grp = C.c_void_p()
        assert L.mdg_group_create(2, C.byref(grp)) == 0
        results = [None, None]
        try:
            for r, d in enumerate(devs):
                assert L.mdg_group_attach(d.handle, grp, r) == 0

            def member(r):
                try:
                    results[r] = mdg.min_weight_dist(G, 128, r, 2, "group", trials=10, seed=1,
                                                     device=devs[r], split_min=mins[r])
                except Exception as e:
                    results[r] = e

            t0 = time.time()
            ts = [threading.Thread(target=member, args=(r,)) for r in range(2)]
            for t in ts:
                t.start()
            for t in ts:
                t.join(timeout=120)
            assert not any(t.is_alive() for t in ts), "diverged members hung"
            assert time.time() - t0 < 60
            assert isinstance(results[0], mdg.MdgError) and "diverged" in str(results[0]), results
        finally:
            L.mdg_group_free(grp)
            for d in devs:
                d.close()


@pytest.mark.parametrize("kernel", KERNELS)
def test_unit_column_elision_vs_oracle(mdg, device, kernel, monkeypatch):
    """A partial Gamma whose rows [rank, k) each still own a weight-1 column (the previous
    block's identity, untouched by the last block's row operations) is compacted like a
    full-rank one (|S| + popcount of the non-unit columns). Per-round minima, evaluated counts
    and witnesses equal the oracle's on the uncompacted Gammas, with the elision on and off
    (MDG_NO_UNIT_ELISION), on config 4 and on partial blocks of other shapes, including
    sparse codes whose last rows may own no unit column (the identity-only fallback)."""
    device.set_kernel(kernel)
    rng = np.random.default_rng(99)
    codes = [(mdg.gen_matrix(n, k, s, True), n) for (n, k, s) in
             [(300, 200, 11), (70, 40, 2), (45, 40, 6), (130, 64, 11), (301, 150, 6), (33, 20, 3)]]
    while len(codes) < 14:
        k = int(rng.integers(6, 20))
        n = int(rng.integers(k + 2, 2 * k))
        codes.append((_sparse_code(rng, k, n, float(rng.choice([0.2, 0.5]))), n))
    partial = 0
    for G, n in codes:
        gs = mdg.GammaSet.build(G, n, 3, 1)
        partial += gs.ranks[-1] < gs.gamma(0).shape[0]
        for off in (False, True):
            if off:
                monkeypatch.setenv("MDG_NO_UNIT_ELISION", "1")
            else:
                monkeypatch.delenv("MDG_NO_UNIT_ELISION", raising=False)
            device.load_gset(gs)
            j = gs.m - 1
            g = gs.gamma(j)
            for c in range(1, 4 if n > 100 else 5):
                w, combos = port.round_min(g, n, c)
                out = device.round(j, c)
                assert (out.min_weight, out.evaluated) == (w, combos), (n, off, c, kernel)
                idx = device.round_witness(j, c, out)
                assert popcount_rows(g, idx)[0] == w
    monkeypatch.delenv("MDG_NO_UNIT_ELISION", raising=False)
    assert partial >= 6


_RING_WORKER = r"""
import os, sys
import numpy as np
sys.path.insert(0, %(root)r)
import paper_1911_08963_b200 as mdg
from oracle import port
rng = np.random.default_rng(%(seed)d)
dev = mdg.Device(0)
checked = bad = 0
while checked < %(count)d:
    k = int(rng.integers(3, %(kmax)d)); n = int(rng.integers(k + 1, 4 * k + 20))
    dens = float(rng.choice([0.1, 0.25, 0.5]))
    dense = (rng.random((k, n)) < dens).astype(np.uint64)
    rows = np.zeros((k, (n + 63) // 64), dtype=np.uint64)
    for c in range(n):
        rows[:, c // 64] |= dense[:, c] << np.uint64(c %% 64)
    if port.rank(rows, n) != k:
        continue
    s = int(rng.integers(0, 1000))
    ref = port.min_weight(rows, n, 10, s)
    for kernel in (0, 1):
        for exact in (True, False):
            try:
                r = mdg.min_weight(rows, n, 10, s, kernel=kernel, device=dev, exact_rounds=exact)
            except Exception:
                bad += 1
                continue
            U, want = n - k + 1, []
            for c, j, w, u in ref.rounds:
                want.append([c, j, w if exact else min(w, U), u])
                U = u
            if not (r.d == ref.d and r.levels == ref.levels and r.rounds == want and r.witness_ok):
                bad += 1
    checked += 1
dev.close()
print("RESULT", checked, bad, flush=True)
"""


@pytest.mark.parametrize("slots,seed,kmax", [(40, 55, 15), (97, 125, 28), (61, 89, 28)])
def test_slot_ring_wraps_keep_rounds_clean(slots, seed, kmax):
    """Hundreds of BZ runs on ONE context with the ring of per-round scratch slots shrunk
    (MDG_SLOTS) so it wraps every few levels: a fused level whose slots straddled the wrap once
    left its first slots dirty for the ring's next cycle, and a stale lighter key then won a
    later round's atomicMin (a wrong d after ~2,400 runs on one context with the full ring; found
    by tools/forced_sweep.py). These three (ring size, seed, k range) sequences each hit the
    hazard in a build without the fix (-DMDG_NO_SLOT_RESERVE: 2, 3 and 3 wrong runs of 1,200;
    profiles/r02f_forced_sweep.txt). d, both traces and the witness against the oracle."""
    import os
    import subprocess
    import sys
    from conftest import ROOT as ROOT_DIR
    env = dict(os.environ, MDG_SLOTS=str(slots))
    script = _RING_WORKER % {"root": ROOT_DIR, "seed": seed, "count": 300, "kmax": kmax}
    p = subprocess.run([sys.executable, "-c", script], env=env, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-2000:]
    line = next(ln for ln in p.stdout.splitlines() if ln.startswith("RESULT"))
    _, checked, bad = line.split()
    assert int(bad) == 0 and int(checked) == 300, line


@pytest.mark.parametrize("slots,seed,ahead", [(0, 21, 0), (40, 22, 0), (0, 23, 1)])
def test_soak_mixed_calls_on_one_context(slots, seed, ahead):
    """tools/soak.py: a random mix of every public call (front door, batch, resident loops,
    single / bounded / split rounds, witnesses, histograms whole and split, brute force,
    rank-deficient inputs, one code split across several contexts) on ONE long-lived context,
    each result against the C oracle; once with the scratch ring shrunk so it wraps every few
    launches, once with at most one level in flight beyond the last closed one."""
    import os
    import subprocess
    import sys
    from conftest import ROOT as ROOT_DIR
    env = dict(os.environ)
    if slots:
        env["MDG_SLOTS"] = str(slots)
    if ahead:  # the chained loop's levels-in-flight throttle (off by default)
        env["MDG_LEVELS_AHEAD"] = str(ahead)
    p = subprocess.run([sys.executable, os.path.join(ROOT_DIR, "tools", "soak.py"), "400", str(seed)],
                       env=env, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, (p.stdout[-1500:], p.stderr[-1500:])
    assert "400 operations, 0 failures" in p.stdout


_XB_WORKER = r"""
import json, os, sys
sys.path.insert(0, %(root)r)
sys.path.insert(0, os.path.join(%(root)r, "tests"))
import numpy as np
import torch.distributed as dist
import paper_1911_08963_b200 as mdg
from conftest import load_golden
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo", rank=rank, world_size=world)
dev = mdg.Device(0)
err = [None]
try:
    h = [dev.shared_bound_create() if rank == 0 else None]
except Exception as e:  # CUDA IPC not available in this environment
    h, err = [None], [str(e)]
dist.broadcast_object_list(h, src=0)
if rank != 0 and h[0] is not None:
    try:
        dev.shared_bound_open(h[0])
    except Exception as e:
        err = [str(e)]
errs = [None] * world
dist.all_gather_object(errs, err[0])
if any(errs):
    print("SKIP " + "; ".join(e for e in errs if e), flush=True)
    dist.destroy_process_group()
    sys.exit(0)
dist.barrier()

def red(keys):  # element-wise u64 min over the ranks (the callback loop: one exchange per split round)
    out = [None] * world
    dist.all_gather_object(out, keys.copy())
    return np.minimum.reduce(out)

cases = {c["name"]: c for c in load_golden("configs")}
out = []
for name in ("cfg1", "cfg2_s8", "cfg2_s1"):
    case = cases[name]
    g = case["gen"]
    G = mdg.gen_matrix(g["n"], g["k"], g["seed"], True)
    for split_min in (1, 10**6):
        r = mdg.min_weight_dist(G, g["n"], rank, world, red, trials=10, seed=g["seed"], device=dev,
                                split_min=split_min)
        out.append({"name": name, "split_min": split_min, "d": r.d, "rounds": r.rounds, "levels": r.levels,
                    "gamma_hash": r.gamma_hash, "witness_ok": r.witness_ok, "evaluated": r.evaluated})
# a [224,112] code whose level-8 round ends by early exit: rows 0..7 are planted to sum to a
# weight-16 codeword, and 16 is the lower bound after level 7 (2 full information sets:
# L(7) = 16; random codewords of such a code weigh > 20), so the round (5.5e11 codewords: ~70 ms
# per rank if run out, far above any start skew between the processes) stops as soon as that
# codeword is seen -- by the rank that owns its tile, and, through the shared word, by the other
from oracle import port
u64 = np.uint64
M1 = u64(0xFFFF000000000000)  # word 1: identity columns 64..111 low, A columns 112..127 high
for sd in range(1, 300):  # a seed whose planted A is invertible: the identity order is then kept
    G = mdg.gen_matrix(224, 112, sd, True).copy()  # (maximal (m, k_last)), information sets = the halves,
    a1, a2, a3 = u64(0), u64(0), u64(0)            # and the planted codeword has 8 ones in each
    for r in range(1, 8):
        a1 ^= G[r, 1] & M1
        a2 ^= G[r, 2]
        a3 ^= G[r, 3]
    G[0, 1] = (G[0, 1] & ~M1) | a1
    G[0, 2] = a2 ^ u64(0xFF)
    G[0, 3] = a3
    A = np.zeros((112, 2), dtype=np.uint64)
    A[:, 0] = (G[:, 1] >> u64(48)) | ((G[:, 2] & u64((1 << 48) - 1)) << u64(16))
    A[:, 1] = (G[:, 2] >> u64(48)) | (G[:, 3] << u64(16))
    if port.rank(A, 112) == 112:
        break
ref = port.min_weight(G, 224, 10, 5, level_cap=5)  # the oracle (no early exit) for levels <= 5
solo = mdg.min_weight(G, 224, 10, 5, device=mdg.Device(0))  # one rank, nothing split or shared
r = mdg.min_weight_dist(G, 224, rank, world, red, trials=10, seed=5, device=dev, split_min=1)
U, want = 224 - 112 + 1, []
for c, j, w, u in ref.rounds:
    want.append([c, j, min(w, U), u])
    U = u
ok = (solo.rounds[:len(want)] == want and solo.levels[:5] == ref.levels and solo.d == 16 and
      solo.rounds[-1] == [8, 0, 16, 16] and
      r.d == 16 and r.witness_ok and r.rounds == solo.rounds and r.levels == solo.levels)
out.append({"name": "planted", "d": r.d, "ok": bool(ok), "evaluated": r.evaluated, "tail": r.rounds[-2:],
            "solo_tail": solo.rounds[-2:], "solo_d": solo.d})
dist.barrier()
dev.shared_bound_close()
dev.close()
print("RESULT " + json.dumps(out), flush=True)
dist.destroy_process_group()
"""


def test_shared_bound_across_processes():
    """SURVEY.md 8e (i) across processes: two processes on this GPU share the round-key ring
    through a CUDA IPC handle (mdg_shared_bound_create / _open); every split round publishes its
    tile results there and polls it. d, traces, Gamma set and witness equal the goldens on both
    ranks, with the shared bound on and off (MDG_NO_SHARED_BOUND); on a code whose level-8 round
    ends by early exit the ranks together evaluate far fewer codewords with it (one rank's find
    stops the other)."""
    import json
    import os
    import socket
    import subprocess
    import sys
    from conftest import ROOT as ROOT_DIR
    cases = {c["name"]: c for c in load_golden("configs")}
    totals = {}
    for off in (False, True):
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port_no = sk.getsockname()[1]
        procs = []
        for r in range(2):
            env = dict(os.environ, RANK=str(r), WORLD_SIZE="2", MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
            if off:
                env["MDG_NO_SHARED_BOUND"] = "1"
            procs.append(subprocess.Popen([sys.executable, "-c", _XB_WORKER % {"root": ROOT_DIR}], env=env,
                                          stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True))
        outs = []
        for p in procs:
            o, e = p.communicate(timeout=600)
            assert p.returncode == 0, e[-2000:]
            skip = [ln for ln in o.splitlines() if ln.startswith("SKIP ")]
            if skip:
                pytest.skip("CUDA IPC unavailable here: " + skip[0][5:200])
            outs.append(json.loads(next(ln for ln in o.splitlines() if ln.startswith("RESULT "))[7:]))
        for rank_out in outs:
            for rec in rank_out:
                if rec["name"] == "planted":
                    assert rec["ok"], rec
                    continue
                case = cases[rec["name"]]
                U, want = case["n"] - case["k"] + 1, []
                for c, j, w, ua in case["rounds"]:
                    want.append([c, j, min(w, U), ua])
                    U = ua
                assert rec["d"] == case["d"] and rec["rounds"] == want and rec["levels"] == case["levels"], rec["name"]
                assert rec["gamma_hash"] == case["gamma_hash"] and rec["witness_ok"], rec["name"]
        totals[off] = sum(rec["evaluated"] for rank_out in outs for rec in rank_out if rec["name"] == "planted")
    print(f"planted code, codewords evaluated by both ranks: shared bound {totals[False]}, off {totals[True]}")
    # without the shared word the rank that does not own the planted codeword's tile runs its
    # whole half of the level-8 round (2.7e11 codewords); with it, it stops after its first tiles
    assert totals[False] < 0.8 * totals[True], totals
