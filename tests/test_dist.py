"""Multi-rank host logic on CPU (gloo, world size 2): every rank runs the native
level loop (run_bz_loop through the RoundRunner seam); each round's rank space
is split contiguously across ranks and the per-round minimum is combined with an
allreduce(min) — the structure mdg_min_weight_dist uses with NCCL on GPUs. The
trace must equal the single-process reference trace."""
import os
import socket
from math import comb

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT, load_golden


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _weight(rows, idx):
    acc = np.zeros(rows.shape[1], dtype=np.uint64)
    for r in idx:
        acc ^= rows[r]
    return int(sum(bin(int(x)).count("1") for x in acc))


def _worker(rank, world, port, names, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import paper_1911_08963_b200 as mdg
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cases = {c["name"]: c for c in load_golden("seeded")}
    out = {}
    try:
        for name in names:
            case = cases[name]
            rows, n = mdg.parse_matrix(case["matrix"])
            gs = mdg.GammaSet.build(rows, n, case["trials"], case["seed"])
            gam = [gs.gamma(j) for j in range(gs.m)]

            def round_fn(j, c, stop_at):
                N = comb(gs.k, c)
                lo, hi = N * rank // world, N * (rank + 1) // world
                best = 1 << 30
                for r in range(lo, hi):  # this rank's contiguous revolving-door range
                    best = min(best, _weight(gam[j], mdg.rd_unrank(c, r)))
                t = torch.tensor([best], dtype=torch.int64)
                dist.all_reduce(t, op=dist.ReduceOp.MIN)
                return int(t.item())

            res = mdg.run_bz_loop(gs, round_fn)
            out[name] = (res.d, res.rounds, res.levels)
        q.put((rank, out, None))
    except Exception as e:  # pragma: no cover
        q.put((rank, None, repr(e)))
    finally:
        dist.destroy_process_group()


def test_two_rank_split_reproduces_reference_trace():
    names = [f"seeded_{i}" for i in (0, 3, 7, 11, 19, 42)]
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, names, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    cases = {c["name"]: c for c in load_golden("seeded")}
    for rank, out, err in results:
        assert err is None, err
        for name in names:
            d, rounds, levels = out[name]
            assert d == cases[name]["d"], (rank, name)
            assert rounds == cases[name]["rounds"], (rank, name)
            assert levels == cases[name]["levels"], (rank, name)


def _hist_worker(rank, world, port, levels, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import paper_1911_08963_b200 as mdg
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        M = mdg.gen_matrix(256, 100, 3, identity=False)
        out = {}
        for c in levels:
            N = comb(100, c)
            lo, hi = N * rank // world, N * (rank + 1) // world
            hist = np.zeros(257, dtype=np.int64)
            for r in range(lo, hi):  # this rank's contiguous revolving-door range
                hist[_weight(M, mdg.rd_unrank(c, r))] += 1
            t = torch.from_numpy(hist)
            dist.all_reduce(t, op=dist.ReduceOp.SUM)  # allreduce(sum) over n + 1 counts
            out[c] = (t.tolist(), hi - lo)
        q.put((rank, out, None))
    except Exception as e:  # pragma: no cover
        q.put((rank, None, repr(e)))
    finally:
        dist.destroy_process_group()


def test_two_rank_histogram_sums_to_reference():
    """Config 5 at N > 1 (host logic of mdg_round_hist_dist): each rank counts the weights of a
    contiguous share of the C(100, c) combinations, the n + 1 counts are summed with an
    allreduce; every rank must hold the reference's histogram."""
    levels = (1, 2, 3)
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_hist_worker, args=(r, world, port, levels, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    gold = {lv["c"]: lv for lv in load_golden("cfg5_hist")["levels"]}
    for rank, out, err in results:
        assert err is None, err
        for c in levels:
            hist, share = out[c]
            assert hist == gold[c]["hist"], (rank, c)
    assert sum(out[3][1] for _, out, _ in results) == comb(100, 3)
