"""Benchmark of the B200 Brouwer–Zimmermann engine (driver contract).

Workload (BASELINE.json configs[1]): config 2, random binary rate-1/2 [128,64]
codes, G = (I_64 | A), A from mt19937_64 seeds 1..8; one
step = the full Brouwer–Zimmermann run to termination (exact d) of all eight
codes. Metric: codewords evaluated per second (BASELINE.json `metric`).

* value  — N = 1: device-resident: the level loops over Gamma sets already in
           HBM (mdg_bz_loop_device_batch: one context per code, --streams codes
           in flight from the library's worker threads), CUDA events around each
           whole step (host gaps included);
           codewords / time. N > 1 (torchrun): the strong leg below is the
           headline ("scaling": "strong"); the eight-code step, run by every rank
           on its own GPU (independent codes, no collective), moves to
           `weak_step`.
* strong — at every N: ONE code (config 4 to level cap 7, 4.7e12 codewords)
           with every round of >= 2e8 codewords split across the ranks and its
           key min-reduced by an in-stream NCCL allreduce(min)
           (mdg_min_weight_dist); N = 1 is its baseline. Parity
           flags against the reference's cap-6 and cap-7 traces.
* configs — N = 1: time-to-d of configs 1, 3, 4 (caps 5, 6), the config-5
           histograms and the histogram of level 6 of the same matrix (1.19e9
           codewords: the kernel's steady state), each with a parity flag against
           the reference goldens.
* e2e    — the public front door from host matrices (mdg_min_weight_batch over
           the rank's codes): row basis +
           Gamma search on the host, H2D of the Gammas, the device loop, D2H of
           every round result and the witness; CUDA-event timed the same way.
* roofline — the dominant kernel (tab_round on the c = 7 rounds, measured in a
           separate pass with one loop at a time): achieved
           codewords/s vs the integer issue-rate roofline of its op mix: ALU pipe
           (LOP3, 64/clk/SM) and XU pipe (POPC, 16/clk/SM) rates measured on B200
           (profiles/r02_pipes_microbench.jsonl) over the ops per codeword ncu counts.
* cpu_baseline — the reference's own engine (oracle/_ref, unmodified sources)
           on this host's cores, one code of the same workload.

`--impl reference` runs the reference CPU implementation (oracle/_ref) on the
same workload: each step is one seed of config 2 to termination, all host
threads (round_saved_parallel, the reference's multi-core path).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N, K, SEEDS = 128, 64, list(range(1, 9))
POPC_PER_S_MEASURED = 4642.3e9   # profiles/r02_pipes_microbench.jsonl (B200, 148 SMs): XU pipe
ALU_PER_S_MEASURED = 18146.5e9   # same file: LOP3 on the ALU pipe (64/clk/SM)
# Pipe operations the bound-pruned level-7 round kernel executes per codeword, from the committed
# ncu capture of that launch (profiles/r02h_tab_round_c7_ncu.txt: tab_round<2,false> on the
# config-2 seed-1 level-7 round at the loop's U = 16): ALU-pipe ops (3 LOP3 per pair bound,
# vote min / compare, loop) and XU ops (POPC). The ALU pipe binds (83 % busy, XU 80 %).
ALU_PER_CW_PRUNED = 2.321
XU_PER_CW_PRUNED = 0.561
DRAM_BYTES_PER_LAUNCH = 4246272  # same capture: dram__bytes_read.sum + dram__bytes_write.sum
WORKLOAD = "cfg2: random [128,64] codes G=(I|A), mt19937_64 seeds 1..8, BZ to termination (exact d)"


def hbm_check(achieved_cw_s):
    """The HBM roofline for the same launch, against MEASURED_PEAKS.json (driver-written): the
    launch's DRAM bytes per second over the measured copy bandwidth."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            hbm = float(json.load(f)["hbm_gbs"])
    except Exception:
        return None
    launch_s = 621216192 / achieved_cw_s if achieved_cw_s else 0.0
    gbs = DRAM_BYTES_PER_LAUNCH / launch_s / 1e9 if launch_s else 0.0
    return {"dram_gbs": gbs, "hbm_peak_gbs": hbm, "frac": gbs / hbm, "source": "MEASURED_PEAKS.json hbm_gbs"}


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.samples = []
        self._proc = None
        self._thr = None

    def start(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self._proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self._proc = None
            return
        self._thr = threading.Thread(target=self._read, daemon=True)
        self._thr.start()

    def _read(self):
        for line in self._proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.samples.append(parts)

    def stop(self):
        if self._proc:
            self._proc.terminate()
            try:
                self._proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self._proc.kill()
        if self._thr:
            self._thr.join(timeout=2)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[3 + i] == "Active"})
        loaded = [x for x in sm if x > 0.5 * (max(mx) if mx else 1)] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def cpu_baseline_reference(seed=1, workers=None):
    """The reference's engine (unmodified sources, oracle/_ref) on this host: one config-2
    code to termination with round_saved_parallel over all host threads."""
    from oracle import ref
    workers = workers or os.cpu_count() or 1
    text = ref.gen(N, K, seed)
    t0 = time.perf_counter()
    tr = ref.trace(text, trials=10, seed=seed, engine="saved", s=5, workers=workers)
    dt = time.perf_counter() - t0
    return tr, dt, workers


def cpu_baseline_port(seed=1, level_cap=6):
    """Fallback when oracle/_ref is absent: the C restatement, single thread, capped."""
    from oracle import port
    G = port.gen_matrix(N, K, seed, True)
    t0 = time.perf_counter()
    tr = port.min_weight(G, N, 10, seed, level_cap=level_cap)
    return tr, time.perf_counter() - t0


def run_reference_arm(args, rank, world):
    if rank != 0:
        return 0
    from oracle import ref
    workers = os.cpu_count() or 1
    kind = "reference" if ref.available() else "port"
    vals, steps_ms = [], []
    total_cw = 0
    t_all = 0.0
    for i in range(args.warmup + args.steps):
        seed = SEEDS[i % len(SEEDS)]
        if kind == "reference":
            tr, dt, _ = cpu_baseline_reference(seed, workers)
            cw = tr["combinations"]
        else:
            tr, dt = cpu_baseline_port(seed)
            cw = tr.combinations
            workers = 1
        if i >= args.warmup:
            total_cw += cw
            t_all += dt
            steps_ms.append(dt * 1e3)
    value = total_cw / t_all
    sample = ("one config-2 code per step (seeds rotate 1..8), full BZ run to termination, "
              "reference round_saved_parallel (s=5) on all host threads, -O3 -march=x86-64-v3"
              if kind == "reference" else "C restatement, one code per step, levels c<=6, 1 thread")
    line = {
        "impl": "reference", "metric": "codewords_evaluated_per_sec", "value": value, "unit": "cw/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": statistics.mean(steps_ms), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic (mt19937_64, SURVEY.md §8d)",
        "config": {"workload": WORKLOAD, "per_step": "one code (seed rotates)"},
        "cpu_baseline": {"value": value, "unit": "cw/s", "cores": workers, "kind": kind,
                         "sample": sample},
        "e2e": {"value": value, "unit": "cw/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


CFG4 = (300, 200, 11)


def _gold(name, file="configs"):
    with open(os.path.join(ROOT, "tests", "golden", file + ".json")) as f:
        return next(c for c in json.load(f)["data"] if c["name"] == name)


def _trace_matches(res, case):
    """bounded-round trace (w = min(exact w, U before the round)) and levels vs a golden"""
    U = case["n"] - case["k"] + 1
    exp = []
    for c, j, w, Ua in case["rounds"]:
        exp.append([c, j, min(w, U), Ua])
        U = Ua
    n = min(len(res.rounds), len(exp))
    return (n == len(exp) and res.rounds[:n] == exp and
            res.levels[:len(case["levels"])] == case["levels"] and
            res.gamma_hash == case["gamma_hash"] and res.witness_ok)


def strong_leg(mdg, torch, dist, rank, world, local, kernel, barrier, warm=1, steps=3):
    """One code's rounds split across the ranks (config 4 to cap 7): see main()."""
    n, k, seed = CFG4
    G = mdg.gen_matrix(n, k, seed, True)
    dev = mdg.Device(local)
    if world > 1:
        u = [mdg.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(u, src=0)
        dev.nccl_init(u[0], rank, world)
    gold6 = _gold("cfg4", "configs_cap4_6")
    try:
        gold7 = _gold("cfg4", "configs_cap4_7")
    except (OSError, StopIteration):
        gold7 = None
    ms, r = [], None
    for step in range(warm + steps):
        barrier()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        if world > 1:
            r = mdg.min_weight_dist(G, n, rank, world, "nccl", trials=10, seed=seed, level_cap=7,
                                    kernel=kernel, device=dev)
        else:
            r = mdg.min_weight(G, n, 10, seed, level_cap=7, kernel=kernel, device=dev)
        ev1.record()
        torch.cuda.synchronize()
        if step >= warm:
            ms.append(ev0.elapsed_time(ev1))
    tot = sum(ms)
    if dist is not None:
        t = torch.tensor([tot], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot = float(t.item())
    dev.close()
    parity6 = r.capped and r.levels[:6] == gold6["levels"] and _trace_matches(r, {**gold6, "rounds": gold6["rounds"]})
    parity7 = (r.levels == gold7["levels"] and _trace_matches(r, gold7)) if gold7 else None
    return {"workload": "cfg4 [300,200] seed 11, BZ to level cap 7: ONE code, every round of >= 2e8 "
                        "codewords split across the ranks (contiguous tile ranges), its key "
                        "min-reduced by an in-stream NCCL allreduce(min); N = 1: the same run on one GPU",
            "ranks": world, "scaling": "strong", "steps": steps,
            "ms_per_run": tot / steps, "codewords": int(r.combinations),
            "cw_per_s": r.combinations / (tot / steps * 1e-3),
            "h2d_bytes_per_run": int(r.h2d_bytes), "d2h_bytes_per_run": int(r.d2h_bytes),
            "levels": r.levels, "parity_cap6_vs_reference": bool(parity6),
            "parity_cap7_vs_reference": parity7,
            "path": "mdg_min_weight_dist (NCCL)" if world > 1 else "mdg_min_weight"}


def configs_table(mdg, dev):
    """Time-to-d (front door, host Gamma search included, one code at a time) of the other
    BASELINE configs with parity flags against the reference goldens (tests/golden)."""
    out = []
    for name, cap, file in (("cfg1", 0, "configs"), ("cfg3", 0, "configs"), ("cfg4", 5, "configs"),
                            ("cfg4", 6, "configs_cap4_6")):
        case = _gold(name, file)
        g = case["gen"]
        G = mdg.gen_matrix(g["n"], g["k"], g["seed"], True)
        best = None
        for _ in range(3):
            t0 = time.perf_counter()
            r = mdg.min_weight(G, g["n"], 10, g["seed"], level_cap=cap, device=dev)
            dt = time.perf_counter() - t0
            best = dt if best is None else min(best, dt)
        ok = (r.d == (case["U_final"] if cap else case["d"])) and _trace_matches(r, case)
        out.append({"config": f"{name}" + (f" cap {cap}" if cap else ""), "d": r.d,
                    "capped": r.capped, "ms": best * 1e3, "codewords": int(r.combinations),
                    "parity_vs_reference": bool(ok)})
    # config 5: the histograms of levels 1..5, every bin against the golden
    with open(os.path.join(ROOT, "tests", "golden", "cfg5_hist.json")) as f:
        h = json.load(f)["data"]
    M = mdg.gen_matrix(256, 100, 3, identity=False)
    dev.load_gammas(M, 256, ranks=None)
    ms, ok, cw = 0.0, True, 0
    for lv in h["levels"]:
        o, hist = dev.round_hist(0, lv["c"], 256)
        ms += o.device_ms
        cw += o.evaluated
        ok = ok and hist.tolist() == lv["hist"] and o.min_weight == lv["min"]
    lv5_ms = o.device_ms
    out.append({"config": "cfg5 histograms c=1..5", "ms_kernels": ms, "codewords": cw,
                "cw_per_s_c1_to_5": cw / (ms * 1e-3), "cw_per_s_c5": h["levels"][-1]["count"] / (lv5_ms * 1e-3),
                "parity_vs_reference": bool(ok)})
    # the same matrix at level 6 (1.19e9 codewords): the histogram kernel's steady state (level
    # 5 is a 0.1 ms launch); 4 POPC per 256-bit codeword bound it at 16 POPC/clk/SM
    with open(os.path.join(ROOT, "tests", "golden", "cfg5_hist_c6.json")) as f:
        lv6 = json.load(f)["data"]["level"]
    best = None
    for _ in range(3):
        o, hist = dev.round_hist(0, 6, 256)
        best = o.device_ms if best is None else min(best, o.device_ms)
    ok6 = hist.tolist() == lv6["hist"] and o.min_weight == lv6["min"]
    rate = lv6["count"] / (best * 1e-3)
    out.append({"config": "cfg5 matrix, histogram of level 6", "ms_kernels": best, "codewords": lv6["count"],
                "cw_per_s": rate, "frac_of_4popc_xu_bound": rate / (POPC_PER_S_MEASURED / 4.0),
                "parity_vs_reference": bool(ok6)})
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="mdg", choices=["mdg", "reference"])
    ap.add_argument("--kernel", default="tab", choices=["tab", "rd"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-strong", action="store_true", help="skip the one-code split (strong) leg")
    ap.add_argument("--no-configs", action="store_true", help="skip the other configs' time-to-d table")
    ap.add_argument("--streams", type=int, default=4,
                    help="codes in flight at once on one GPU (value: threads over resident "
                         "contexts; e2e: mdg_min_weight_batch)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "mdg":
        args.warmup = 3

    rank = env_int("RANK", 0)
    world = env_int("WORLD_SIZE", args.gpus if "RANK" in os.environ else 1)
    local = env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        return run_reference_arm(args, rank, world)

    import numpy as np
    import torch
    import paper_1911_08963_b200 as mdg

    # MDG_BENCH_BACKEND=gloo: plumbing check of the multi-rank path with several ranks on the
    # GPUs present (ranks share a GPU; their kernels never wait on each other) -- not a
    # scaling measurement
    backend = os.environ.get("MDG_BENCH_BACKEND", "nccl")
    if backend == "gloo":
        local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    red_dev = "cpu" if backend == "gloo" else f"cuda:{local}"
    dist = None
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend == "gloo":
            dist.init_process_group("gloo", rank=rank, world_size=world)
        else:
            dist.init_process_group("nccl", rank=rank, world_size=world,
                                    device_id=torch.device("cuda", local))
    kernel = mdg.KERNEL_TAB if args.kernel == "tab" else mdg.KERNEL_RD

    # expected answers (tests/golden, produced from the reference): d per seed
    with open(os.path.join(ROOT, "tests", "golden", "configs.json")) as f:
        gold = {c["name"]: c for c in json.load(f)["data"]}
    expect_d = [gold[f"cfg2_s{s}"]["d"] for s in SEEDS]

    # Codes are independent objects: every rank runs the eight-code step on its GPU (no
    # data-path collective; per-GPU work fixed: weak scaling). One context per code with its
    # Gamma set resident in HBM, plus the host matrices.
    mine = list(range(len(SEEDS)))
    Gs = [mdg.gen_matrix(N, K, SEEDS[i], True) for i in mine]
    gsets = [mdg.GammaSet.build(G, N, 10, SEEDS[i]) for G, i in zip(Gs, mine)]
    devs = [mdg.Device(local) for _ in mine]
    for d, gs in zip(devs, gsets):
        d.load_gset(gs)
    anchor = devs[0] if devs else mdg.Device(local)

    from concurrent.futures import ThreadPoolExecutor
    pool = ThreadPoolExecutor(max_workers=max(1, args.streams))

    def one_loop(x):
        d, gs, i = devs[x], gsets[x], mine[x]
        r = d.bz_loop(gs, kernel=kernel)
        if r.d != expect_d[i] or not r.witness_ok:
            raise SystemExit(f"parity failure on seed {SEEDS[i]}: d={r.d} expected {expect_d[i]}")
        return r

    def device_step():
        """This rank's level loops over the resident Gamma sets: with --streams > 1 up to that
        many codes run at once, each context on its own stream (mdg_bz_loop_device_batch);
        CUDA events on the torch stream bracket the whole step."""
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        if args.streams <= 1:
            runs = [one_loop(x) for x in range(len(devs))]
        elif os.environ.get("MDG_BENCH_PYTHON_POOL"):  # the former path: Python threads over bz_loop
            runs = list(pool.map(one_loop, range(len(devs))))
        else:  # mdg_bz_loop_device_batch: the library's own worker threads
            runs = mdg.bz_loop_batch(devs, gsets, kernel=kernel, streams=args.streams)
            for x, r in enumerate(runs):
                if r.d != expect_d[mine[x]] or not r.witness_ok:
                    raise SystemExit(f"parity failure on seed {SEEDS[mine[x]]}: d={r.d}")
        ev1.record()
        torch.cuda.synchronize()
        return ev0.elapsed_time(ev1), sum(r.evaluated for r in runs), sum(r.launches for r in runs)

    # the level-7 rounds of every code with the bound U they run under in the loop (the U
    # after the code's previous round), from one traced loop per code
    c7_rounds = []
    for x in range(len(devs)):
        r = one_loop(x)
        U = N - K + 1
        for (c, j, w, U_after) in r.rounds:
            if c == 7:
                c7_rounds.append((x, j, U))
            U = U_after

    def kernel_pass():
        """The dominant kernel alone (roofline): each level-7 round as one tab_round launch,
        bounded by its loop U, timed with CUDA events on the engine's stream, one launch at a
        time so each has the GPU to itself."""
        c7_cw, c7_ms = 0, 0.0
        for (x, j, U) in c7_rounds:
            o = devs[x].round_bounded(j, 7, U)
            c7_cw += o.evaluated
            c7_ms += o.device_ms
        return c7_cw, c7_ms

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=f"cuda:{local}")

    def l2_flush():
        flush.zero_()
        torch.cuda.synchronize()

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    # clocks sampled every 20 ms from the start of warm-up to the end of the e2e loop
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.05)
    for _ in range(args.warmup):
        device_step()

    ms_steps, cw_total, launches_total = [], 0, 0
    for _ in range(args.steps):
        l2_flush()
        barrier()
        ms, cw, ln = device_step()
        barrier()
        ms_steps.append(ms)
        cw_total += cw
        launches_total += ln
    c7_cw, c7_ms = 0, 0.0
    for _ in range(max(1, min(args.steps, 3))):
        l2_flush()
        barrier()
        a, b = kernel_pass()
        c7_cw += a
        c7_ms += b
    # BASELINE.md's roofline case: the config-2 level-7 round with early exit and bound
    # pruning off (exact minimum of all C(64,7) codewords), seed 1, Gamma_0
    ex_ms = []
    if rank == 0 and devs:
        devs[0].set_pruning(False)
        for _ in range(3):
            l2_flush()
            o = devs[0].round(0, 7)
            ex_ms.append(o.device_ms)
        ex_cw = o.evaluated
        devs[0].set_pruning(True)

    # e2e through the public front door from host buffers (pinned copies of G): this rank's
    # codes through mdg_min_weight_batch (--streams codes in flight); CUDA events on the
    # torch stream bracket each step, max over ranks
    e2e_ms, e2e_cw, h2d, d2h = [], 0, 0, 0
    Gpin = [torch.from_numpy(G).pin_memory().numpy() for G in Gs]
    for step in range(args.warmup + args.steps):
        l2_flush()
        barrier()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        runs = mdg.min_weight_batch(Gpin, N, trials=10, seed=[SEEDS[i] for i in mine], kernel=kernel,
                                    device=anchor, streams=args.streams)
        ev1.record()
        torch.cuda.synchronize()
        for x, r in enumerate(runs):
            if r.d != expect_d[mine[x]] or not r.witness_ok:
                raise SystemExit(f"e2e parity failure on seed {SEEDS[mine[x]]}")
        barrier()
        if step >= args.warmup:
            e2e_ms.append(ev0.elapsed_time(ev1))
            e2e_cw += sum(r.evaluated for r in runs)
            h2d += sum(r.h2d_bytes for r in runs)
            d2h += sum(r.d2h_bytes for r in runs)

    # SURVEY.md §8e's split of ONE code (the strong-scaling leg, at every N): config 4 to
    # level cap 7 (BASELINE.md's throughput / scaling case, 4.7e12 codewords): every round of
    # >= 2e8 codewords has its tiles split across the ranks and its key min-reduced by an
    # in-stream NCCL allreduce(min) (mdg_min_weight_dist); N = 1 is its single-GPU baseline.
    # Sigma C(k, c) over the executed rounds / max-rank wall (CUDA events on the torch stream).
    strong = None
    if world > 1 and backend == "gloo":
        strong = {"skipped": "MDG_BENCH_BACKEND=gloo plumbing run (ranks share a GPU; NCCL needs one GPU per rank)"}
    elif not args.no_strong:
        try:
            strong = strong_leg(mdg, torch, dist, rank, world, local, kernel, barrier,
                                warm=1, steps=max(1, min(args.steps, 3)))
        except Exception as e:  # reported, never fatal
            strong = {"error": str(e)[:300]}
    configs = None
    if rank == 0 and world == 1 and not args.no_configs:
        try:
            configs = configs_table(mdg, devs[0])
        except Exception as e:  # reported, never fatal
            configs = {"error": str(e)[:300]}
    clocks = sampler.stop()

    # max over ranks of time, sum over ranks of codewords
    tot_ms = sum(ms_steps)
    tot_e2e = sum(e2e_ms)
    if dist is not None:
        t = torch.tensor([tot_ms, tot_e2e, float(c7_ms)], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        c = torch.tensor([cw_total, e2e_cw, c7_cw, launches_total, h2d, d2h], dtype=torch.float64,
                         device=red_dev)
        dist.all_reduce(c, op=dist.ReduceOp.SUM)
        tot_ms, tot_e2e, c7_ms = [float(x) for x in t.tolist()]
        cw_total, e2e_cw, c7_cw, launches_total, h2d, d2h = [int(x) for x in c.tolist()]

    if rank == 0:
        value = cw_total / (tot_ms * 1e-3)
        e2e_value = e2e_cw / (tot_e2e * 1e-3)
        sms = devs[0].info()["sm_count"]
        nw = 2  # popcounts per codeword of the unpruned kernel (64 non-identity columns)
        achieved = c7_cw / (c7_ms * 1e-3) / world if c7_ms > 0 else 0.0
        popc = POPC_PER_S_MEASURED * sms / 148
        alu = ALU_PER_S_MEASURED * sms / 148
        peak_alu, peak_xu = alu / ALU_PER_CW_PRUNED, popc / XU_PER_CW_PRUNED
        peak = min(peak_alu, peak_xu)
        roofline = {
            "bound": "int_alu" if peak_alu <= peak_xu else "int_popc",
            "achieved": achieved / 1e9, "peak": peak / 1e9, "unit": "Gcw/s",
            "frac": achieved / peak, "traffic": DRAM_BYTES_PER_LAUNCH, "traffic_unit": "DRAM bytes per launch (ncu)",
            "kernel": ("tab_round<2,false>: one level-7 round per launch (621,216,192 codewords), "
                       "bound-pruned by the loop's U, CUDA-event timed on the engine stream "
                       "(in the chained loop both rounds of the level run as one tab_level launch, "
                       "profiles/r01m_tab_level_c7_ncu.txt)"),
            "peak_basis": ("integer issue-rate roofline of this kernel's op mix: min(ALU pipe 64/clk/SM = "
                           f"1.81e13 LOP3/s / {ALU_PER_CW_PRUNED} ALU ops per codeword, XU pipe 16/clk/SM = "
                           f"4.64e12 POPC/s / {XU_PER_CW_PRUNED} POPC per codeword); rates measured on B200 "
                           "(tools/pipes_microbench.cu), ops per codeword from ncu "
                           "(profiles/r02h_tab_round_c7_ncu.txt)"),
            "peak_alu": peak_alu / 1e9, "peak_xu": peak_xu / 1e9,
            "op_mix_per_codeword": ("stage 1: one bound per pair of codewords, popc(fold_a & fold_b) with "
                                    "fold = OR of the words of X ^ Y, built in 3 LOP3 from per-pair constants "
                                    "(1.5 LOP3 + 0.5 POPC per codeword), one min / warp vote per 16 codewords "
                                    "(two smem items); "
                                    "single-codeword folds (1 POPC) for vote groups the pair bound cannot "
                                    "reject; exact weight only where a codeword can still beat the bound"),
            "frac_vs_unpruned_popc_roofline": achieved / (popc / nw),
            "unpruned_c7": ({
                "what": "exact config-2 level-7 round with early exit and bound pruning off "
                        "(every codeword's weight computed), seed 1, Gamma_0, best of 3 "
                        "CUDA-event timings",
                "achieved": ex_cw / (min(ex_ms) * 1e-3) / 1e9, "unit": "Gcw/s",
                "peak_baseline_def": popc / 4 / 1e9,
                "frac_baseline_def": ex_cw / (min(ex_ms) * 1e-3) / (popc / 4),
                "baseline_def": "BASELINE.md: SMs x 16 POPC/clk x f / (2W), W = 2 u64 words per row",
                "peak_elided": popc / nw / 1e9,
                "frac_elided": ex_cw / (min(ex_ms) * 1e-3) / (popc / nw),
                "elided_def": "identity block elided: 64 compacted bits = 2 POPC per codeword",
            } if ex_ms else None),
            "frac_fixed_unit": (ex_cw / (min(ex_ms) * 1e-3) / (popc / nw) if ex_ms else None),
            "frac_fixed_unit_def": ("the exact-weight level-7 kernel (pruning off, every codeword weighed: "
                                    "2 POPC per codeword on the 64 non-identity columns) over the XU "
                                    "roofline of that fixed unit, 4.64e12 POPC/s / 2; `frac` above is the "
                                    "pruned kernel's issue efficiency on its own op mix, which a better "
                                    "pruning stage can lower"),
            "traffic_note": "DRAM 4.25 MB per launch (the tables, read once), 0.6% of HBM bandwidth: compute-bound",
            "hbm_check": hbm_check(achieved),
        }
        if clocks.get("sm_mhz"):
            roofline["frac_at_measured_clock"] = achieved / (peak * clocks["sm_mhz"] / 1965.0)
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            try:
                from oracle import ref
                if ref.available():
                    tr, dt, workers = cpu_baseline_reference(1)
                    cpu = {"value": tr["combinations"] / dt, "unit": "cw/s", "cores": workers,
                           "kind": "reference",
                           "sample": f"config-2 seed 1 to termination (d={tr['d']}, "
                                     f"{tr['combinations']} codewords, {dt:.2f} s), reference "
                                     "round_saved_parallel s=5, -O3 -march=x86-64-v3"}
                else:
                    tr, dt = cpu_baseline_port(1)
                    cpu = {"value": tr.combinations / dt, "unit": "cw/s", "cores": 1, "kind": "port",
                           "sample": "config-2 seed 1, levels c<=6, C restatement, 1 thread"}
            except Exception as e:  # reported, never fatal
                cpu = {"value": None, "unit": "cw/s", "cores": 0, "kind": "unavailable",
                       "sample": str(e)[:200]}
        e2e_weak = {"value": e2e_value, "unit": "cw/s", "h2d_bytes_per_step": h2d // args.steps,
                    "d2h_bytes_per_step": d2h // args.steps, "ms_per_step": tot_e2e / args.steps,
                    "workload": WORKLOAD,
                    "path": "mdg_min_weight_batch (C ABI) from pinned host matrices: row basis + Gamma "
                            "search + H2D + level loop + witness + D2H"}
        weak = {"value": value, "unit": "cw/s", "ms_per_step": tot_ms / args.steps,
                "workload": WORKLOAD, "scaling": "weak", "e2e": e2e_weak,
                "parallelism": (f"{world} ranks, each running the eight-code step ({args.streams} "
                                "codes in flight per GPU); independent codes, no data-path collective"
                                if world > 1 else
                                f"single GPU, {min(args.streams, len(SEEDS))} codes in flight")}
        # N > 1: the headline is the strong leg (one code's rounds split across the ranks,
        # north_star's per-level partition); the eight-code step stays as `weak_step`
        strong_ok = isinstance(strong, dict) and "cw_per_s" in strong
        headline_strong = world > 1 and strong_ok
        line = {
            "metric": "codewords_evaluated_per_sec",
            "value": strong["cw_per_s"] if headline_strong else value, "unit": "cw/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": strong["ms_per_run"] if headline_strong else tot_ms / args.steps,
            "higher_is_better": True, "scaling": "strong" if headline_strong else "weak",
            "vs_baseline": None, "dtype": "u32",
            "data": "synthetic (mt19937_64 seeds 1..8, SURVEY.md §8d)",
            "config": {"workload": strong["workload"] if headline_strong else WORKLOAD,
                       "kernel": args.kernel,
                       "parallelism": (f"{world} ranks over NCCL: one code, rounds split" if headline_strong
                                       else weak["parallelism"]),
                       "counting": ("value counts codewords the way the reference's RoundStats.combinations "
                                    "does (C(k,c) per executed round; the device evaluates each against "
                                    "the running bound, most of them with a pair / fold lower bound only: "
                                    "bound-screened, not all weighed exactly -- roofline.frac_fixed_unit "
                                    "is the exact-weight kernel on a fixed unit)"),
                       "l2": "flushed between steps (256 MiB write); working set < 1 MiB",
                       "codewords_per_step": cw_total // args.steps,
                       "ms_step_min_median_max": [min(ms_steps), statistics.median(ms_steps), max(ms_steps)],
                       "e2e_ms_step_min_median_max": [min(e2e_ms), statistics.median(e2e_ms), max(e2e_ms)],
                       "ms_per_code_amortized": tot_ms / args.steps / len(SEEDS),
                       "d": expect_d},
            "weak_step": weak if world > 1 else None,
            "strong": strong,
            "configs": configs,
            # N > 1: the strong leg IS the front-door call on a host matrix (row basis, Gamma
            # search, H2D, split level loop, witness, D2H inside its timed region), so the
            # headline is its own end-to-end number; the eight-code e2e stays in weak_step
            "e2e": ({"value": strong["cw_per_s"], "unit": "cw/s",
                     "h2d_bytes_per_step": strong["h2d_bytes_per_run"],
                     "d2h_bytes_per_step": strong["d2h_bytes_per_run"],
                     "ms_per_step": strong["ms_per_run"], "workload": strong["workload"],
                     "path": "mdg_min_weight_dist (C ABI) from the host matrix, per rank: row basis + Gamma "
                             "search + H2D + split level loop (NCCL) + witness + D2H"}
                    if headline_strong else e2e_weak),
            "roofline": roofline,
            "cpu_baseline": cpu,
            "clocks": clocks,
            "gpu_launches": launches_total,
        }
        print(json.dumps(line), flush=True)
    for d in devs:
        d.close()
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
