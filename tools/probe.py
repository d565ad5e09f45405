"""Quick per-round throughput probe (development tool, not the bench)."""
import sys
import time

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_1911_08963_b200 as mdg  # noqa: E402


def probe(n, k, seed, levels, kernel=0, reps=3, cutoff=0):
    G = mdg.gen_matrix(n, k, seed, True)
    gs = mdg.GammaSet.build(G, n, 10, seed)
    dev = mdg.Device(0)
    dev.load_gset(gs)
    dev.set_kernel(kernel)
    sms = dev.info()["sm_count"]
    for c in levels:
        for j in range(gs.m):
            best = None
            for _ in range(reps):
                o = dev.round_bounded(j, c, cutoff) if cutoff else dev.round(j, c)
                best = o if best is None or o.device_ms < best.device_ms else best
            cw = best.evaluated / (best.device_ms * 1e-3)
            print(f"[{n},{k}] kernel={'tab' if kernel == 0 else 'rd'} cut={cutoff} c={c} j={j} w={best.min_weight} "
                  f"cw={best.evaluated} ms={best.device_ms:.3f} cw/s={cw:.3e} "
                  f"cw/clk/SM@1.965={cw / (sms * 1.965e9):.2f}", flush=True)
    dev.close()


if __name__ == "__main__":
    probe(128, 64, 1, [5, 6, 7])
    probe(128, 64, 1, [6, 7], cutoff=15)
    probe(128, 64, 1, [6, 7], cutoff=17)
    probe(300, 200, 11, [5], reps=1, cutoff=26)
    probe(256, 32, 7, [9], cutoff=76)
    probe(128, 64, 1, [5, 6], kernel=1, reps=1)
    probe(256, 32, 7, [7, 9])
    probe(300, 200, 11, [4, 5, 6], reps=1)
    G = mdg.gen_matrix(256, 100, 3, identity=False)
    dev = mdg.Device(0)
    dev.load_gammas(G, 256, ranks=None)
    for c in (4, 5):
        o = dev.round(0, c)
        o = dev.round(0, c)
        oh, _ = dev.round_hist(0, c, 256)
        oh, _ = dev.round_hist(0, c, 256)
        print(f"cfg5 c={c} min={o.min_weight} ms={o.device_ms:.3f} cw/s={o.evaluated/(o.device_ms*1e-3):.3e} "
              f"hist_ms={oh.device_ms:.3f} hist cw/s={oh.evaluated/(oh.device_ms*1e-3):.3e}")
    t0 = time.time()
    r = mdg.min_weight(mdg.gen_matrix(128, 64, 1, True), 128, 10, 1)
    print(f"cfg2 s1 e2e: d={r.d} wall={time.time()-t0:.3f}s loop={r.loop_seconds:.4f}s dev={r.device_seconds:.4f}s "
          f"gamma={r.gamma_seconds:.4f}s evaluated={r.evaluated} launches={r.launches}")
