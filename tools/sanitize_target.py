"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck): config 1 end to end
(chained loop, fused levels, witness), config 2 seed 1 to level cap 4 in both kernels and round
modes, a split round pair through the in-process exchange group, a config-5 level-2 histogram,
the brute force on a [24,12] code and the GPU permutation search. Every result is checked."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_08963_b200 as mdg  # noqa: E402

dev = mdg.Device(0)
G = mdg.gen_matrix(80, 40, 1, True)
r = mdg.min_weight(G, 80, 10, 1, device=dev)
assert r.d == 9 and r.witness_ok
G2 = mdg.gen_matrix(128, 64, 1, True)
for kernel in (mdg.KERNEL_TAB, mdg.KERNEL_RD):
    for exact in (False, True):
        r2 = mdg.min_weight(G2, 128, 10, 1, level_cap=4, kernel=kernel, exact_rounds=exact, device=dev)
        assert r2.capped and r2.witness_ok
d1 = mdg.Device(0)
runs = mdg.min_weight_multi(G, 80, [dev, d1], trials=10, seed=1, split_min=1)
assert all(x.d == 9 and x.witness_ok for x in runs)
d1.close()
M = mdg.gen_matrix(256, 100, 3, identity=False)
dev.load_gammas(M, 256, ranks=None)
o, h = dev.round_hist(0, 2, 256)
assert int(h.sum()) == 4950 and o.min_weight == int((h != 0).argmax())
B = mdg.gen_matrix(24, 12, 5, True)
b = mdg.brute_force(B, 24, device=dev)
assert b.witness_ok
gs_gpu = mdg.GammaSet.build(G2, 128, 200, 1, device=dev)
gs_host = mdg.GammaSet.build(G2, 128, 200, 1)
assert [gs_gpu.hash(j) for j in range(gs_gpu.m)] == [gs_host.hash(j) for j in range(gs_host.m)]
dev.close()
print("sanitize target ok")
