import sys; sys.path.insert(0,'.')
import paper_1911_08963_b200 as mdg, time
dev = mdg.Device(0)
Gs=[mdg.gen_matrix(128,64,s,True) for s in range(1,9)]
for rep in range(4):
    t0=time.perf_counter(); runs=mdg.min_weight_batch(Gs,128,trials=10,seed=list(range(1,9)),device=dev,streams=4); t1=time.perf_counter()
    print("batch ms", (t1-t0)*1e3, file=sys.stderr, flush=True)
