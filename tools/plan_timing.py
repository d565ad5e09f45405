import sys, time
sys.path.insert(0, '.')
import paper_1911_08963_b200 as mdg
dev = mdg.Device(0)
for (n,k,s) in [(256,32,7),(128,64,1),(80,40,1)]:
    G = mdg.gen_matrix(n,k,s,True)
    for rep in range(3):
        t0=time.perf_counter(); r = mdg.min_weight(G, n, 10, s, device=dev); t=time.perf_counter()-t0
        print(n,k,s,'wall_ms',round(t*1e3,3),'loop',round(r.loop_seconds*1e3,3),'dev',round(r.device_seconds*1e3,3),'gamma',round(r.gamma_seconds*1e3,3), flush=True)
