import sys, time
sys.path.insert(0,'.')
import paper_1911_08963_b200 as mdg
dev=mdg.Device(0)
G=mdg.gen_matrix(256,32,7,True)
for rep in range(3):
    t0=time.perf_counter(); r=mdg.min_weight(G,256,10,7,device=dev); t1=time.perf_counter()
    print(f"front: wall {1e3*(t1-t0):.3f} gamma {1e3*r.gamma_seconds:.3f} loop {1e3*r.loop_seconds:.3f} dev {1e3*r.device_seconds:.3f} launches {r.launches}")
gs=mdg.GammaSet.build(G,256,10,7)
for rep in range(3):
    t0=time.perf_counter(); dev.load_gset(gs); t1=time.perf_counter(); r=dev.bz_loop(gs); t2=time.perf_counter(); r2=dev.bz_loop(gs); t3=time.perf_counter()
    print(f"load {1e3*(t1-t0):.3f} cold loop wall {1e3*(t2-t1):.3f} (timer {1e3*r.loop_seconds:.3f}) warm loop wall {1e3*(t3-t2):.3f} (timer {1e3*r2.loop_seconds:.3f})")
