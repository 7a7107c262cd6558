import sys, time, os
sys.path.insert(0, '/root/repo')
import torch, ctypes
import bench
import paper_1406_5687_b200 as tcb
from paper_1406_5687_b200 import graph as G, _lib
raw = bench.host_raw_edges("cfg2", pin=True)
orig_call = _lib.call
log = []
def timed_call(name, *a):
    t0 = time.perf_counter(); r = orig_call(name, *a); log.append((name, t0, time.perf_counter())); return r
_lib.call = timed_call
G._lib.call = timed_call
for it in range(6):
    log.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    nr = tcb.normalize(tcb.RawGraph(n=0, edges=raw))
    t1 = time.perf_counter()
    g = tcb.build_graph(nr)
    t2 = time.perf_counter()
    T = tcb.count_triangles_seq(g)
    t3 = time.perf_counter()
    if it >= 3:
        print(f"normalize {1e3*(t1-t0):.3f} ms, build (host, async) {1e3*(t2-t1):.3f} ms, count {1e3*(t3-t2):.3f} ms")
        for name, a, b in log:
            print(f"   {name:24s} start +{1e3*(a-t0):8.3f} ms  dur {1e3*(b-a):8.3f} ms")
    del g, nr
