import sys, time, os, ctypes
sys.path.insert(0, '/root/repo')
import torch
import bench
import paper_1406_5687_b200 as tcb
from paper_1406_5687_b200 import graph as G, _lib
raw = bench.host_raw_edges("cfg2", pin=True)
for _ in range(3):
    g = tcb.build_graph(tcb.normalize(tcb.RawGraph(n=0, edges=raw))); tcb.count_triangles_seq(g); del g
torch.cuda.synchronize()
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h = raw
    ok = h.is_pinned()
    t1 = time.perf_counter()
    m_raw = h.shape[0]
    staging = torch.empty((m_raw, 2), dtype=torch.int32, device="cuda")
    out = torch.empty((m_raw, 2), dtype=torch.int32, device="cuda")
    deg = torch.empty(2 * m_raw + 1, dtype=torch.int32, device="cuda")
    t2 = time.perf_counter()
    m, n, valid = ctypes.c_int64(0), ctypes.c_int64(0), ctypes.c_int32(0)
    _lib.call("tc_normalize_host", _lib.ptr(h), m_raw, _lib.ptr(staging), _lib.ptr(out), ctypes.byref(m), ctypes.byref(n), _lib.ptr(deg), ctypes.byref(valid), _lib.stream())
    t3 = time.perf_counter()
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    print(f"is_pinned {1e3*(t1-t0):.3f} ms, allocs {1e3*(t2-t1):.3f} ms, tc_normalize_host call {1e3*(t3-t2):.3f} ms, tail {1e3*(t4-t3):.3f}")
    del staging, out, deg
