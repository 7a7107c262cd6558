import os, sys, ctypes
sys.path.insert(0, '/root/repo')
import torch, numpy as np
import bench
from paper_1406_5687_b200 import sharded as S, _lib
raw = bench.host_raw_edges(sys.argv[1], pin=True).cuda()
P = int(sys.argv[2])
shards, _ = S.emulate_build(raw, P, cost=sys.argv[3])
del raw
ops = S.ShardOps()
def timing(fn, reps=5):
    _lib.lib().tc_engine_timing(1, None, None, None)
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    tot, nl = ctypes.c_double(), ctypes.c_longlong(); tiers = (ctypes.c_double * 3)()
    _lib.lib().tc_engine_timing(0, ctypes.byref(tot), ctypes.byref(nl), tiers)
    k = max(1, nl.value); return tot.value / k, [t / k for t in tiers], nl.value
for r, sh in enumerate(shards):
    o, plan = ops.start_local(sh); torch.cuda.synchronize()
    d = (sh.indptr[1:] - sh.indptr[:-1])
    print(f"rank {r}: [{sh.lo},{sh.hi}) m_local {sh.m_local} d^ mean {float(d.float().mean()):.0f} local engine ms %.3f tiers %s" % (lambda x: (x[0], [round(v,3) for v in x[1]]))(timing(lambda: ops.start_local(sh))), flush=True)
