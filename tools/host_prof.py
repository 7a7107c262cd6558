import sys, time
sys.path.insert(0, "/root/repo")
import torch
import bench
import paper_1406_5687_b200 as tcb
from paper_1406_5687_b200 import distributed as D, space_efficient as SE, _lib
from paper_1406_5687_b200.partitioning import partition_ranges, range_bounds
raw = bench.host_raw_edges("cfg2", pin=True)
g = tcb.build_graph(tcb.normalize(tcb.RawGraph(n=0, edges=raw.cuda())))
ops = D.DeviceOps()
P = 8
sb = range_bounds(partition_ranges(g, tcb.CostKind.PRED_SUM, P))
shards = [D.shard_of(g, int(sb[r]), int(sb[r + 1])) for r in range(P)]
def T(name, fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize(); t0 = time.perf_counter(); out = fn(); torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    print(f"  {name:28s} {best*1e3:7.3f} ms"); return out
for r in (0, 7):
    sh = shards[r]
    print("rank", r)
    rec_v, counts = T("records", lambda: ops.records(sh, sb, P, r))
    lens, ids = T("pack", lambda: ops.pack(sh, rec_v))
    # fake inbox: rank 7 receives everyone's lists -> emulate with its own
    o1 = T("owner_segments local", lambda: SE.owner_segments(sh.indptr, sh.indices, sh.lo, sh.hi, 0))
    owner, segs, k = o1
    T("count_segments local", lambda: SE.count_segments(sh.indptr, sh.indices, sh.indices, owner[:k].contiguous(), segs[:2*k].contiguous(), k, sh.hi - sh.lo))
    def csr():
        dev = owner.device; n_owner = sh.hi - sh.lo
        row = torch.empty(n_owner + 1, dtype=torch.int64, device=dev)
        rsegs = torch.empty(max(2 * k, 2), dtype=torch.int32, device=dev)
        cost = torch.empty(n_owner + 1, dtype=torch.int64, device=dev)
        _lib.call("tc_segments_csr", _lib.ptr(owner), _lib.ptr(segs), int(k), int(n_owner), _lib.ptr(sh.indptr), _lib.ptr(row), _lib.ptr(rsegs), _lib.ptr(cost), _lib.stream())
    T("  segments_csr only", csr)
