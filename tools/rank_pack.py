"""One rank's surrogate pack (tc_shard_send_pack) in isolation: timing and, under ncu, counters (dev tool)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1406_5687_b200 import sharded as S  # noqa: E402

cfg, P, rank = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
raw = bench.host_raw_edges(cfg, pin=True).cuda()
shards, _ = S.emulate_build(raw, P, cost="engine")
del raw
sh = shards[rank]
ops = S.ShardOps()
sd, sz = ops.send_sizes(sh, P, rank)
nl, nw = int(sz[0].sum()), int(sz[1].sum())
print(f"{cfg} P={P} rank {rank}: rows {sh.hi - sh.lo} ids {sh.m_local} -> lists {nl} words {nw} ({sz[0].tolist()} / {sz[1].tolist()})")
from paper_1406_5687_b200 import _lib as L  # noqa: E402

lens = torch.empty(max(nl, 1), dtype=torch.int32, device="cuda")
ids = torch.empty(max(nw, 4), dtype=torch.int32, device="cuda")
for _ in range(5):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    L.call("tc_shard_send_pack", L.ptr(sh.indptr), L.ptr(sh.indices), sh.hi - sh.lo, L.ptr(sh.pool_indptr),
           L.ptr(sh.pool), L.ptr(sh.cache["bounds_dev"]), P, rank, L.ptr(sd), L.ptr(lens), L.ptr(ids), L.stream())
    e.record()
    torch.cuda.synchronize()
    t = s.elapsed_time(e) / 1e3
    print(f"pack {1e3 * t:.2f} ms  ({8 * nw / t / 1e9:.0f} GB/s read+write)")
