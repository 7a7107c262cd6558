import os, sys, time
sys.path.insert(0, "/root/repo")
import torch
from torch.profiler import ProfilerActivity, profile
import bench
import paper_1406_5687_b200 as tcb
from paper_1406_5687_b200 import distributed as D
from paper_1406_5687_b200.partitioning import partition_ranges, range_bounds
raw = bench.host_raw_edges("cfg2", pin=True)
g = tcb.build_graph(tcb.normalize(tcb.RawGraph(n=0, edges=raw.cuda())))
ops = D.DeviceOps()
for P in (2, 8):
    sb = range_bounds(partition_ranges(g, tcb.CostKind.PRED_SUM, P))
    shards = [D.shard_of(g, int(sb[r]), int(sb[r + 1])) for r in range(P)]
    inbox = {r: [] for r in range(P)}
    for r, sh in enumerate(shards):
        rec_v, counts = ops.records(sh, sb, P, r)
        lens, ids = ops.pack(sh, rec_v)
        ln = lens.cpu().numpy(); s = i = 0
        for j in range(P):
            c = int(counts[j]); k = int(ln[s:s+c].sum())
            if c: inbox[j].append((lens[s:s+c], ids[i:i+k]))
            s += c; i += k
    for r in (0, P - 1):
        sh = shards[r]
        rl = torch.cat([x[0] for x in inbox[r]]) if inbox[r] else torch.zeros(0, dtype=torch.int64, device="cuda")
        ri = torch.cat([x[1] for x in inbox[r]]) if inbox[r] else torch.zeros(0, dtype=torch.int32, device="cuda")
        def step():
            rec_v, counts = ops.records(sh, sb, P, r)
            ops.pack(sh, rec_v)
            ops.count(sh, rl, ri)
        step(); torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
            t0 = time.perf_counter(); step(); torch.cuda.synchronize(); wall = time.perf_counter() - t0
        rows = {}
        for e in prof.events():
            if e.device_type == torch.autograd.DeviceType.CUDA:
                k = e.name[:70]; t, c = rows.get(k, (0.0, 0)); rows[k] = (t + e.device_time / 1000.0, c + 1)
        tot = sum(t for t, _ in rows.values())
        print(f"P={P} r={r}: wall {wall*1e3:.2f} ms, device {tot:.2f} ms, recv ids {ri.numel()/1e6:.1f}M, own m {sh.m/1e6:.1f}M")
        for k, (t, c) in sorted(rows.items(), key=lambda kv: -kv[1][0])[:9]:
            print(f"    {t:7.3f} ms x{c:3d} {k}")
