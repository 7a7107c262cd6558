"""Distribution of owner-table id spans, weighted by probe work, per engine tier (dev tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1406_5687_b200 as tcb  # noqa: E402

for cfg in sys.argv[1].split(","):
    raw = bench.host_raw_edges(cfg, pin=True)
    g = tcb.build_graph(tcb.normalize(tcb.RawGraph(n=0, edges=raw.cuda())))
    ip = g.eff_indptr
    d = (ip[1:] - ip[:-1])
    ix = g.eff_indices.long()
    nz = d > 0
    first = torch.zeros_like(d)
    last = torch.zeros_like(d)
    first[nz] = ix[ip[:-1][nz]]
    last[nz] = ix[ip[1:][nz] - 1]
    span = (last - first + 1).clamp(min=0)
    work = (g._rev_cost[1:] - g._rev_cost[:-1]).double()
    tot = work.sum().item()
    print(f"{cfg}: n={g.n} m={g.m} total probe work {tot:.3e}")
    for name, lo, hi in (("small", 1, 256), ("mid", 257, 512), ("block", 513, 4096), ("global", 4097, 1 << 40)):
        sel = (d >= lo) & (d <= hi)
        w = work[sel]
        s = span[sel]
        wt = w.sum().item()
        row = f"  {name:6s} owners={int(sel.sum()):9d} work={wt / max(tot, 1):6.1%}"
        for lim in (1 << 12, 1 << 14, 1 << 16, 1 << 18, 1 << 19, 1 << 20):
            row += f"  span<={lim >> 10}K:{(w[s <= lim].sum().item() / max(wt, 1)):6.1%}"
        print(row, flush=True)
    del g
    torch.cuda.empty_cache()
