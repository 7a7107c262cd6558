"""Dev tool: block-tier owners (d^ > 512) by id span of N^_u, weighted by
their engine cost, for one config."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1406_5687_b200 as tcb

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
raw = bench.host_raw_edges(cfg, pin=True)
g = tcb.build_graph(tcb.normalize(tcb.RawGraph(n=0, edges=raw.cuda())))
ip, ix = g.eff_indptr, g.eff_indices
d = ip[1:] - ip[:-1]
cost = g._rev_cost[1:] - g._rev_cost[:-1]
for lo, hi in ((256, 512), (512, 1 << 40)):
    sel = (d > lo) & (d <= hi)
    u = torch.nonzero(sel).flatten()
    first = ix[ip[u]].long()
    last = ix[ip[u + 1] - 1].long()
    span = last - first + 1
    c = cost[u].double()
    tot = c.sum().item()
    print(f"{cfg} tier d in ({lo},{hi}]: owners {u.numel()} cost {tot:.3e} (of {cost.double().sum().item():.3e})")
    for lim in (1 << 15, 1 << 18, 262144, 1 << 19, 1 << 20, 1 << 21, 1 << 22):
        f = c[span <= lim].sum().item() / max(tot, 1)
        print(f"  span <= {lim:>8}: owners {(span <= lim).sum().item():>8}  cost share {f:.3f}")
    print(f"  max span {span.max().item() if u.numel() else 0}, n = {g.n}")
