"""Per-tier engine rates (dev tool): probes, segments, table ids and owners of
each engine tier against its measured device time, per config."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1406_5687_b200 as tcb  # noqa: E402
from paper_1406_5687_b200.sequential import count_middle  # noqa: E402

flush = torch.empty(1 << 28, dtype=torch.uint8, device="cuda")
for cfg in sys.argv[1].split(","):
    raw = bench.host_raw_edges(cfg, pin=True)
    g = tcb.build_graph(tcb.normalize(tcb.RawGraph(n=0, edges=raw)))
    out = torch.empty(1, dtype=torch.int64, device="cuda")
    count_middle(g, out=out)
    ms, tiers = bench._engine_ms(lambda: count_middle(g, out=out), 5, flush)
    d = g.eff_deg.to(torch.int64)
    cost = g._rev_cost[1:] - g._rev_cost[:-1]
    preds = g._rev_indptr[1:] - g._rev_indptr[:-1]
    own = cost > 0
    probes = torch.where(own, cost - 2 * preds - d - 16, torch.zeros_like(cost))
    tier = torch.where(d <= 128, 0, torch.where(d <= 512, 1, 2))
    for k, name in enumerate(("small", "mid", "block")):
        sel = own & (tier == k)
        P_, S_, T_, O_ = (int(probes[sel].sum()), int(preds[sel].sum()), int(d[sel].sum()), int(sel.sum()))
        if O_ == 0:
            continue
        t = tiers[k]
        print(f"{cfg} {name}: {t:.2f} ms owners {O_} probes {P_ / 1e6:.1f}M segs {S_ / 1e6:.1f}M tab {T_ / 1e6:.1f}M "
              f"-> {t * 1e6 / max(P_, 1):.3f} ns/probe, {t * 1e6 / max(S_, 1):.2f} ns/seg, "
              f"{t * 1e6 / max(O_, 1):.1f} ns/owner", flush=True)
    del g
    torch.cuda.empty_cache()
