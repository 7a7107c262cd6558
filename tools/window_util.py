"""Lane utilisation of the engine's 32-chunk windows (dev tool): probes /
(windows x 128 id slots), from the reverse CSR of a config."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1406_5687_b200 as tcb  # noqa: E402

for cfg in sys.argv[1].split(","):
    raw = bench.host_raw_edges(cfg, pin=True)
    g = tcb.build_graph(tcb.normalize(tcb.RawGraph(n=0, edges=raw.cuda())))
    seg = g._rev_seg.view(-1, 2).long()
    s, e = seg[:, 0], seg[:, 1]
    ln = e - s
    nz = ln > 0
    ch = torch.where(nz, (e + 3) // 4 - s // 4, torch.zeros_like(s))
    rip = g._rev_indptr
    row = torch.repeat_interleave(torch.arange(g.n, device="cuda"), rip[1:] - rip[:-1])
    pos = torch.arange(seg.shape[0], device="cuda") - rip[row]
    grp = row * 4096 + pos // 32  # (owner, group) key; < 4096 groups per owner assumed
    ukeys, inv = torch.unique(grp, return_inverse=True)
    tot = torch.zeros(ukeys.numel(), dtype=torch.long, device="cuda").index_add_(0, inv, ch)
    windows = ((tot + 31) // 32).sum().item()
    probes = ln.sum().item()
    d = g.eff_indptr[1:] - g.eff_indptr[:-1]
    indeg = rip[1:] - rip[:-1]
    w = (g._rev_cost[1:] - g._rev_cost[:-1]).double()
    frac_small = (w[indeg < 8].sum() / w.sum()).item()
    print(f"{cfg}: probes {probes/1e9:.3f} G, windows {windows/1e6:.1f} M, utilisation {probes / (windows * 128):.2%}, "
          f"groups {ukeys.numel()/1e6:.1f} M, avg seg len {probes / max(1, int(nz.sum())):.1f}, "
          f"work share of owners with < 8 preds {frac_small:.1%}", flush=True)
    del g
    torch.cuda.empty_cache()
