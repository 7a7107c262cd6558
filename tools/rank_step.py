"""Per-rank step time of the multi-GPU surrogate / direct / replicated
steps, emulated on one GPU (dev tool): each rank's device work runs in turn
with the exchange replaced by local buffer passing, so max over ranks
approximates the N-GPU step minus NCCL transfer time."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1406_5687_b200 as tcb  # noqa: E402
from paper_1406_5687_b200 import distributed as D  # noqa: E402
from paper_1406_5687_b200.partitioning import balanced_bounds, partition_ranges, range_bounds  # noqa: E402
from paper_1406_5687_b200.sequential import count_middle, count_middle_part  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--ranks", default="2,4,8")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--modes", default="surrogate,direct,replicated")
a = ap.parse_args()
MODES = set(a.modes.split(","))
raw = bench.host_raw_edges(a.config, pin=True)
g = tcb.build_graph(tcb.normalize(tcb.RawGraph(n=0, edges=raw.cuda())))
ops = D.DeviceOps()
out = torch.empty(1, dtype=torch.int64, device="cuda")


def timed(fn):
    best = 1e9
    for _ in range(a.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best * 1e3




def surrogate_step(P, sb):
    shards = [D.shard_of(g, int(sb[r]), int(sb[r + 1])) for r in range(P)]
    # surrogate: records+pack on the sender, segments+count on the receiver
    send = [timed(lambda sh=sh, r=r: ops.pack(sh, ops.records(sh, sb, P, r)[0])) for r, sh in enumerate(shards)]
    inbox = {r: [] for r in range(P)}
    for r, sh in enumerate(shards):
        rec_v, counts = ops.records(sh, sb, P, r)
        lens, ids = ops.pack(sh, rec_v)
        lens_np = lens.cpu().numpy()
        s = i = 0
        for j in range(P):
            c = int(counts[j])
            k = int(lens_np[s: s + c].sum())
            if c:
                inbox[j].append((lens[s: s + c], ids[i: i + k]))
            s += c
            i += k
    recv = []
    for r, sh in enumerate(shards):
        rl = torch.cat([x[0] for x in inbox[r]]) if inbox[r] else torch.zeros(0, dtype=torch.int64, device="cuda")
        ri = torch.cat([x[1] for x in inbox[r]]) if inbox[r] else torch.zeros(0, dtype=torch.int32, device="cuda")
        recv.append(timed(lambda sh=sh, rl=rl, ri=ri: ops.count(sh, rl, ri)))
    surr = [s + c for s, c in zip(send, recv)]
    return surr


def direct_step(P):
    # direct pull (deduplicated requests, lowest-vertex partials via the
    # middle engine over the shard's cached pull index)
    for cname, ck in (("predsum", tcb.CostKind.PRED_SUM), ("succsum", tcb.CostKind.SUCC_SUM)):
        db = range_bounds(partition_ranges(g, ck, P))
        dsh = [D.shard_of(g, int(db[r]), int(db[r + 1])) for r in range(P)]
        asks = [ops.requests(sh, db, P, r) for r, sh in enumerate(dsh)]
        t_req = [timed(lambda sh=sh, r=r: ops.requests(sh, db, P, r)) for r, sh in enumerate(dsh)]
        serve = [0.0] * P
        fetched = []
        for i in range(P):
            ids_i, _, counts_i, _ = asks[i]
            parts = []
            a0 = 0
            for j in range(P):
                c = int(counts_i[j])
                if c:
                    q = ids_i[a0: a0 + c]
                    serve[j] += timed(lambda sh=dsh[j], q=q: ops.pack(sh, q))
                    parts.append(ops.pack(dsh[j], q))
                a0 += c
            fl = torch.cat([p_[0] for p_ in parts]) if parts else torch.zeros(0, dtype=torch.int64, device="cuda")
            fi = torch.cat([p_[1] for p_ in parts]) if parts else torch.zeros(0, dtype=torch.int32, device="cuda")
            fetched.append((fl, fi))
        cnt = [timed(lambda r=r: ops.count_direct(dsh[r], asks[r][0], *fetched[r])) for r in range(P)]
        tot = [t_req[r] + serve[r] + cnt[r] for r in range(P)]
        words = sum(int(f[1].numel()) for f in fetched)
        print(f"P={P}: direct-pull[{cname}] max {max(tot):.3f} ms (req {max(t_req):.3f}, serve {max(serve):.3f}, "
              f"count {max(cnt):.3f}; fetched {words / 1e6:.1f}M ids) -> eff {t1 / (P * max(tot)):.2f}")


t1 = timed(lambda: count_middle(g, out=out))
print(f"{a.config}: 1 GPU count {t1:.3f} ms (wall, incl. host overhead)", flush=True)
for P in [int(x) for x in a.ranks.split(",")]:
    sb = range_bounds(partition_ranges(g, tcb.CostKind.PRED_SUM, P))
    surr = surrogate_step(P, sb) if "surrogate" in MODES else [0.0]
    if "surrogate" in MODES:  # the same scheme on ranges balanced by the engine's own cost prefix
        ucost = (g._rev_cost[1:] - g._rev_cost[:-1]).contiguous()
        eb = balanced_bounds(ucost, 0, g.n, P).cpu().numpy()
        se = surrogate_step(P, eb)
        print(f"P={P}: surrogate[engine-cost ranges] max {max(se):.3f} ms (ranks {' '.join(f'{x:.2f}' for x in se)}) "
              f"-> eff {t1 / (P * max(se)):.2f}; [predsum ranges] ranks {' '.join(f'{x:.2f}' for x in surr)}", flush=True)
    if "direct" in MODES:
        direct_step(P)
    rep = [0.0]
    if "replicated" in MODES:
        ucost = (g._rev_cost[1:] - g._rev_cost[:-1]).contiguous()
        ub = balanced_bounds(ucost, 0, g.n, P).cpu().numpy()
        rep = [timed(lambda r=r: count_middle(g, int(ub[r]), int(ub[r + 1]), out=out)) for r in range(P)]
    # replicated, interleaved: rank r runs chunks c = r (mod P) of the plan cut for P GPUs
    if "replicated" not in MODES:
        continue
    tot = 0
    ilv = []
    for r in range(P):
        ilv.append(timed(lambda r=r: count_middle_part(g, r, P, out=out)))
        tot += int(out.item())
    ref = int(count_middle(g).item())
    assert tot == ref, (tot, ref)
    eff = lambda t: t1 / (P * max(t)) if max(t) else 0.0  # noqa: E731
    print(f"P={P}: surrogate max {max(surr):.3f} ms -> eff {eff(surr):.2f}; replicated[ranges] max {max(rep):.3f} ms "
          f"(ranks {' '.join(f'{x:.3f}' for x in rep)}) -> eff {eff(rep):.2f}; replicated[interleaved] max "
          f"{max(ilv):.3f} ms (ranks {' '.join(f'{x:.3f}' for x in ilv)}) -> eff {eff(ilv):.2f}", flush=True)
