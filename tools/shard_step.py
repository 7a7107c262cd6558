"""Per-rank device time of the sharded pipeline (sharded.py), emulated on one
GPU: every rank's build and count steps run in lockstep with the collectives
replaced by buffer passing (transfer time excluded; in the N-GPU run the
exchange overlaps the local engine).  Efficiency = 1-GPU engine / (P x max
rank count time)."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1406_5687_b200 as tcb  # noqa: E402
from paper_1406_5687_b200 import sharded as S  # noqa: E402
from paper_1406_5687_b200.sequential import count_middle  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg5")
ap.add_argument("--ranks", default="2,4,8")
ap.add_argument("--costs", default="predsum,engine")
ap.add_argument("--round-words", type=int, default=1 << 28)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--rebalance", type=int, default=2, help="measured refinements of the partition after the first count")
ap.add_argument("--no-prof", action="store_true")
a = ap.parse_args()
raw = bench.host_raw_edges(a.config, pin=True)
g = tcb.build_graph(tcb.normalize(tcb.RawGraph(n=0, edges=raw)))
out = torch.empty(1, dtype=torch.int64, device="cuda")
T = int(count_middle(g, out=out).item())
from bench import _engine_ms  # noqa: E402
flush = torch.empty(1 << 28, dtype=torch.uint8, device="cuda")
t1, _ = _engine_ms(lambda: count_middle(g, out=out), 5, flush)
gbytes = sum(int(t.numel()) * t.element_size() for t in (g.eff_indptr, g.eff_indices, g._rev_indptr, g._rev_seg,
                                                          g._rev_cost, g._pool_indptr, g._pool))
print(f"{a.config}: n={g.n} m={g.m} T={T}; 1 GPU engine {t1:.3f} ms; 1-GPU graph {gbytes / 2**20:.0f} MiB", flush=True)
del g
torch.cuda.empty_cache()
dev_raw = raw.cuda()
for cost in a.costs.split(","):
    for P in [int(x) for x in a.ranks.split(",")]:
        t0 = time.perf_counter()
        shards, bms = S.emulate_build(dev_raw, P, cost=cost, timed=True)
        tb = time.perf_counter() - t0
        rops = [S.ShardOps() for _ in range(P)]  # one per emulated rank, kept across counts (streams, allocator pools)
        for it in range(a.rebalance + 1):
            best, bbusy = None, None
            for _ in range(a.reps):
                busy = [0.0] * P
                tot, mets, ms = S.emulate_count(shards, ops=rops, round_words=a.round_words, timed=True, busy=busy)
                assert tot == T, (tot, T)
                best = ms if best is None else [min(x, y) for x, y in zip(best, ms)]  # per-rank minimum
                bbusy = busy if bbusy is None else [min(x, y) for x, y in zip(bbusy, busy)]
            res = [sh.resident_bytes() / 2**20 for sh in shards]
            tag = f"cost={cost}" + (f" +{it} measured refinement(s)" if it else "")
            print(f"{a.config} P={P} {tag}: count ranks ms {' '.join(f'{x:.2f}' for x in best)} max {max(best):.2f} "
                  f"(sum {sum(best):.1f}) -> eff {t1 / (P * max(best)):.2f}; own kernels ms "
                  f"{' '.join(f'{x:.2f}' for x in bbusy)} max {max(bbusy):.2f} -> eff {t1 / (P * max(bbusy)):.2f}; "
                  f"build ranks ms max {max(bms):.1f} (wall {tb:.1f}s); "
                  f"resident MiB max {max(res):.0f}; bounds {shards[0].bounds.tolist()}", flush=True)
            labels = [dict() for _ in range(P)]
            S.emulate_count(shards, ops=rops, round_words=a.round_words, timed=True, busy=[0.0] * P, labels=labels)
            print("      split " + " | ".join(" ".join(f"{k[0]}{v:.1f}" for k, v in sorted(lb.items())) for lb in labels), flush=True)
            if it < a.rebalance:
                shards = S.emulate_rebalance(shards, bbusy)
        if not a.no_prof:
            profs = [dict() for _ in range(P)]
            S.emulate_count(shards, round_words=a.round_words, profs=profs)
            for r, pr in enumerate(profs):
                print(f"   rank {r}: " + " ".join(f"{k} {v:.2f}" for k, v in pr.items() if k != "start"), flush=True)
        del shards
        torch.cuda.empty_cache()
