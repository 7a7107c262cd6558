"""Per-phase device time of the e2e path (dev tool): H2D, normalize, build, count."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1406_5687_b200 as tcb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
raw = bench.host_raw_edges(a.config, pin=True)
dev = torch.device("cuda")
tot = {"h2d": 0.0, "normalize": 0.0, "build": 0.0, "count": 0.0}
for i in range(a.reps + 2):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    ev[0].record()
    d = raw.to(dev, non_blocking=True)
    ev[1].record()
    norm = tcb.normalize(tcb.RawGraph(n=0, edges=d))
    ev[2].record()
    g = tcb.build_graph(norm)
    ev[3].record()
    T = tcb.count_triangles_seq(g)
    ev[4].record()
    torch.cuda.synchronize()
    if i >= 2:
        for k, name in enumerate(tot):
            tot[name] += ev[k].elapsed_time(ev[k + 1])
    del d, norm, g
print(a.config, {k: round(v / a.reps, 3) for k, v in tot.items()}, "total", round(sum(tot.values()) / a.reps, 3), "ms")
