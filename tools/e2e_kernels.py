"""Per-kernel device time of the e2e path via torch.profiler/CUPTI (dev tool)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
import paper_1406_5687_b200 as tcb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
raw = bench.host_raw_edges(a.config, pin=True)
dev = torch.device("cuda")


def step():
    g = tcb.build_graph(tcb.normalize(tcb.RawGraph(n=0, edges=raw)))
    return tcb.count_triangles_seq(g)


for _ in range(2):
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(a.reps):
        step()
    torch.cuda.synchronize()
rows = {}
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        k = e.name[:90]
        t, c = rows.get(k, (0.0, 0))
        rows[k] = (t + e.device_time / 1000.0, c + 1)
tot = sum(t for t, _ in rows.values())
print(f"{a.config}: total device time per step {tot / a.reps:.3f} ms")
for k, (t, c) in sorted(rows.items(), key=lambda kv: -kv[1][0])[:40]:
    print(f"  {t / a.reps:8.3f} ms  x{c // a.reps:3d}  {k}")
