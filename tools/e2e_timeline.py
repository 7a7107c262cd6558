"""Device timeline of one e2e step (dev tool): every kernel / copy with its
stream, start and end relative to the step start, plus the API phases
(normalize / build_graph / count) as host ranges, and the idle gaps of the
compute stream after the H2D copy ends.  torch.profiler (CUPTI)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile, record_function  # noqa: E402

import bench  # noqa: E402
import paper_1406_5687_b200 as tcb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--gap-us", type=float, default=5.0)
a = ap.parse_args()
raw = bench.host_raw_edges(a.config, pin=True)


def step():
    with record_function("api:normalize"):
        nr = tcb.normalize(tcb.RawGraph(n=0, edges=raw))
    with record_function("api:build_graph"):
        g = tcb.build_graph(nr)
    with record_function("api:count"):
        return tcb.count_triangles_seq(g)


for _ in range(3):
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    step()
    torch.cuda.synchronize()

ev = []
for e in prof.profiler.kineto_results.events():
    ev.append((e.start_ns(), e.start_ns() + e.duration_ns(), e.device_type(), e.device_resource_id(), e.name()))
dev = [x for x in ev if x[2] == torch.autograd.DeviceType.CUDA]
host = [x for x in ev if x[4].startswith("api:")]
t0 = min(x[0] for x in dev + host)
print(f"{a.config}: step span {(max(x[1] for x in dev) - t0) / 1e3:.1f} us")
for s, e, _, _, name in sorted(host):
    print(f"HOST {(s - t0) / 1e3:9.1f} .. {(e - t0) / 1e3:9.1f} us  {name}")
for s, e, _, sid, name in sorted(dev):
    print(f"s{sid:<3} {(s - t0) / 1e3:9.1f} .. {(e - t0) / 1e3:9.1f} us {(e - s) / 1e3:8.1f}  {name[:100]}")
# idle gaps across all streams (no device activity at all)
busy = sorted((s, e) for s, e, *_ in dev)
cur = busy[0][1]
gaps = []
for s, e in busy[1:]:
    if s > cur + a.gap_us * 1e3:
        gaps.append((cur, s))
    cur = max(cur, e)
print(f"device idle gaps > {a.gap_us} us: {len(gaps)}, total {sum(e - s for s, e in gaps) / 1e3:.1f} us")
for s, e in gaps:
    print(f"  idle {(s - t0) / 1e3:9.1f} .. {(e - t0) / 1e3:9.1f} us ({(e - s) / 1e3:.1f})")
