"""Per-kernel device time of the sharded build, summed over the emulated ranks (torch.profiler; dev tool)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
from paper_1406_5687_b200 import sharded as S  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg4")
ap.add_argument("--ranks", type=int, default=8)
ap.add_argument("--cost", default="engine")
a = ap.parse_args()
raw = bench.host_raw_edges(a.config, pin=True).cuda()
S.emulate_build(raw, a.ranks, cost=a.cost)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    shards, ms = S.emulate_build(raw, a.ranks, cost=a.cost, timed=True)
    torch.cuda.synchronize()
rows = {}
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        k = e.name[:110]
        t, c = rows.get(k, (0.0, 0))
        rows[k] = (t + e.device_time / 1000.0, c + 1)
tot = sum(t for t, _ in rows.values())
print(f"{a.config} P={a.ranks} cost={a.cost}: build ranks ms {' '.join(f'{x:.0f}' for x in ms)}; total device time (all ranks) {tot:.1f} ms")
for k, (t, c) in sorted(rows.items(), key=lambda kv: -kv[1][0])[:30]:
    print(f"  {t:8.2f} ms  x{c:4d}  {k}")
