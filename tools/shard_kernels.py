"""Per-kernel device time of the sharded count, summed over the emulated ranks
(torch.profiler/CUPTI; dev tool)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
from paper_1406_5687_b200 import sharded as S  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg5")
ap.add_argument("--ranks", type=int, default=8)
ap.add_argument("--cost", default="engine")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--rebalance", type=int, default=0)
a = ap.parse_args()
raw = bench.host_raw_edges(a.config, pin=True).cuda()
shards, _ = S.emulate_build(raw, a.ranks, cost=a.cost)
del raw
for _ in range(2):
    S.emulate_count(shards)
for it in range(a.rebalance):
    busy = [0.0] * a.ranks
    S.emulate_count(shards, busy=busy)
    print(f"refinement {it}: own kernels ms {' '.join(f'{x:.2f}' for x in busy)}; bounds {shards[0].bounds.tolist()}")
    shards = S.emulate_rebalance(shards, busy)
    S.emulate_count(shards)
busy = [0.0] * a.ranks
S.emulate_count(shards, busy=busy)
print(f"profiled partition: own kernels ms {' '.join(f'{x:.2f}' for x in busy)}; bounds {shards[0].bounds.tolist()}")
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(a.reps):
        S.emulate_count(shards)
    torch.cuda.synchronize()
rows = {}
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        k = e.name[:110]
        t, c = rows.get(k, (0.0, 0))
        rows[k] = (t + e.device_time / 1000.0, c + 1)
tot = sum(t for t, _ in rows.values())
print(f"{a.config} P={a.ranks} cost={a.cost}: total device time per count (all ranks) {tot / a.reps:.3f} ms")
for k, (t, c) in sorted(rows.items(), key=lambda kv: -kv[1][0])[:45]:
    print(f"  {t / a.reps:8.3f} ms  x{c // a.reps:4d}  {k}")
