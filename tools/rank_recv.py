"""Per-rank cost of processing received lists in the sharded count (dev
tool): time of tc_shard_index, of planning, and of the engine run (tiers)."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1406_5687_b200 import _lib  # noqa: E402
from paper_1406_5687_b200 import sharded as S  # noqa: E402

raw = bench.host_raw_edges(sys.argv[1], pin=True).cuda()
P = int(sys.argv[2])
cost = sys.argv[3] if len(sys.argv) > 3 else "engine"
shards, _ = S.emulate_build(raw, P, cost=cost)
del raw
ops = S.ShardOps()
# every rank's messages, then each rank's received set as one batch
msgs = []
for r, sh in enumerate(shards):
    sd, sz = ops.send_sizes(sh, P, r)
    lens, ids = ops.send_pack(sh, P, r, sd, int(sz[0].sum()), int(sz[1].sum()))
    msgs.append((sz, lens, ids))


def sync_t():
    torch.cuda.synchronize()
    return time.perf_counter()


for r, sh in enumerate(shards):
    parts_l, parts_w = [], []
    for s in range(r):
        sz, lens, ids = msgs[s]
        lo_, wo_ = np.concatenate([[0], np.cumsum(sz[0])]), np.concatenate([[0], np.cumsum(sz[1])])
        parts_l.append(lens[int(lo_[r]): int(lo_[r + 1])])
        parts_w.append(ids[int(wo_[r]): int(wo_[r + 1])])
    if not parts_l:
        continue
    rl = torch.cat(parts_l)
    nw = sum(int(p.numel()) for p in parts_w)
    buf, pool = ops.recv_pool(nw)
    pool.copy_(torch.cat(parts_w))
    for rep in range(3):
        t0 = sync_t()
        plan = ops._plan(sh, rl, pool)
        t1 = sync_t()
        _lib.lib().tc_engine_timing(1, None, None, None)
        o = torch.empty(1, dtype=torch.int64, device="cuda")
        _lib.call("tc_plan_run", plan.handle, _lib.ptr(o), _lib.stream())
        t2 = sync_t()
        tot, nl = ctypes.c_double(), ctypes.c_longlong()
        tiers = (ctypes.c_double * 3)()
        _lib.lib().tc_engine_timing(0, ctypes.byref(tot), ctypes.byref(nl), tiers)
    print(f"rank {r}: received lists {rl.numel()} ids {nw / 1e6:.1f}M; index+plan {1e3 * (t1 - t0):.2f} ms, "
          f"run {1e3 * (t2 - t1):.2f} ms (engine {tot.value:.2f}: tiers {' '.join(f'{x:.2f}' for x in tiers)})",
          flush=True)
