"""Quick device timing of the count engines on one or more configs (dev loop)."""
import argparse
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1406_5687_b200 as tcb  # noqa: E402
from paper_1406_5687_b200 import _lib  # noqa: E402
from paper_1406_5687_b200.sequential import count_lowest, count_middle  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="cfg2")
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--lowest", action="store_true")
ap.add_argument("--no-tiled", action="store_true")
ap.add_argument("--merge", action="store_true", help="also time the warp-per-edge merge-path comparator")
ap.add_argument("--caps", default="", help="small,mid,block tier caps (tc_set_tuning), e.g. 128,256,4096")
a = ap.parse_args()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
if a.caps:
    c = [int(x) for x in a.caps.split(",")]
    for key, val in ((0, c[0]), (2, c[1]), (1, c[2])):
        _lib.call("tc_set_tuning", key, val)
for cfg in a.configs.split(","):
    t0 = time.perf_counter()
    raw = bench.host_raw_edges(cfg, pin=True)
    tg = time.perf_counter() - t0
    dev_raw = raw.cuda()
    torch.cuda.synchronize()
    for _ in range(2):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        g = tcb.build_graph(tcb.normalize(tcb.RawGraph(n=0, edges=dev_raw)))
        e.record()
        torch.cuda.synchronize()
    build_ms = s.elapsed_time(e)
    engines = [("middle", lambda: count_middle(g, tiled=False))]
    engines += [] if a.no_tiled else [("tiled", lambda: count_middle(g, tiled=True))]
    engines += [("lowest", lambda: count_lowest(g))] if a.lowest else []
    if a.merge:
        from paper_1406_5687_b200.sequential import count_merge_path
        T0 = int(count_middle(g, tiled=False).item())
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        assert int(count_merge_path(g).item()) == T0
        flush.fill_(1)
        ev[0].record()
        count_merge_path(g)
        ev[1].record()
        torch.cuda.synchronize()
        print(f"{cfg} merge-path: T={T0} {ev[0].elapsed_time(ev[1]):.3f} ms -> {g.m / ev[0].elapsed_time(ev[1]) / 1e6:.2f} G edges/s",
              flush=True)
    from paper_1406_5687_b200.graph import tiled_index
    import paper_1406_5687_b200.graph as G
    if G.TILE_IDS == 0:
        G.TILE_IDS = 8 << 20
    if not a.no_tiled:
        ti = tiled_index(g, 0, g.n)
        print(f"{cfg}: tiles={ti.ntiles} virtual owners={ti.k}", flush=True)
    for name, fn in engines:
        T = int(fn().item())
        _lib.lib().tc_engine_timing(1, None, None, None)
        for _ in range(a.reps):
            flush.fill_(1)
            fn()
        torch.cuda.synchronize()
        tot, nl = ctypes.c_double(), ctypes.c_longlong()
        tiers = (ctypes.c_double * 3)()
        _lib.lib().tc_engine_timing(0, ctypes.byref(tot), ctypes.byref(nl), tiers)
        ms = tot.value / nl.value
        print(f"{cfg} {name}: n={g.n} m={g.m} T={T} engine {ms:.3f} ms  -> {g.m / ms / 1e6:.2f} G edges/s; "
              f"build {build_ms:.1f} ms; gen {tg:.1f}s; tiers ms " + " / ".join(f"{x / nl.value:.2f}" for x in tiers), flush=True)
    del g, dev_raw
    torch.cuda.empty_cache()
