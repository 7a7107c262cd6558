"""Short profiling target: build one config, run the count a few times."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1406_5687_b200 as tcb  # noqa: E402
from paper_1406_5687_b200.sequential import count_lowest  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--engine", default="middle", choices=["middle", "lowest"])
a = ap.parse_args()
raw = bench.host_raw_edges(a.config, pin=True)
g = tcb.build_graph(tcb.normalize(tcb.RawGraph(n=0, edges=raw)))
for _ in range(a.reps):
    t = tcb.count_triangles_seq(g) if a.engine == "middle" else int(count_lowest(g).item())
torch.cuda.synchronize()
print("triangles", t, "n", g.n, "m", g.m)
