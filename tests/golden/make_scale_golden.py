"""Full-scale golden totals for configs 3-5 (run on a GPU box: the edges come
from the device generators, the answers from the CPU oracle -- itself pinned
to the reference by tests/test_oracle_golden.py -- on all host cores).

    python tests/golden/make_scale_golden.py cfg3 cfg5 cfg4

Writes/updates tests/golden/scale.json: n, m, T, W and order-sensitive
checksums of the raw pairs and of the oracle's relabel / eff_indptr /
eff_indices, so the GPU build and count can be compared bit-exactly at full
size (tests/test_gpu_parity.py::test_full_scale_configs)."""

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

import bench  # noqa: E402
from oracle import gen_twin  # noqa: E402
from oracle import oracle as O  # noqa: E402


def main():
    path = os.environ.get("SCALE_OUT", os.path.join(HERE, "scale.json"))
    out = json.load(open(path)) if os.path.exists(path) else {}
    threads = len(os.sched_getaffinity(0))
    for cfg in sys.argv[1:]:
        t0 = time.time()
        raw = bench.host_raw_edges(cfg, pin=False).numpy()
        rec = {"desc": bench.CONFIGS[cfg]["desc"], "raw_pairs": int(raw.shape[0]),
               "raw_checksum": gen_twin.checksum(raw)}
        n, e = O.normalize(raw.astype(np.int64))
        del raw
        g = O.build_graph(n, e, full=False)
        del e
        t1 = time.time()
        W = int(O.node_costs(g, "succsum").sum())
        plan = O.plan_tasks(O.node_costs(g, "succsum"), 4 * threads + 1)
        ib = plan["initial_bounds"]
        tv = [int(x) for x in ib[:-1]] + [v for v, _ in plan["queue"]]
        tt = [int(x) for x in np.diff(ib)] + [t for _, t in plan["queue"]]
        keep = [i for i in range(len(tv)) if tt[i] > 0]
        T = O.count_tasks_threaded(g.eff_indptr, g.eff_indices, [tv[i] for i in keep], [tt[i] for i in keep], threads)
        t2 = time.time()
        rec.update(n=int(g.n), m=int(g.m), T=int(T), W=W, max_deg=int(g.deg.max()), max_eff_deg=int(g.eff_deg.max()),
                   relabel_checksum=gen_twin.checksum(g.relabel), eff_indptr_checksum=gen_twin.checksum(g.eff_indptr),
                   eff_indices_checksum=gen_twin.checksum(g.eff_indices), oracle_build_s=round(t1 - t0, 1),
                   oracle_count_s=round(t2 - t1, 1), oracle_threads=threads)
        out[cfg] = rec
        print(cfg, rec, flush=True)
        with open(path, "w") as f:
            json.dump(out, f, indent=1)
        del g


if __name__ == "__main__":
    main()
