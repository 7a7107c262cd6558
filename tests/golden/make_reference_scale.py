"""Pin a full-size config to the REFERENCE itself (run in the development
container, where /root/reference exists; CPU only, tens of minutes):

    python tests/golden/make_reference_scale.py cfg5

The raw pairs come from the bit-identical numpy twin of the device generator
(oracle/gen_twin.py; its checksum must equal scale.json's raw_checksum, which
the GPU box computed from the device stream), the graph and the count from
the reference's own normalize / build_graph / count_triangles_seq.  Adds a
"reference" block to tests/golden/scale.json next to the oracle's numbers;
tests/test_oracle_golden.py asserts that the two agree."""

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, HERE)

from make_golden import import_reference  # noqa: E402
from oracle import gen_twin  # noqa: E402

CFG = {"cfg5": lambda: gen_twin.er_gnm(2_000_000, 400_000_000, 1)}


def main():
    tc = import_reference()
    path = os.path.join(HERE, "scale.json")
    out = json.load(open(path))
    for cfg in sys.argv[1:]:
        t0 = time.time()
        raw = CFG[cfg]().astype(np.int64)
        ck = gen_twin.checksum(raw)
        assert ck == out[cfg]["raw_checksum"], (ck, out[cfg]["raw_checksum"])
        print(cfg, "raw pairs", raw.shape[0], "checksum ok", round(time.time() - t0, 1), "s", flush=True)
        norm = tc.normalize(tc.RawGraph(n=0, edges=raw))
        del raw
        print(cfg, "normalize", round(time.time() - t0, 1), "s", flush=True)
        g = tc.build_graph(norm)
        del norm
        t1 = time.time()
        print(cfg, "build_graph", round(t1 - t0, 1), "s", flush=True)
        T = int(tc.count_triangles_seq(g))
        t2 = time.time()
        rec = {"n": int(g.n), "m": int(g.m), "T": T,
               "relabel_checksum": gen_twin.checksum(np.asarray(g.relabel)),
               "eff_indptr_checksum": gen_twin.checksum(np.asarray(g.eff_indptr)),
               "eff_indices_checksum": gen_twin.checksum(np.asarray(g.eff_indices)),
               "build_s": round(t1 - t0, 1), "count_s": round(t2 - t1, 1),
               "how": "reference normalize + build_graph + count_triangles_seq on gen_twin pairs "
                      "(tests/golden/make_reference_scale.py)"}
        print(cfg, rec, flush=True)
        out = json.load(open(path))
        out[cfg]["reference"] = rec
        with open(path, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
