"""Generate golden fixtures by running the REFERENCE implementation.

Run in the development container (where /root/reference exists):

    python tests/golden/make_golden.py            # small fixtures + cfg1
    python tests/golden/make_golden.py --big      # + cfg2 PA(1M, d=100, seed 1)

It imports /root/reference/pkg/src/tricount with a raising greenlet stub
(only backend="par" runs need the runtime) and writes:

    tests/golden/known.json        frozen known answers (counts, plans, ranges)
    tests/golden/small.npz         per-case reference outputs for small graphs
    tests/golden/configs.json      per-config totals / checksums (cfg1, cfg2)
    tests/golden/suites_*.csv      the reference bench suites' CSV output

The fixtures are consumed by tests/ on CPU (oracle pinning) and on the GPU
(parity).  Nothing at test time reads /root/reference.
"""

import argparse
import json
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

from oracle import gen_twin  # noqa: E402

REF_SRC = "/root/reference/pkg/src"


def import_reference():
    shim = tempfile.mkdtemp(prefix="greenlet_stub_")
    with open(os.path.join(shim, "greenlet.py"), "w") as f:
        f.write(
            "class GreenletExit(BaseException):\n    pass\n"
            "class greenlet:\n    def __init__(self, *a, **k):\n"
            "        raise RuntimeError('greenlet stub')\n"
            "def getcurrent():\n    raise RuntimeError('greenlet stub')\n"
        )
    os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp(prefix="numba_"))
    sys.path.insert(0, shim)
    sys.path.insert(0, REF_SRC)
    import tricount  # noqa: F401

    return tricount


def er_pairs(n, p, seed):
    """Same construction as the reference's test fixture generator (G(n,p) over
    triu pairs with np.random.default_rng(seed))."""
    rng = np.random.default_rng(seed)
    iu, iv = np.triu_indices(n, 1)
    mask = rng.random(len(iu)) < p
    return np.stack([iu[mask], iv[mask]], axis=1).astype(np.int64).reshape(-1, 2)


def small_cases(tc):
    cases = {}
    for (n, p, s) in [(25, 0.5, 3), (40, 0.3, 11), (60, 0.2, 21), (90, 0.25, 31),
                      (120, 0.2, 9), (200, 0.05, 7), (150, 0.5, 5), (300, 0.1, 12)]:
        cases[f"er_{n}_{p}_{s}"] = er_pairs(n, p, s)
    for (n, d, s) in [(500, 8, 11), (1500, 12, 3), (2000, 10, 3), (SCAN := 256 * 3 + 17, 6, 4)]:
        cases[f"pa_{n}_{d}_{s}"] = tc.generate_pa(tc.PaParams(n=n, d=d, seed=s)).edges
    # sparse labels, self-loops and duplicates: exercises first-seen compaction
    rng = np.random.default_rng(99)
    labels = rng.choice(10**7, size=400, replace=False)
    pairs = labels[rng.integers(0, 400, size=(3000, 2))]
    pairs[::37, 1] = pairs[::37, 0]                      # self-loops
    pairs = np.concatenate([pairs, pairs[::5][:, ::-1]])  # reversed duplicates
    cases["sparse_labels"] = pairs.astype(np.int64)
    # dense-but-shuffled labels with duplicates
    rng = np.random.default_rng(7)
    cases["dense_dups"] = rng.integers(0, 64, size=(900, 2)).astype(np.int64)
    cases["k9"] = np.array([(a, b) for a in range(9) for b in range(a + 1, 9)], np.int64)
    cases["star"] = np.array([(0, i) for i in range(1, 50)], np.int64)
    cases["path"] = np.array([(0, 1), (1, 2)], np.int64)
    cases["tie_break"] = np.array([(0, 1), (0, 2), (1, 3)], np.int64)
    cases["compact_first_seen"] = np.array([(5, 9), (9, 7)], np.int64)
    # small R-MAT (device generator's numpy twin) -> skewed degrees
    cases["rmat_s10"] = gen_twin.rmat(10, 8, 5).astype(np.int64)
    cases["gnm_2000_16000"] = gen_twin.er_gnm(2000, 16000, 3).astype(np.int64)
    return cases


def reference_outputs(tc, raw_edges):
    out = {}
    raw = tc.RawGraph.from_pairs(raw_edges) if len(raw_edges) else tc.RawGraph.from_pairs([])
    norm = tc.normalize(raw)
    g = tc.build_graph(norm)
    out["raw"] = np.asarray(raw_edges, np.int64).reshape(-1, 2)
    out["norm_n"] = np.array([norm.n])
    out["norm_edges"] = norm.edges
    for f in ("eff_indptr", "eff_indices", "full_indptr", "full_indices", "relabel",
              "orig_ids", "deg", "eff_deg"):
        out[f] = np.asarray(getattr(g, f))
    out["T"] = np.array([tc.count_triangles_seq(g)])
    for kind in tc.CostKind:
        out[f"cost_{kind.value}"] = tc.node_costs(g, kind)
    for P in (2, 3, 5, 8):
        for kind in (tc.CostKind.PRED_SUM, tc.CostKind.SUCC_SUM, tc.CostKind.DEGREE):
            bounds = tc.range_bounds(tc.partition_ranges(g, kind, P)) if g.n else np.zeros(P + 1, np.int64)
            out[f"bounds_{kind.value}_{P}"] = bounds
        if g.n:
            bounds = out[f"bounds_predsum_{P}"]
            total, rr = tc.count_space_surrogate(g, P, tc.CostKind.PRED_SUM, backend="par")
            assert total == out["T"][0]
            out[f"surr_tri_{P}"] = np.array([m.triangles for m in rr.metrics], np.int64)
            out[f"surr_census_{P}"] = np.stack([m.data_msgs_to for m in rr.metrics])
            out[f"surr_msgs_{P}"] = np.array([m.data_msgs_sent for m in rr.metrics], np.int64)
            out[f"surr_bytes_{P}"] = np.array([m.bytes_sent for m in rr.metrics], np.int64)
            out[f"surr_pbytes_{P}"] = np.array([m.partition_bytes for m in rr.metrics], np.int64)
            total_d, rd = tc.count_space_direct(g, P, tc.CostKind.PRED_SUM, backend="par")
            assert total_d == out["T"][0]
            out[f"direct_tri_{P}"] = np.array([m.triangles for m in rd.metrics], np.int64)
            out[f"direct_req_{P}"] = np.stack([m.requests_to for m in rd.metrics])
            out[f"direct_census_{P}"] = np.stack([m.data_msgs_to for m in rd.metrics])
            out[f"direct_stats_{P}"] = np.array(
                [[m.requests_sent, m.data_msgs_sent, m.bytes_sent, m.completion_msgs_sent, m.partition_bytes]
                 for m in rd.metrics], np.int64)
            out[f"lowest_{P}"] = np.array(
                [tc.count_task(g, tc.Task(int(bounds[i]), int(bounds[i + 1] - bounds[i])))
                 if bounds[i + 1] > bounds[i] else 0 for i in range(P)], np.int64)
            plan = tc.plan_tasks(tc.node_costs(g, tc.CostKind.DEGREE), P + 1)
            out[f"plan_split_{P}"] = np.array([plan.split])
            out[f"plan_initial_{P}"] = tc.range_bounds(plan.initial)
            out[f"plan_queue_{P}"] = np.array([(t.v, t.t) for t in plan.queue], np.int64).reshape(-1, 2)
            out[f"plan_targets_{P}"] = plan.targets
    return out


PARSE_INPUTS = [
    b"# c\n0 1\n\n1 2\n", b"0 1\n0 1\n", b"0 x\n", b"0 1\n1 2 3\n", b"0 -1\n", b"1_000 2\n",
    b"  7\t8  \r\n# x\n\n9 10", b"+3 -0\n", b"1__0 2\n", b"a b c\n0 1\n", b"\x1c1\x1d2\x1e\n",
    b"0 1\n#\n   \n2 3 # c\n", b"0 1\n\xff 2\n", b"x -1\n", b"-1 x\n", b"3 4\n-2 5\n", b"\n\n", b"5 5\n5 5",
    b"007 08\n", b"1 2\x0b\x0c\n3\t\t4\n", b"12 2147483647\n",
]


def parse_cases(tc):
    """The reference's load_edge_list on edge cases and on a larger random
    file: expected edges, or (lineno, message) of the EdgeListParseError."""
    cases = list(PARSE_INPUTS)
    rng = np.random.default_rng(11)
    lines = []
    for i in range(3000):
        r = rng.random()
        if r < 0.05:
            lines.append(b"# comment %d" % i)
        elif r < 0.08:
            lines.append(b"   ")
        else:
            u, v = rng.integers(0, 10**6, size=2)
            sep = [b" ", b"\t", b"  "][i % 3]
            lines.append(b"%d%s%d" % (u, sep, v))
    cases.append(b"\n".join(lines) + b"\n")
    out = []
    for data in cases:
        rec = {"input": data.decode("latin-1")}
        try:
            raw = tc.load_edge_list(data)
            rec["n"] = int(raw.n)
            if len(raw.edges) > 50:
                rec["m"] = int(len(raw.edges))
                rec["edges_checksum"] = gen_twin.checksum(raw.edges)
            else:
                rec["edges"] = raw.edges.tolist()
        except tc.EdgeListParseError as e:
            rec["lineno"] = e.lineno
            rec["message"] = str(e)
        out.append(rec)
    return out


def known_answers(tc):
    def gp(pairs, n=None):
        return tc.build_graph(tc.normalize(tc.RawGraph.from_pairs(pairs, n=n)))

    def complete(n):
        return gp([(a, b) for a in range(n) for b in range(a + 1, n)])

    k = {}
    k["K3"] = tc.count_triangles_seq(complete(3))
    k["K4"] = tc.count_triangles_seq(complete(4))
    k["K9"] = tc.count_triangles_seq(complete(9))
    k["path"] = tc.count_triangles_seq(gp([(0, 1), (1, 2)]))
    g25 = tc.build_graph(tc.normalize(tc.RawGraph.from_pairs(er_pairs(25, 0.5, 3))))
    g40 = tc.build_graph(tc.normalize(tc.RawGraph.from_pairs(er_pairs(40, 0.3, 11))))
    k["ER_25_0.5_3"] = tc.count_triangles_brute(g25)
    k["ER_40_0.3_11"] = tc.count_triangles_brute(g40)
    assert tc.count_triangles_seq(g25) == k["ER_25_0.5_3"]
    pa = tc.build_graph(tc.normalize(tc.generate_pa(tc.PaParams(n=10_000, d=20, seed=1))))
    k["PA_10000_20_1_m"] = int(pa.m)
    k["PA_10000_20_1_maxdeg"] = int(pa.deg.max())
    k["PA_10000_20_1_T"] = tc.count_triangles_seq(pa)
    k["PA_101_2_7_m"] = len(tc.generate_pa(tc.PaParams(n=101, d=2, seed=7)).edges)
    plan = tc.plan_tasks(np.ones(100, dtype=np.int64), 5)
    k["plan_unit_100_5"] = dict(split=plan.split, initial=[r.count for r in plan.initial],
                                queue=[t.t for t in plan.queue])
    plan = tc.plan_tasks(np.ones(4, dtype=np.int64), 2)
    k["plan_unit_4_2"] = dict(split=plan.split, initial=[(r.start, r.count) for r in plan.initial],
                              queue=[(t.v, t.t) for t in plan.queue])
    k3 = complete(3)
    k["costs_K3"] = {kind.value: tc.node_costs(k3, kind).tolist() for kind in tc.CostKind}
    k["ranges"] = [
        dict(costs=c, k=kk, out=[(r.start, r.count) for r in tc.balanced_ranges(c, tc.NodeRange(0, len(c)), kk)])
        for c, kk in [([1] * 10, 2), ([9, 1, 1, 1], 2), ([3, 3], 1), ([1, 1], 5), ([0, 0, 0, 0], 2)]
    ]
    k["tie_break_relabel"] = gp([(0, 1), (0, 2), (1, 3)]).relabel.tolist()
    k["star_relabel0"] = int(gp([(0, 1), (0, 2), (0, 3)]).relabel[0])
    k["k3_succ"] = [list(map(int, complete(3).succ(v))) for v in range(3)]
    k["dedup_send_targets"] = [
        tc.dedup_send_targets(np.array([3, 4, 9]), np.array([0, 5, 10])),
        tc.dedup_send_targets(np.array([3, 4, 9]), np.array([0, 5, 10]), self_rank=0),
    ]
    k["parse"] = parse_cases(tc)
    # the partitioned schemes on tiny graphs, including more ranks than nodes
    edge = {}
    tiny = {"K3": complete(3), "K4": complete(4), "edge": gp([(0, 1)]), "star": gp([(0, 1), (0, 2), (0, 3)]),
            "empty": gp([])}
    for name, g in tiny.items():
        for P in (1, 2, 5):
            for fn in ("count_space_surrogate", "count_space_direct"):
                tot, rr = getattr(tc, fn)(g, P, backend="par")
                edge[f"{name}/{P}/{fn}"] = dict(
                    total=int(tot), triangles=[int(m.triangles) for m in rr.metrics],
                    bytes_sent=[int(m.bytes_sent) for m in rr.metrics],
                    data_msgs_to=[m.data_msgs_to.tolist() for m in rr.metrics],
                    requests_to=[m.requests_to.tolist() for m in rr.metrics],
                    partition_bytes=[int(m.partition_bytes) for m in rr.metrics])
            try:
                tot, rr = tc.count_dynamic(g, P, backend="par")
                edge[f"{name}/{P}/count_dynamic"] = dict(total=int(tot), nmetrics=len(rr.metrics))
            except ValueError as e:
                edge[f"{name}/{P}/count_dynamic"] = dict(error="ValueError", msg=str(e))
    k["ranks_edge_cases"] = edge
    k["surrogate_count_k3"] = [
        tc.surrogate_count([], tc.NodeRange(0, 3), k3),
        tc.surrogate_count(k3.succ(0), tc.NodeRange(2, 1), k3),
        tc.surrogate_count(k3.succ(0), tc.NodeRange(1, 1), k3),
    ]
    return k


def config_summary(tc, raw_edges, with_partials=True, with_direct=False):
    norm = tc.normalize(tc.RawGraph.from_pairs(raw_edges))
    g = tc.build_graph(norm)
    succ = tc.node_costs(g, tc.CostKind.SUCC_SUM)
    out = dict(n=int(g.n), m=int(g.m), T=int(tc.count_triangles_seq(g)), W=int(succ.sum()),
               raw_checksum=gen_twin.checksum(raw_edges),
               eff_indptr_checksum=gen_twin.checksum(g.eff_indptr),
               eff_indices_checksum=gen_twin.checksum(g.eff_indices),
               relabel_checksum=gen_twin.checksum(g.relabel),
               max_deg=int(g.deg.max()), max_eff_deg=int(g.eff_deg.max()))
    if with_partials:
        for P in (2, 4, 8):
            bounds = tc.range_bounds(tc.partition_ranges(g, tc.CostKind.PRED_SUM, P))
            total, rr = tc.count_space_surrogate(g, P, tc.CostKind.PRED_SUM, backend="par")
            assert total == out["T"]
            out[f"bounds_predsum_{P}"] = bounds.tolist()
            out[f"surr_tri_{P}"] = [int(m.triangles) for m in rr.metrics]
            out[f"surr_census_{P}"] = np.stack([m.data_msgs_to for m in rr.metrics]).tolist()
            out[f"lowest_{P}"] = [int(tc.count_task(g, tc.Task(int(bounds[i]), int(bounds[i + 1] - bounds[i]))))
                                  for i in range(P)]
            if with_direct:
                total_d, rd = tc.count_space_direct(g, P, tc.CostKind.PRED_SUM, backend="par")
                assert total_d == out["T"]
                out[f"direct_tri_{P}"] = [int(m.triangles) for m in rd.metrics]
                out[f"direct_req_{P}"] = np.stack([m.requests_to for m in rd.metrics]).tolist()
                out[f"direct_bytes_{P}"] = [int(m.bytes_sent) for m in rd.metrics]
    return out


def suite_csvs(tc):
    """CSV output of the reference's bench suites (bench.py:79-145) through
    its metrics writers (metrics.py:105-119), backend "par"."""
    import io
    from tricount import bench as tb
    from tricount import metrics as tm

    g = tb.pa_graph(2000, 10, 3)
    label = tb.pa_label(2000, 10, 3)
    pred, deg = tc.CostKind.PRED_SUM, tc.CostKind.DEGREE
    recs = tb.bench_strong(g, label, "space-surrogate", [2, 4], pred, "par", 0)
    recs += tb.bench_strong(g, label, "space-direct", [2, 3], pred, "par", 0)
    recs += tb.bench_weak(400, 8, "space-surrogate", [1, 2, 3], pred, "par", 1)
    recs += tb.bench_idle(g, label, 4, deg, 2, "par", 5)
    recs.append(tb._record("space-surrogate", g, label, 0, pred, "par", 0, "count"))  # error row
    run = io.StringIO()
    tm.write_run_csv(recs, run)
    mem = io.StringIO()
    tm.write_memory_csv(tb.bench_memory(1500, [4, 8, 12], 4, pred, 2), mem)
    return run.getvalue(), mem.getvalue()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true")
    args = ap.parse_args()
    tc = import_reference()

    known = known_answers(tc)
    with open(os.path.join(HERE, "known.json"), "w") as f:
        json.dump(known, f, indent=1, default=int)

    arrays = {}
    for name, raw in small_cases(tc).items():
        for key, val in reference_outputs(tc, raw).items():
            arrays[f"{name}/{key}"] = val
    np.savez_compressed(os.path.join(HERE, "small.npz"), **arrays)

    run_csv, mem_csv = suite_csvs(tc)
    with open(os.path.join(HERE, "suites_run.csv"), "w") as f:
        f.write(run_csv)
    with open(os.path.join(HERE, "suites_memory.csv"), "w") as f:
        f.write(mem_csv)

    cfg_path = os.path.join(HERE, "configs.json")
    configs = json.load(open(cfg_path)) if os.path.exists(cfg_path) else {}
    raw1 = gen_twin.er_gnm(16384, 131072, 1).astype(np.int64)
    configs["cfg1_er_gnm_16384_131072_seed1"] = config_summary(tc, raw1, with_direct=True)
    if args.big:
        raw2 = tc.generate_pa(tc.PaParams(1_000_000, 100, seed=1)).edges
        configs["cfg2_pa_1000000_100_seed1"] = config_summary(tc, raw2)
    with open(cfg_path, "w") as f:
        json.dump(configs, f, indent=1)
    print("wrote", sorted(os.listdir(HERE)))


if __name__ == "__main__":
    main()
