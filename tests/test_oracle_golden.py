"""Pin the CPU oracle (oracle/) against vectors produced by the reference
itself (tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from conftest import SMALL, SMALL_NAMES
from oracle import gen_twin
from oracle import oracle as O


def _graph(case):
    n, e = O.normalize(case["raw"])
    return O.build_graph(n, e)


@pytest.mark.parametrize("name", SMALL_NAMES)
def test_normalize_matches_reference(name):
    case = SMALL[name]
    n, e = O.normalize(case["raw"])
    assert n == int(case["norm_n"][0])
    assert np.array_equal(e, case["norm_edges"].reshape(-1, 2))


@pytest.mark.parametrize("name", SMALL_NAMES)
def test_build_matches_reference(name):
    case = SMALL[name]
    g = _graph(case)
    for f in ("eff_indptr", "eff_indices", "full_indptr", "full_indices", "relabel",
              "orig_ids", "deg", "eff_deg"):
        assert np.array_equal(getattr(g, f), case[f]), f


@pytest.mark.parametrize("name", SMALL_NAMES)
def test_count_costs_partition_match_reference(name):
    case = SMALL[name]
    g = _graph(case)
    assert O.count_triangles(g) == int(case["T"][0])
    for kind in ("unit", "degree", "succsum", "predsum"):
        assert np.array_equal(O.node_costs(g, kind), case[f"cost_{kind}"]), kind
    if g.n == 0:
        return
    for P in (2, 3, 5, 8):
        for kind in ("predsum", "succsum", "degree"):
            b = O.balanced_bounds(O.node_costs(g, kind), 0, g.n, P)
            assert np.array_equal(b, case[f"bounds_{kind}_{P}"]), (kind, P)
        bounds = case[f"bounds_predsum_{P}"]
        partials, census = O.surrogate(g, bounds)
        assert np.array_equal(partials, case[f"surr_tri_{P}"])
        assert np.array_equal(census, case[f"surr_census_{P}"])
        dp, dreq, dwords = O.direct(g, bounds)
        assert np.array_equal(dp, case[f"direct_tri_{P}"])
        assert np.array_equal(dreq, case[f"direct_req_{P}"])
        assert np.array_equal(dreq.T, case[f"direct_census_{P}"])
        st = case[f"direct_stats_{P}"]
        assert np.array_equal(dreq.sum(1), st[:, 0]) and np.array_equal(dreq.sum(0), st[:, 1])
        assert np.array_equal(8 * (2 * dreq.sum(1) + dwords + (P - 1)), st[:, 2])
        low = [O.count_node_range(g.eff_indptr, g.eff_indices, bounds[i], bounds[i + 1])
               for i in range(P)]
        assert low == case[f"lowest_{P}"].tolist()
        plan = O.plan_tasks(O.node_costs(g, "degree"), P + 1)
        assert plan["split"] == int(case[f"plan_split_{P}"][0])
        assert np.array_equal(plan["initial_bounds"], case[f"plan_initial_{P}"])
        q = np.array(plan["queue"], np.int64).reshape(-1, 2)
        assert np.array_equal(q, case[f"plan_queue_{P}"].reshape(-1, 2))
        assert np.allclose(plan["targets"], case[f"plan_targets_{P}"])


@pytest.mark.parametrize("name", SMALL_NAMES)
def test_brute_agrees(name):
    case = SMALL[name]
    g = _graph(case)
    if g.n <= 400:
        assert O.count_triangles_brute(g.n, g.full_indptr, g.full_indices) == int(case["T"][0])


def test_known_answers(known):
    def comp(n):
        return O.build_graph(*O.normalize([(a, b) for a in range(n) for b in range(a + 1, n)]))

    assert O.count_triangles(comp(3)) == known["K3"]
    assert O.count_triangles(comp(4)) == known["K4"]
    assert O.count_triangles(comp(9)) == known["K9"]
    pa = O.build_graph(*O.normalize(O.pa_edge_list(10_000, 20, 1)))
    assert pa.m == known["PA_10000_20_1_m"]
    assert int(pa.deg.max()) == known["PA_10000_20_1_maxdeg"]
    assert O.count_triangles(pa) == known["PA_10000_20_1_T"]
    assert len(O.pa_edge_list(101, 2, 7)) == known["PA_101_2_7_m"]
    plan = O.plan_tasks(np.ones(100, np.int64), 5)
    assert plan["split"] == known["plan_unit_100_5"]["split"]
    ib = plan["initial_bounds"]
    assert list(np.diff(ib)) == known["plan_unit_100_5"]["initial"]
    assert [t for _, t in plan["queue"]] == known["plan_unit_100_5"]["queue"]
    for r in known["ranges"]:
        b = O.balanced_bounds(r["costs"], 0, len(r["costs"]), r["k"])
        assert [[int(b[i]), int(b[i + 1] - b[i])] for i in range(r["k"])] == r["out"]
    g = O.build_graph(*O.normalize([(0, 1), (0, 2), (1, 3)]))
    assert g.relabel.tolist() == known["tie_break_relabel"]


def test_pa_generator_matches_reference_fixture(small):
    for name in ("pa_500_8_11", "pa_1500_12_3", "pa_2000_10_3"):
        _, n, d, s = name.split("_")
        assert np.array_equal(O.pa_edge_list(int(n), int(d), int(s)), small[name]["raw"])


def test_cfg1_instance(configs):
    c = configs["cfg1_er_gnm_16384_131072_seed1"]
    raw = gen_twin.er_gnm(16384, 131072, 1)
    assert gen_twin.checksum(raw) == c["raw_checksum"]
    g = O.build_graph(*O.normalize(raw))
    assert (g.n, g.m) == (c["n"], c["m"])
    assert gen_twin.checksum(g.eff_indices) == c["eff_indices_checksum"]
    assert O.count_triangles(g) == c["T"]
    assert int(O.node_costs(g, "succsum").sum()) == c["W"]
    for P in (2, 4, 8):
        b = O.balanced_bounds(O.node_costs(g, "predsum"), 0, g.n, P)
        assert b.tolist() == c[f"bounds_predsum_{P}"]
        partials, census = O.surrogate(g, b)
        assert partials.tolist() == c[f"surr_tri_{P}"]
        assert census.tolist() == c[f"surr_census_{P}"]
        if f"direct_tri_{P}" in c:
            dp, dreq, dwords = O.direct(g, b)
            assert dp.tolist() == c[f"direct_tri_{P}"]
            assert dreq.tolist() == c[f"direct_req_{P}"]
            assert (8 * (2 * dreq.sum(1) + dwords + (P - 1))).tolist() == c[f"direct_bytes_{P}"]


def test_threaded_tasks_sum_to_total():
    g = O.build_graph(*O.normalize(O.pa_edge_list(3000, 12, 5)))
    plan = O.plan_tasks(O.node_costs(g, "degree"), 5)
    ib = plan["initial_bounds"]
    tv = list(ib[:-1]) + [v for v, _ in plan["queue"]]
    tt = list(np.diff(ib)) + [t for _, t in plan["queue"]]
    keep = [i for i in range(len(tv)) if tt[i] > 0]
    tv = [tv[i] for i in keep]
    tt = [tt[i] for i in keep]
    assert O.count_tasks_threaded(g.eff_indptr, g.eff_indices, tv, tt, 4) == O.count_triangles(g)


def test_partitioned_schemes_tiny_graphs_oracle(known):
    """The oracle's surrogate / direct restatements on tiny graphs with 1, 2
    and 5 ranks (more ranks than nodes) against the reference's outputs."""
    tiny = {"K3": [(a, b) for a in range(3) for b in range(a + 1, 3)],
            "K4": [(a, b) for a in range(4) for b in range(a + 1, 4)],
            "edge": [(0, 1)], "star": [(0, 1), (0, 2), (0, 3)], "empty": []}
    for name, pairs in tiny.items():
        raw = np.asarray(pairs, np.int64).reshape(-1, 2)
        g = O.build_graph(*O.normalize(raw))
        for P in (1, 2, 5):
            b = O.balanced_bounds(O.node_costs(g, "predsum"), 0, g.n, P) if g.n else np.zeros(P + 1, np.int64)
            sur = known["ranks_edge_cases"][f"{name}/{P}/count_space_surrogate"]
            partials, census = O.surrogate(g, b)
            assert partials.tolist() == sur["triangles"] and census.tolist() == sur["data_msgs_to"], (name, P)
            dire = known["ranks_edge_cases"][f"{name}/{P}/count_space_direct"]
            dp, dreq, dwords = O.direct(g, b)
            assert dp.tolist() == dire["triangles"] and dreq.tolist() == dire["requests_to"], (name, P)
            assert (8 * (2 * dreq.sum(1) + dwords + (P - 1))).tolist() == dire["bytes_sent"], (name, P)


def test_scale_goldens_reference_pin():
    """Where the reference itself was run at a full-size config
    (tests/golden/make_reference_scale.py adds a "reference" block to
    scale.json), its graph and count equal the oracle's numbers the GPU tests
    compare against."""
    import json
    import os

    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "scale.json")
    scale = json.load(open(path))
    pinned = [c for c in scale if "reference" in scale[c]]
    for c in pinned:
        ref = scale[c]["reference"]
        for k in ("n", "m", "T", "relabel_checksum", "eff_indptr_checksum", "eff_indices_checksum"):
            assert ref[k] == scale[c][k], (c, k)
