"""CPU-only checks: the C-ABI library loads and exports every symbol the
header declares, host-side generators and logic match the reference
fixtures, and the product refuses to run without a GPU (no CPU fallback)."""

import os
import re

import numpy as np
import pytest
import torch

from conftest import REPO, SMALL
import paper_1406_5687_b200 as tcb
from paper_1406_5687_b200 import _lib
from paper_1406_5687_b200.graph_io import pa_edges_host
from oracle import gen_twin


def header_symbols():
    src = open(os.path.join(REPO, "include", "tcb200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:const char\*|unsigned long long|int64_t|int)\s+(tc_\w+)\(", src, re.M)))


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_lib.EXPORTED)
    assert L.tc_abi_version() == 1


def test_pa_host_generator_matches_reference(small):
    for name in ("pa_500_8_11", "pa_1500_12_3", "pa_2000_10_3", "pa_785_6_4"):
        _, n, d, s = name.split("_")
        e = pa_edges_host(tcb.PaParams(int(n), int(d), int(s))).numpy().astype(np.int64)
        assert np.array_equal(e, small[name]["raw"]), name


def test_pa_param_validation():
    with pytest.raises(ValueError):
        tcb.PaParams(n=10, d=3)
    with pytest.raises(ValueError):
        tcb.PaParams(n=4, d=4)


def test_twin_generators_are_deterministic():
    a = gen_twin.er_gnm(1000, 5000, 7)
    assert np.array_equal(a, gen_twin.er_gnm(1000, 5000, 7))
    assert not np.array_equal(a, gen_twin.er_gnm(1000, 5000, 8))
    assert a.min() >= 0 and a.max() < 1000
    r = gen_twin.rmat(8, 4, 1)
    assert r.shape == (1024, 2) and r.max() < 256


def test_api_surface_mirrors_reference_hot_path():
    names = ["RawGraph", "Graph", "normalize", "build_graph", "count_triangles_seq", "intersect_count",
             "count_triangles_brute", "CostKind", "NodeRange", "node_costs", "balanced_ranges",
             "range_bounds", "owner_of", "partition_ranges", "Task", "TaskPlan", "plan_tasks",
             "count_task", "count_space_surrogate", "count_dynamic", "dedup_send_targets",
             "surrogate_count", "PaParams", "generate_pa"]
    for n in names:
        assert hasattr(tcb, n), n


def test_host_logic_without_gpu(known):
    assert tcb.dedup_send_targets(np.array([3, 4, 9]), np.array([0, 5, 10])) == known["dedup_send_targets"][0]
    assert tcb.dedup_send_targets(np.array([3, 4, 9]), np.array([0, 5, 10]), self_rank=0) == known["dedup_send_targets"][1]
    assert tcb.dedup_send_targets(np.array([], dtype=np.int64), np.array([0, 5, 10])) == []
    b = tcb.range_bounds([tcb.NodeRange(0, 5), tcb.NodeRange(5, 5)])
    assert [tcb.owner_of(b, v) for v in (0, 4, 5, 9)] == [0, 0, 1, 1]
    with pytest.raises(ValueError):
        tcb.NodeRange(-1, 2)
    with pytest.raises(ValueError):
        tcb.Task(0, 0)
    with pytest.raises(ValueError):
        tcb.CostKind.parse("nope")
    assert tcb.CostKind.parse("PredSum") is tcb.CostKind.PRED_SUM


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure mode")
def test_no_cpu_fallback():
    raw = tcb.RawGraph.from_pairs([(0, 1), (1, 2), (0, 2)])
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        tcb.normalize(raw)


def test_tuning_ranges():
    """tc_set_tuning validates its caps on the host (no GPU work): the small
    warp-tier cap accepts 0..256 (129..256 force the tier's wide form) and
    rejects anything beyond; -1 restores the default."""
    from paper_1406_5687_b200 import _lib
    L = _lib.lib()
    try:
        for ok in (0, 8, 128, 129, 256):
            assert L.tc_set_tuning(0, ok) == 0, ok
        for bad in (257, 4096, -2):
            assert L.tc_set_tuning(0, bad) != 0, bad
        assert L.tc_set_tuning(2, 513) != 0 and L.tc_set_tuning(1, 4097) != 0
        assert L.tc_set_tuning(9, 1) != 0
    finally:
        for key in (0, 2, 1):
            assert L.tc_set_tuning(key, -1) == 0
