"""The sharded multi-GPU pipeline (paper_1406_5687_b200/sharded.py): a
distributed normalize + build_graph where each rank keeps only its node
range, and the surrogate count over bounded exchange rounds.

CPU: the protocol with the numpy per-rank steps (tests/dist_helpers.py),
emulated in one process and over gloo at world size 2 / 3.  GPU: the
device steps (csrc/shard.cu) emulated rank by rank on one B200.  Every case
is checked against the reference's own outputs (tests/golden): each rank's
forward lists equal the reference graph's rows of its range, the PRED_SUM
bounds equal partition_ranges, the rank partials / census / bytes_sent equal
count_space_surrogate's metrics, and the total equals T."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import SMALL
from dist_helpers import NumpyShardOps
from paper_1406_5687_b200 import sharded as S

CASES = ["er_60_0.2_21", "pa_500_8_11", "sparse_labels", "gnm_2000_16000"]


def _check_build(case, shards, P):
    assert shards[0].bounds.tolist() == case[f"bounds_predsum_{P}"].tolist()
    ip, ix = case["eff_indptr"], case["eff_indices"]
    for sh in shards:
        lo, hi = sh.lo, sh.hi
        assert sh.n == len(case["relabel"]) and sh.m == len(ix)
        assert np.array_equal(sh.indptr.cpu().numpy(), ip[lo: hi + 1] - ip[lo])
        assert np.array_equal(sh.indices.cpu().numpy(), ix[ip[lo]: ip[hi]])
        if sh.relabel is not None:
            assert np.array_equal(sh.relabel.cpu().numpy(), case["relabel"])
            assert np.array_equal(sh.orig_ids.cpu().numpy(), case["orig_ids"])


def _check_count(case, tot, mets, P):
    assert tot == int(case["T"][0])
    assert [m.triangles for m in mets] == case[f"surr_tri_{P}"].tolist()
    assert np.stack([m.data_msgs_to for m in mets]).tolist() == case[f"surr_census_{P}"].tolist()
    assert [m.bytes_sent for m in mets] == case[f"surr_bytes_{P}"].tolist()
    assert [m.data_msgs_sent for m in mets] == case[f"surr_msgs_{P}"].tolist()


@pytest.mark.parametrize("name", CASES)
def test_sharded_protocol_emulated_numpy(name):
    case = SMALL[name]
    raw = torch.as_tensor(case["raw"].astype(np.int32))
    ops = NumpyShardOps()
    for P in (2, 3):
        shards, _ = S.emulate_build(raw, P, ops=ops, keep_maps=True)
        _check_build(case, shards, P)
        for rw in (8, 1 << 27):  # many small rounds / one round
            tot, mets, _ = S.emulate_count(shards, ops=ops, round_words=rw)
            _check_count(case, tot, mets, P)
        eshards, _ = S.emulate_build(raw, P, cost="engine", ops=ops)
        assert sum(sh.m_local for sh in eshards) == len(case["eff_indices"])
        assert S.emulate_count(eshards, ops=ops)[0] == int(case["T"][0])


def _check_rebalanced(case, shards, P):
    """Ranges tile [0, n), every rank holds exactly the reference rows of its
    range, partials sum to T."""
    ip, ix = case["eff_indptr"], case["eff_indices"]
    b = shards[0].bounds.tolist()
    assert b[0] == 0 and b[-1] == len(case["relabel"]) and all(x <= y for x, y in zip(b, b[1:]))
    for r, sh in enumerate(shards):
        assert sh.bounds.tolist() == b and (sh.lo, sh.hi) == (b[r], b[r + 1])
        assert np.array_equal(sh.indptr.cpu().numpy(), ip[sh.lo: sh.hi + 1] - ip[sh.lo])
        assert np.array_equal(sh.indices.cpu().numpy(), ix[ip[sh.lo]: ip[sh.hi]])


@pytest.mark.parametrize("name", ["pa_500_8_11", "gnm_2000_16000"])
def test_sharded_rebalance_emulated_numpy(name):
    """The measured refinement: skewed rank times move the bounds towards
    the slow rank's side, the shards stay the reference's rows and the count
    stays T."""
    case = SMALL[name]
    raw = torch.as_tensor(case["raw"].astype(np.int32))
    ops = NumpyShardOps()
    for P in (2, 3):
        shards, _ = S.emulate_build(raw, P, cost="engine", ops=ops)
        b0 = shards[0].bounds.tolist()
        shards = S.emulate_rebalance(shards, [10.0] + [1.0] * (P - 1), ops=ops)  # rank 0 was slow
        _check_rebalanced(case, shards, P)
        assert shards[0].bounds[1] < b0[1]
        tot, mets, _ = S.emulate_count(shards, ops=ops, round_words=64)
        assert tot == int(case["T"][0]) and sum(m.triangles for m in mets) == tot
        shards = S.emulate_rebalance(shards, [1.0] * P, ops=ops)  # equal times: weights already balanced
        _check_rebalanced(case, shards, P)
        assert S.emulate_count(shards, ops=ops)[0] == int(case["T"][0])


def test_sharded_run_record_matches_reference_rows():
    """Per-rank rows of the run CSV from an emulated 3-rank sharded count:
    gathered by one all-reduce, equal to each rank's own metrics and to the
    reference's count_space_surrogate rows (triangles, messages, bytes)."""
    import io

    from paper_1406_5687_b200.metrics import RUN_COLUMNS, write_run_csv

    case = SMALL["pa_500_8_11"]
    raw = torch.as_tensor(case["raw"].astype(np.int32))
    ops = NumpyShardOps()
    P = 3
    shards, _ = S.emulate_build(raw, P, ops=ops)
    tot, mets, _ = S.emulate_count(shards, ops=ops)
    res, _ = S.emulate([S.gather_metrics_gen(mets[r], P, r, busy_ms=1.5 * (r + 1)) for r in range(P)])
    for r in range(P):  # every rank holds every rank's row
        assert [m.triangles for m in res[r]] == case["surr_tri_3"].tolist()
        assert [m.bytes_sent for m in res[r]] == case["surr_bytes_3"].tolist()
        assert [m.data_msgs_sent for m in res[r]] == case["surr_msgs_3"].tolist()
        assert np.stack([m.data_msgs_to for m in res[r]]).tolist() == case["surr_census_3"].tolist()
        assert [m.partition_bytes for m in res[r]] == [m.partition_bytes for m in mets]
    rec = S.run_record(tot, res[0], 0.004, graph="pa_500_8_11", seed=11)
    fh = io.StringIO()
    write_run_csv([rec], fh)
    rows = [ln.split(",") for ln in fh.getvalue().strip().split("\n")]
    assert rows[0] == RUN_COLUMNS and len(rows) == 1 + P
    tri = RUN_COLUMNS.index("triangles")
    assert [int(r[tri]) for r in rows[1:]] == case["surr_tri_3"].tolist()
    assert rows[1][RUN_COLUMNS.index("busy_time")] == "0.001500"


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, name, cost, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from conftest import SMALL as SM
    from dist_helpers import NumpyShardOps as Ops
    from paper_1406_5687_b200 import sharded as SS

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        case = SM[name]
        raw = torch.as_tensor(case["raw"].astype(np.int32))
        sl, base = SS.slice_of(raw, world, rank)
        sh = SS.build_sharded(sl.contiguous(), base, cost=cost, ops=Ops(), keep_maps=True)
        tot, met = SS.count_sharded(sh, ops=Ops(), round_words=16)
        if cost == "engine":
            # the measured refinement and the metrics gather over real collectives:
            # rank 0 "was slow", so its range shrinks; the count must not move
            b1 = int(sh.bounds[1])
            sh = SS.rebalance_sharded(sh, 9.0 if rank == 0 else 1.0, ops=Ops())
            assert int(sh.bounds[1]) < b1
            tot2, met = SS.count_sharded(sh, ops=Ops(), round_words=64)
            assert tot2 == tot
            rows = SS.gather_metrics(met, busy_ms=float(rank + 1))
            assert [m.rank for m in rows] == list(range(world)) and sum(m.triangles for m in rows) == tot
            assert rows[rank].bytes_sent == met.bytes_sent and abs(rows[rank].busy_time - (rank + 1) / 1e3) < 1e-9
        q.put((rank, sh.lo, sh.hi, sh.bounds.tolist(), sh.indptr.numpy().tolist(), sh.indices.numpy().tolist(),
               tot, met.triangles, met.data_msgs_to.tolist(), met.bytes_sent, met.data_msgs_sent))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("name", ["pa_500_8_11", "sparse_labels"])
@pytest.mark.parametrize("cost", ["predsum", "engine"])
def test_sharded_gloo(name, world, cost):
    case = SMALL[name]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, cost, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ip, ix = case["eff_indptr"], case["eff_indices"]
    T = int(case["T"][0])
    for rank, lo, hi, bounds, sip, six, tot, tri, to, bts, sent in res:
        assert tot == T
        assert np.array_equal(np.asarray(sip), ip[lo: hi + 1] - ip[lo])
        assert np.array_equal(np.asarray(six, np.int64), ix[ip[lo]: ip[hi]])
        if cost == "predsum":
            assert bounds == case[f"bounds_predsum_{world}"].tolist()
            assert tri == int(case[f"surr_tri_{world}"][rank])
            assert to == case[f"surr_census_{world}"][rank].tolist()
            assert bts == int(case[f"surr_bytes_{world}"][rank])
            assert sent == int(case[f"surr_msgs_{world}"][rank])
    # the ranges tile [0, n)
    assert res[0][1] == 0 and res[-1][2] == len(case["relabel"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(SMALL))
def test_sharded_device_emulated(name):
    """The device steps (csrc/shard.cu) for every fixture at P = 2, 3, 5, 8."""
    case = SMALL[name]
    if "bounds_predsum_2" not in case:
        pytest.skip("fixture without partition goldens")
    raw = torch.as_tensor(case["raw"].astype(np.int32)).cuda()
    for P in (2, 3, 5, 8):
        if f"surr_tri_{P}" not in case:
            continue
        shards, _ = S.emulate_build(raw, P, keep_maps=True)
        _check_build(case, shards, P)
        for rw in (64, 1 << 27, 64):  # the third count re-uses the kept round plans (index_emit + rebind)
            tot, mets, _ = S.emulate_count(shards, round_words=rw)
            _check_count(case, tot, mets, P)
        eshards, _ = S.emulate_build(raw, P, cost="engine")
        assert S.emulate_count(eshards)[0] == int(case["T"][0])
        if P == 3:  # shards cut out of a replicated Graph (count_space_surrogate_dist's path)
            import paper_1406_5687_b200 as tcb
            g = tcb.build_graph(tcb.normalize(tcb.RawGraph.from_pairs(case["raw"])))
            gsh = [S.shard_from_graph(g, case["bounds_predsum_3"], r) for r in range(P)]
            tot, mets, _ = S.emulate_count(gsh)
            _check_count(case, tot, mets, P)
        eshards = S.emulate_rebalance(eshards, [float(1 + (r % 3)) for r in range(P)])
        _check_rebalanced(case, eshards, P)
        assert S.emulate_count(eshards, round_words=64)[0] == int(case["T"][0])


@pytest.mark.gpu
@pytest.mark.parametrize("P", [12, 20, 32])
@pytest.mark.parametrize("name", ["pa_2000_10_3", "gnm_2000_16000", "rmat_s10"])
def test_sharded_device_many_ranks(name, P):
    """More than 8 ranks (16 / 32 lanes per row in the pack kernels, ranks
    with empty ranges): the device send sizes equal the numpy restatement's,
    the packed messages carry exactly those lists, and the total is T."""
    case = SMALL[name]
    raw = torch.as_tensor(case["raw"].astype(np.int32)).cuda()
    shards, _ = S.emulate_build(raw, P)
    nops, dops = NumpyShardOps(), S.ShardOps()
    for r, sh in enumerate(shards):
        _, want = nops.send_sizes(sh, P, r)
        sd, got = dops.send_sizes(sh, P, r)
        assert got.tolist() == want.tolist(), (name, P, r)
        lens, ids = dops.send_pack(sh, P, r, sd, int(got[0].sum()), int(got[1].sum()))
        wl, wi = nops.send_pack(sh, P, r, None, int(want[0].sum()), int(want[1].sum()))
        lo = np.concatenate([[0], np.cumsum(got[0])])
        wo = np.concatenate([[0], np.cumsum(got[1])])
        for j in range(P):  # per destination: the same multiset of lists (order inside a destination is free)
            a = sorted(lens[lo[j]: lo[j + 1]].cpu().tolist())
            assert a == sorted(wl[lo[j]: lo[j + 1]].tolist()), (name, P, r, j)
            assert sorted(ids[wo[j]: wo[j + 1]].cpu().tolist()) == sorted(wi[wo[j]: wo[j + 1]].tolist()), (name, P, r, j)
    tot, mets, _ = S.emulate_count(shards, round_words=512)
    assert tot == int(case["T"][0]) and sum(m.triangles for m in mets) == tot


@pytest.mark.gpu
def test_sharded_device_long_lists():
    """Rows of a few hundred ids (32 lanes per row in the receive index, rows
    beyond the pack kernel's 128-id staging) against the oracle."""
    from oracle import oracle as O

    rng = np.random.default_rng(3)
    n = 1600
    iu, iv = np.triu_indices(n, 1)
    keep = rng.random(len(iu)) < 0.35
    raw_np = np.stack([iu[keep], iv[keep]], 1).astype(np.int64)
    og = O.build_graph(*O.normalize(raw_np))
    assert float(og.eff_deg.mean()) > 200
    T = O.count_triangles(og)
    raw = torch.as_tensor(raw_np.astype(np.int32)).cuda()
    for P in (3, 8):
        for cost in ("predsum", "engine"):
            shards, _ = S.emulate_build(raw, P, cost=cost)
            for sh in shards:
                assert np.array_equal(sh.indices.cpu().numpy(), og.eff_indices[og.eff_indptr[sh.lo]: og.eff_indptr[sh.hi]])
            assert S.emulate_count(shards, round_words=1 << 16)[0] == T
            assert S.emulate_count(shards, round_words=1 << 16)[0] == T


@pytest.mark.gpu
@pytest.mark.parametrize("P", [2, 4, 8])
def test_sharded_device_cfg2(configs, P):
    """cfg 2 (PA n = 10^6, 50 M edges) at full size: the reference's PRED_SUM
    bounds, surrogate partials and census, per rank."""
    import bench

    c = configs["cfg2_pa_1000000_100_seed1"]
    raw = bench.host_raw_edges("cfg2", pin=False).cuda()
    shards, _ = S.emulate_build(raw, P)
    del raw
    assert shards[0].bounds.tolist() == c[f"bounds_predsum_{P}"]
    assert sum(sh.m_local for sh in shards) == c["m"]
    for rep in range(2):  # the second count runs on the kept send plan, exchange plan and round plans
        tot, mets, _ = S.emulate_count(shards, round_words=1 << 22)
        assert tot == c["T"]
        assert [m.triangles for m in mets] == c[f"surr_tri_{P}"]
        assert np.stack([m.data_msgs_to for m in mets]).tolist() == c[f"surr_census_{P}"]
    # the pack is deterministic: two packs of one shard are byte-identical
    ops = S.ShardOps()
    sh = shards[0]
    sd, sz = ops.send_sizes(sh, P, 0)
    a = ops.send_pack(sh, P, 0, sd, int(sz[0].sum()), int(sz[1].sum()))
    b = ops.send_pack(sh, P, 0, sd, int(sz[0].sum()), int(sz[1].sum()))
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])
    assert int(a[0].sum()) <= int(sz[1].sum()) and int((a[0] > 0).all())
