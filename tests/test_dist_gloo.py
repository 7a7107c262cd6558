"""The multi-GPU surrogate protocol (paper_1406_5687_b200/distributed.py)
over torch.distributed with the gloo backend at world_size 2 and 3, on CPU.
The per-rank device kernels are replaced by NumpyOps (tests/dist_helpers.py);
collectives, buffer layout, metrics and the reduction are the product's."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import SMALL

CASES = ["er_60_0.2_21", "pa_500_8_11", "sparse_labels", "gnm_2000_16000"]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, name, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from conftest import SMALL as S
    from dist_helpers import NumpyOps, shard_from_arrays
    from paper_1406_5687_b200.distributed import surrogate_rank

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        case = S[name]
        bounds = case[f"bounds_predsum_{world}"]
        sh = shard_from_arrays(case["eff_indptr"], case["eff_indices"], int(bounds[rank]), int(bounds[rank + 1]))
        total, met = surrogate_rank(sh, bounds, ops=NumpyOps(), device=torch.device("cpu"))
        q.put((rank, total, met.triangles, met.data_msgs_to.tolist(), met.data_msgs_sent, met.bytes_sent,
               met.partition_bytes))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("name", CASES)
def test_surrogate_protocol_gloo(name, world):
    case = SMALL[name]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    T = int(case["T"][0])
    for rank, total, tri, to, sent, bts, pb in res:
        assert total == T
        assert tri == int(case[f"surr_tri_{world}"][rank])
        assert to == case[f"surr_census_{world}"][rank].tolist()
        assert sent == int(case[f"surr_msgs_{world}"][rank])
        assert bts == int(case[f"surr_bytes_{world}"][rank])
        assert pb == int(case[f"surr_pbytes_{world}"][rank])


def _direct_worker(rank, world, port, name, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from conftest import SMALL as S
    from dist_helpers import NumpyOps, shard_from_arrays
    from paper_1406_5687_b200.distributed import direct_rank

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        case = S[name]
        bounds = case[f"bounds_predsum_{world}"]
        sh = shard_from_arrays(case["eff_indptr"], case["eff_indices"], int(bounds[rank]), int(bounds[rank + 1]))
        total, met = direct_rank(sh, bounds, ops=NumpyOps(), device=torch.device("cpu"))
        q.put((rank, total, met.triangles, met.requests_to.tolist(), met.data_msgs_to.tolist(), met.requests_sent,
               met.data_msgs_sent, met.bytes_sent, met.completion_msgs_sent, met.partition_bytes, met.wire_bytes))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("name", CASES)
def test_direct_protocol_gloo(name, world):
    """count_space_direct's deduplicated pull (distributed.direct_rank):
    per-rank lowest-vertex partials and the reference's per-pair counters."""
    case = SMALL[name]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_direct_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    T = int(case["T"][0])
    st = case[f"direct_stats_{world}"]
    for rank, total, tri, req_to, data_to, nreq, nsent, bts, ncomp, pb, wire in res:
        assert total == T
        assert tri == int(case[f"direct_tri_{world}"][rank])
        assert req_to == case[f"direct_req_{world}"][rank].tolist()
        assert data_to == case[f"direct_census_{world}"][rank].tolist()
        assert [nreq, nsent, bts, ncomp, pb] == st[rank].tolist()
