"""The NCCL plumbing of the multi-GPU schemes (distributed.py) on one GPU:
a world-size-1 NCCL process group runs every collective the N-GPU path
issues (all_to_all_single of counts, lists and ids; all_reduce of the
uint64-as-int64 partials) on device tensors.  Rank interplay at N > 1 is
covered by the gloo tests (test_dist_gloo.py) and the per-rank emulation
(test_gpu_parity.py); this checks that the same code drives NCCL."""

import socket

import pytest
import torch
import torch.distributed as dist

import paper_1406_5687_b200 as tcb
from paper_1406_5687_b200.distributed import count_space_direct_dist, count_space_surrogate_dist
from paper_1406_5687_b200.graph_io import rmat_edges
from paper_1406_5687_b200.sequential import count_middle, count_middle_part

pytestmark = pytest.mark.gpu


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module")
def nccl_group():
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_port()}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


def test_nccl_world1_schemes(nccl_group):
    assert dist.get_backend() == "nccl"
    raw = rmat_edges(14, 16, 5)
    g = tcb.build_graph(tcb.normalize(tcb.RawGraph(n=1 << 14, edges=raw)))
    T = tcb.count_triangles_seq(g)
    total, met = count_space_surrogate_dist(g)
    assert total == T and met.triangles == T
    total, met = count_space_direct_dist(g)
    assert total == T and met.triangles == T
    c = count_middle(g, 0, g.n)  # range count + all_reduce
    dist.all_reduce(c)
    assert int(c.item()) == T
    c = count_middle_part(g, 0, 1)  # bench.py's replicated step at world size 1
    dist.all_reduce(c)
    assert int(c.item()) == T
    # the sharded space-efficient pipeline: distributed build + bounded-round count
    from paper_1406_5687_b200.sharded import build_sharded, count_sharded
    for cost in ("predsum", "engine"):
        sh = build_sharded(raw.contiguous(), 0, cost=cost)
        assert sh.n == g.n and sh.m == g.m
        assert torch.equal(sh.indices, g.eff_indices) and torch.equal(sh.indptr, g.eff_indptr)
        total, met = count_sharded(sh, round_words=1024)
        assert total == T and met.triangles == T


@pytest.mark.parametrize("mode", ["replicated", "surrogate", "direct"])
def test_bench_multi_gpu_path_world1(mode, tmp_path):
    """bench.py's N-GPU step (torchrun, NCCL process group, the rank's share
    of the count, all-reduce, max over ranks) at world size 1
    (TCB_BENCH_DIST=1): the JSON line carries the reference's total."""
    import json
    import os
    import subprocess
    import sys

    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, TCB_BENCH_DIST="1")
    for attempt in range(3):  # a rendezvous port can be taken between _port() and torchrun's bind
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
               "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(repo, "bench.py"),
               "--gpus", "1", "--steps", "2", "--warmup", "3", "--mode", mode, "--no-e2e", "--no-cpu-baseline",
               "--config", "cfg1", "--partitioned", "cfg1" if mode == "replicated" else ""]
        out = subprocess.run(cmd, cwd=repo, env=env, capture_output=True, text=True, timeout=600)
        transient = ("address already in use", "eaddrinuse", "connection refused", "rendezvous", "timed out")
        if out.returncode == 0 or not any(t in out.stderr.lower() for t in transient):
            break
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([x for x in out.stdout.splitlines() if x.startswith("{")][-1])
    assert line["workload_detail"]["triangles"] == 722 and line["n_gpus"] == 1
    assert {"replicated": "replicated", "surrogate": "surrogate", "direct": "pull"}[mode] in \
        line["workload_detail"]["parallelism"]
    if mode == "replicated":  # the sharded space-efficient scheme through NCCL (sharded.py)
        part = line["partitioned"][0]
        assert part.get("error") is None, part
        assert part["triangles"] == 722 and part["triangles_ok"] and part["n_gpus"] == 1
        # the run CSV of the reference's schema: header + one row per rank
        assert part["run_csv"][0].startswith("suite,algo,mode,ranks") and len(part["run_csv"]) == 2
        assert part["run_csv"][1].split(",")[12] == "722" and len(part["refinement_trail"]) == 3


def test_capi_nccl_layer_world1():
    """The C ABI's own NCCL layer (tc_nccl_*, tc_allreduce_u64,
    tc_exchange_lists) at world size 1, and the sharded pipeline driven
    through it without torch.distributed."""
    import ctypes

    import numpy as np

    from paper_1406_5687_b200 import _lib
    from paper_1406_5687_b200 import sharded as S

    torch.cuda.set_device(0)
    comm = S.CComm(S.CComm.unique_id(), 1, 0)
    try:
        x = torch.arange(5, dtype=torch.int64, device="cuda")
        _lib.call("tc_allreduce_u64", _lib.ptr(x), 5, comm.h, _lib.stream())
        assert x.tolist() == [0, 1, 2, 3, 4]
        src = torch.arange(10, dtype=torch.int32, device="cuda")
        dst = torch.zeros(10, dtype=torch.int32, device="cuda")
        n = np.array([10], np.int64)
        _lib.call("tc_exchange_lists", _lib.ptr(src), n.ctypes.data_as(ctypes.c_void_p), _lib.ptr(dst),
                  n.ctypes.data_as(ctypes.c_void_p), 1, comm.h, _lib.stream())
        assert torch.equal(src, dst)
        raw = rmat_edges(13, 16, 7)
        g = tcb.build_graph(tcb.normalize(tcb.RawGraph(n=0, edges=raw)))
        T = tcb.count_triangles_seq(g)
        sh = S.run_capi(S.build_gen(raw.contiguous(), 0, 1, 0, "engine"), comm)
        assert torch.equal(sh.indices, g.eff_indices)
        total, met = S.run_capi(S.count_gen(sh, 1, 0, round_words=4096), comm)
        assert total == T and met.triangles == T
    finally:
        comm.close()
