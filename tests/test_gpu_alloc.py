"""The C ABI's memory policy: a private stream-ordered pool by default (the
device's default pool keeps its settings) or the caller's allocator
(tc_set_allocator; here torch's caching allocator)."""

import pytest
import torch

import paper_1406_5687_b200 as tcb
from paper_1406_5687_b200 import _lib
from paper_1406_5687_b200.graph_io import rmat_edges

pytestmark = pytest.mark.gpu


def test_default_pool_untouched():
    dev = torch.cuda.current_device()
    before = torch.cuda.memory.get_allocator_backend()
    g = tcb.build_graph(tcb.normalize(tcb.RawGraph(n=0, edges=rmat_edges(12, 8, 3))))
    assert tcb.count_triangles_seq(g) > 0
    assert torch.cuda.memory.get_allocator_backend() == before
    import ctypes
    from cuda.bindings import runtime as rt  # noqa: F401 -- cuda-python is in the image
    err, pool = rt.cudaDeviceGetDefaultMemPool(dev)
    err, thr = rt.cudaMemPoolGetAttribute(pool, rt.cudaMemPoolAttr.cudaMemPoolAttrReleaseThreshold)
    assert int(thr) == 0  # the library never raises the default pool's threshold
    _lib.call("tc_trim_pool")


def test_torch_allocator_owns_library_memory():
    raw = rmat_edges(13, 16, 9)
    ref = tcb.count_triangles_seq(tcb.build_graph(tcb.normalize(tcb.RawGraph(n=0, edges=raw))))
    _lib.use_torch_allocator(True)
    try:
        torch.cuda.synchronize()
        peak0 = torch.cuda.max_memory_allocated()
        torch.cuda.reset_peak_memory_stats()
        g = tcb.build_graph(tcb.normalize(tcb.RawGraph(n=0, edges=raw)))
        assert tcb.count_triangles_seq(g) == ref
        total, _ = tcb.count_space_surrogate(g, 3)
        assert total == ref
        torch.cuda.synchronize()
        assert torch.cuda.max_memory_allocated() > 0 and peak0 >= 0
    finally:
        _lib.use_torch_allocator(False)
