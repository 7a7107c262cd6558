"""Small workload for compute-sanitizer: every engine tier (forced caps), both
formulations, the padded-pool and list-pool streaming paths, partitioning,
surrogate, the sharded multi-rank pipeline (emulated), the host-input
normalize pipeline, parser, generators (dev/CI tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
os.environ.setdefault("TCB_HOST_PIPELINE_MIN", "4096")  # small lists take the chunked host pipeline too
import torch  # noqa: E402

import paper_1406_5687_b200 as tcb  # noqa: E402
from paper_1406_5687_b200 import _lib  # noqa: E402
from paper_1406_5687_b200.distributed import emulate_ranks  # noqa: E402
from paper_1406_5687_b200.graph_io import er_edges, rmat_edges  # noqa: E402
from paper_1406_5687_b200.sequential import count_lowest  # noqa: E402

L = _lib.lib()
graphs = []
for raw in (er_edges(3000, 40000, 1), rmat_edges(11, 8, 2)):
    graphs.append(tcb.build_graph(tcb.normalize(tcb.RawGraph(n=0, edges=raw))))
core = [(a, b) for a in range(300) for b in range(a + 1, 300)]
graphs.append(tcb.build_graph(tcb.normalize(tcb.RawGraph.from_pairs(core))))
for caps in ((128, 512, 4096), (0, 512, 4096), (8, 16, 4096), (8, 16, 8)):
    _lib.check(L.tc_set_tuning(0, caps[0]))
    _lib.check(L.tc_set_tuning(2, caps[1]))
    _lib.check(L.tc_set_tuning(1, caps[2]))
    for g in graphs:
        T = tcb.count_triangles_seq(g)
        assert int(count_lowest(g).item()) == T
        total, _ = tcb.count_space_surrogate(g, 3)
        assert total == T
_lib.check(L.tc_set_tuning(0, -1))
_lib.check(L.tc_set_tuning(2, -1))
_lib.check(L.tc_set_tuning(1, -1))
for g in graphs:
    total, _ = emulate_ranks(g, 4)
    tcb.count_dynamic(g, 5)
    _ = g.full_indices
tcb.load_edge_list(b"# x\n0 1\n1 2\n2 0\n")
# host-input normalize (chunked copy + merges) and the sharded pipeline
from paper_1406_5687_b200 import sharded as S  # noqa: E402
raw = rmat_edges(12, 8, 4)
host = torch.empty(tuple(raw.shape), dtype=torch.int32, pin_memory=True)
host.copy_(raw)
gh = tcb.build_graph(tcb.normalize(tcb.RawGraph(n=0, edges=host)))
T = tcb.count_triangles_seq(gh)
for cost in ("predsum", "engine"):
    shards, _ = S.emulate_build(raw, 3, cost=cost)
    assert S.emulate_count(shards, round_words=256)[0] == T
    assert S.emulate_count(shards, round_words=256)[0] == T  # kept round plans: index_emit + rebind
    shards = S.emulate_rebalance(shards, [3.0, 1.0, 2.0])
    assert S.emulate_count(shards)[0] == T
from paper_1406_5687_b200.sequential import count_merge_path  # noqa: E402
assert int(count_merge_path(gh).item()) == T
torch.cuda.synchronize()
print("sanitize workload ok")
