"""ctypes binding of libtcb200.so (the C ABI declared in include/tcb200.h).

The product has no CPU fallback: if the shared library is missing or no CUDA
device is present, every compute entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.environ.get("TCB_LIB") or os.path.join(_HERE, "libtcb200.so")
_LIB = None

TC_OK, TC_EINVAL, TC_EINDEX, TC_ECUDA, TC_ENOMEM = 0, -1, -2, -3, -4

_i64, _i32, _u64, _vp = ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64, ctypes.c_void_p
_pi64 = ctypes.POINTER(ctypes.c_int64)

# name -> argtypes (every device pointer / stream is passed as c_void_p)
_SIGS = {
    "tc_abi_version": [],
    "tc_trim_pool": [],
    "tc_set_allocator": [_vp, _vp, _vp],
    "tc_normalize": [_vp, _i64, _vp, _pi64, _pi64, _vp],
    "tc_build_graph": [_vp, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "tc_build_graph_deg": [_vp, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "tc_normalize_host": [_vp, _i64, _vp, _vp, _pi64, _pi64, _vp, _vp, _vp],
    "tc_build_full": [_vp, _vp, _vp, _vp, _vp, _i64, _vp, _vp, _vp],
    "tc_count_middle": [_vp, _vp, _vp, _vp, _vp, _vp, _i32, _i64, _i64, _i64, _vp, _i32, _vp, _vp],
    "tc_count_merge_path": [_vp, _vp, _i64, _vp, _vp],
    "tc_count_lowest": [_vp, _vp, _i64, _i64, _i64, _vp, _i32, _vp, _vp],
    "tc_plan_middle": [_vp, _vp, _vp, _vp, _vp, _vp, _i32, _i64, _i64, _i64, _vp, _i32, ctypes.POINTER(_vp), _vp],
    "tc_plan_run": [_vp, _vp, _vp],
    "tc_plan_rebind": [_vp, _vp, _vp],
    "tc_plan_middle_parts": [_vp, _vp, _vp, _vp, _vp, _vp, _i32, _i64, _i64, _i64, _vp, _i32, _i32,
                             ctypes.POINTER(_vp), _vp],
    "tc_plan_run_part": [_vp, _i32, _vp, _vp],
    "tc_plan_free": [_vp],
    "tc_count_owners": [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _vp, _i32, _vp, _i32, _vp],
    "tc_tile_pull": [_vp, _vp, _i64, _vp, _vp, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _pi64, _pi64, _vp],
    "tc_intersect_count": [_vp, _i64, _vp, _i64, _vp, _vp],
    "tc_engine_timing": [_i32, _vp, _vp, _vp],
    "tc_set_tuning": [_i32, _i64],
    "tc_count_brute": [_vp, _vp, _i64, _vp, _vp],
    "tc_node_costs": [_i32, _vp, _vp, _vp, _vp, _i64, _vp, _vp],
    "tc_balanced_bounds": [_vp, _i64, _i64, _i64, _vp, _vp],
    "tc_plan_tasks": [_vp, _i64, _i64, _vp, _vp, _vp, _vp, _pi64, _pi64, _pi64, _vp],
    "tc_surrogate_census": [_vp, _vp, _i64, _vp, _i32, _vp, _vp, _vp],
    "tc_direct_census": [_vp, _vp, _i64, _vp, _i32, _vp, _vp, _vp],
    "tc_direct_requests": [_vp, _vp, _i64, _i64, _vp, _i32, _vp, _vp, _i64, _vp, _vp, _vp, _vp],
    "tc_direct_table": [_vp, _i64, _i64, _vp, _vp, _i64, _i64, _vp, _vp],
    "tc_surrogate_records": [_vp, _vp, _i64, _vp, _i32, _i32, _i64, _vp, _vp, _i64, _vp, _pi64, _vp],
    "tc_surrogate_pack_sizes": [_vp, _vp, _i64, _vp, _pi64, _vp],
    "tc_surrogate_pack": [_vp, _vp, _vp, _i64, _vp, _vp, _vp],
    "tc_owner_segments": [_vp, _vp, _i64, _i64, _i64, _i64, _vp, _vp, _i64, _pi64, _vp],
    "tc_segments_csr": [_vp, _vp, _i64, _i64, _vp, _vp, _vp, _vp, _vp],
    "tc_shard_minmax": [_vp, _i64, ctypes.POINTER(_i32), ctypes.POINTER(_i32), _vp],
    "tc_shard_label_scan": [_vp, _i64, _i64, _i64, _vp, _vp, _vp],
    "tc_shard_relabel_map": [_vp, _vp, _i64, _vp, _pi64, ctypes.POINTER(_i32), _vp],
    "tc_shard_keys": [_vp, _i64, _vp, _i32, _vp, _vp, _vp],
    "tc_shard_dedup": [_vp, _i64, _i32, _vp, _pi64, _vp],
    "tc_shard_degrees": [_vp, _i64, _vp, _vp],
    "tc_shard_order": [_vp, _i64, _vp, _vp, _vp],
    "tc_shard_orient": [_vp, _i64, _vp, _vp, _vp, _vp],
    "tc_shard_predsum": [_vp, _i64, _vp, _vp, _vp],
    "tc_shard_route": [_vp, _i64, _vp, _i32, _vp, _vp, _vp],
    "tc_shard_csr": [_vp, _i64, _i64, _i64, _vp, _vp, _vp],
    "tc_shard_pool": [_vp, _vp, _i64, _vp, _vp, _vp],
    "tc_shard_engine_cost": [_vp, _vp, _i64, _i64, _vp, _vp],
    "tc_shard_engine_cost_fin": [_vp, _vp, _i64, _i64, _i64, _vp, _vp],
    "tc_shard_send_plan_len": [_i64, _i32, _pi64],
    "tc_shard_send_sizes": [_vp, _vp, _i64, _vp, _vp, _i32, _i32, _vp, _vp, _vp],
    "tc_shard_send_pack": [_vp, _vp, _i64, _vp, _vp, _vp, _i32, _i32, _vp, _vp, _vp, _vp],
    "tc_shard_index": [_vp, _i64, _vp, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _pi64, _vp],
    "tc_shard_index_emit": [_vp, _i64, _vp, _i64, _i64, _i64, _vp, _vp, _vp, _vp],
    "tc_nccl_unique_id": [_vp],
    "tc_nccl_init_rank": [_vp, _i32, _i32, ctypes.POINTER(_vp)],
    "tc_nccl_init_all": [_i32, _vp, _vp],
    "tc_nccl_free": [_vp],
    "tc_allreduce": [_vp, _i64, _i32, _i32, _vp, _vp],
    "tc_allreduce_u64": [_vp, _i64, _vp, _vp],
    "tc_exchange": [_vp, _vp, _vp, _vp, _i32, _i32, _vp, _vp],
    "tc_exchange_lists": [_vp, _vp, _vp, _vp, _i32, _vp, _vp],
    "tc_parse_edge_list": [_vp, _i64, _vp, _i64, _pi64, _pi64, _pi64, ctypes.POINTER(ctypes.c_int32),
                           ctypes.POINTER(ctypes.c_int32), _vp],
    "tc_gen_er": [_i64, _i64, _u64, _vp, _vp],
    "tc_gen_rmat": [_i32, _i64, _u64, _vp, _vp],
    "tc_gen_chung_lu": [_i64, ctypes.c_double, ctypes.c_double, ctypes.c_double, _u64, _vp, _i64, _pi64, _vp],
    "tc_pa_num_edges": [_i64, _i64],
    "tc_gen_pa_host": [_i64, _i64, _u64, _vp],
}
EXPORTED = sorted(_SIGS) + ["tc_last_error", "tc_launch_count"]


def build_library(force=False):
    """Compile libtcb200.so in-tree (nvcc, sm_100a)."""
    if force or not os.path.exists(_SO):
        subprocess.run(["make", "-s", "-j8", "-C", _HERE], check=True)
    return _SO


def _nccl_path():
    """The NCCL the C ABI's collectives dlopen (torch's pip NCCL), unless
    TCB_NCCL_LIB says otherwise."""
    if os.environ.get("TCB_NCCL_LIB"):
        return
    try:
        import nvidia.nccl as nn

        p = os.path.join(list(nn.__path__)[0], "lib", "libnccl.so.2")
        if os.path.exists(p):
            os.environ["TCB_NCCL_LIB"] = p
    except ImportError:
        pass


def lib():
    """Load the library (build it first if absent)."""
    global _LIB
    if _LIB is None:
        _nccl_path()
        if not os.path.exists(_SO):
            build_library()
        L = ctypes.CDLL(_SO)
        for name, args in _SIGS.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = _i64 if name == "tc_pa_num_edges" else ctypes.c_int
        L.tc_launch_count.argtypes = []
        L.tc_launch_count.restype = ctypes.c_ulonglong
        L.tc_last_error.argtypes = []
        L.tc_last_error.restype = ctypes.c_char_p
        _LIB = L
    return _LIB


def check(rc):
    if rc == TC_OK:
        return
    msg = lib().tc_last_error().decode(errors="replace")
    if rc == TC_EINVAL:
        raise ValueError(msg)
    if rc == TC_EINDEX:
        raise IndexError(msg)
    raise RuntimeError(f"libtcb200 error {rc}: {msg}")


def call(name, *args):
    check(getattr(lib(), name)(*args))


def device():
    """The CUDA device the product runs on; raises loudly without one."""
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1406_5687_b200 needs a CUDA device (B200); no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t):
    """Device pointer of a tensor (None -> NULL)."""
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr())


_ALLOC_CB = []  # every registered callback pair stays alive: blocks are freed by the allocator that made them


def use_torch_allocator(enable=True):
    """Route the library's scratch and plan memory through torch's caching
    allocator (tc_set_allocator), so torch owns every device byte."""
    L = lib()
    if not enable:
        check(L.tc_set_allocator(None, None, None))
        return
    AF = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p)
    FF = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p)

    def _alloc(nbytes, stream, _ctx):
        try:
            return torch.cuda.caching_allocator_alloc(int(nbytes), stream=int(stream or 0))
        except Exception:  # noqa: BLE001 -- reported to the library as NULL (TC_ENOMEM)
            return None

    def _free(ptr, _stream, _ctx):
        torch.cuda.caching_allocator_delete(int(ptr))

    cb = (AF(_alloc), FF(_free))
    _ALLOC_CB.append(cb)
    check(L.tc_set_allocator(ctypes.cast(cb[0], ctypes.c_void_p), ctypes.cast(cb[1], ctypes.c_void_p), None))
