// nccl.cu -- the NCCL layer of the C ABI (tc_nccl_init_all,
// tc_exchange_lists, tc_allreduce_u64): the collectives of the multi-GPU
// schemes for a caller that binds the library directly (a reference-side
// ctypes / cgo binding) instead of going through
// torch.distributed.  They replace the reference's in-process message
// runtime: reduce_sum / barrier (runtime.py:255-259, 402-414) and the list
// exchange of _surrogate_rank (space_efficient.py:116-144).
//
// libnccl is resolved at the first call (dlopen of TCB_NCCL_LIB, else
// libnccl.so.2 -- the pip NCCL torch bundles), so the rest of the library
// loads without it.  Types come from the NCCL header the build points at.
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>
#include <string>

#include "common.cuh"

namespace tcb {
namespace {

struct NcclApi {
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) init_rank = nullptr;
  decltype(&ncclCommInitAll) init_all = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    const char* env = getenv("TCB_NCCL_LIB");
    void* h = dlopen(env ? env : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      err = std::string("cannot load NCCL (") + (env ? env : "libnccl.so.2") + "): " + dlerror();
      return;
    }
#define TCB_SYM(field, name) api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name))
    TCB_SYM(get_unique_id, "ncclGetUniqueId");
    TCB_SYM(init_rank, "ncclCommInitRank");
    TCB_SYM(init_all, "ncclCommInitAll");
    TCB_SYM(destroy, "ncclCommDestroy");
    TCB_SYM(all_reduce, "ncclAllReduce");
    TCB_SYM(send, "ncclSend");
    TCB_SYM(recv, "ncclRecv");
    TCB_SYM(group_start, "ncclGroupStart");
    TCB_SYM(group_end, "ncclGroupEnd");
    TCB_SYM(error_string, "ncclGetErrorString");
#undef TCB_SYM
    if (!api.all_reduce || !api.send || !api.group_end) err = "NCCL library lacks the required symbols";
  });
  TC_REQUIRE(err.empty() && api.all_reduce, TC_ECUDA, err.empty() ? "NCCL unavailable" : err);
  return api;
}

void check_nccl(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw Error(TC_ECUDA, std::string(what) + ": " + (nccl().error_string ? nccl().error_string(r) : "NCCL error"));
}

ncclDataType_t nccl_type(int32_t dtype) {
  switch (dtype) {  // TC_DT_* (include/tcb200.h)
    case TC_DT_U8: return ncclUint8;
    case TC_DT_I32: return ncclInt32;
    case TC_DT_I64: return ncclInt64;
    case TC_DT_U64: return ncclUint64;
    default: throw Error(TC_EINVAL, "unknown dtype");
  }
}

size_t type_bytes(int32_t dtype) { return dtype == TC_DT_U8 ? 1 : (dtype == TC_DT_I32 ? 4 : 8); }

ncclRedOp_t nccl_op(int32_t op) {
  switch (op) {  // TC_OP_*
    case TC_OP_SUM: return ncclSum;
    case TC_OP_MAX: return ncclMax;
    case TC_OP_MIN: return ncclMin;
    default: throw Error(TC_EINVAL, "unknown reduction");
  }
}

}  // namespace
}  // namespace tcb

using namespace tcb;

extern "C" {

int tc_nccl_unique_id(void* id_out) {
  return guarded([&] {
    TC_REQUIRE(id_out != nullptr, TC_EINVAL, "NULL id buffer");
    ncclUniqueId id;
    check_nccl(nccl().get_unique_id(&id), "ncclGetUniqueId");
    memcpy(id_out, &id, sizeof(id));
  });
}

int tc_nccl_init_rank(const void* id, int32_t nranks, int32_t rank, tc_nccl_t* comm) {
  return guarded([&] {
    TC_REQUIRE(id && comm, TC_EINVAL, "NULL argument");
    TC_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, TC_EINVAL, "bad rank / nranks");
    ncclUniqueId uid;
    memcpy(&uid, id, sizeof(uid));
    ncclComm_t c = nullptr;
    check_nccl(nccl().init_rank(&c, nranks, uid, rank), "ncclCommInitRank");
    *comm = reinterpret_cast<tc_nccl_t>(c);
  });
}

int tc_nccl_init_all(int32_t ndev, const int32_t* devices, tc_nccl_t* comms) {
  return guarded([&] {
    TC_REQUIRE(ndev >= 1 && comms, TC_EINVAL, "bad device list");
    std::vector<ncclComm_t> c(ndev);
    check_nccl(nccl().init_all(c.data(), ndev, reinterpret_cast<const int*>(devices)), "ncclCommInitAll");
    for (int i = 0; i < ndev; ++i) comms[i] = reinterpret_cast<tc_nccl_t>(c[i]);
  });
}

int tc_nccl_free(tc_nccl_t comm) {
  return guarded([&] {
    if (comm) check_nccl(nccl().destroy(reinterpret_cast<ncclComm_t>(comm)), "ncclCommDestroy");
  });
}

int tc_allreduce(void* buf, int64_t count, int32_t dtype, int32_t op, tc_nccl_t comm, tc_stream_t stream) {
  return guarded([&] {
    TC_REQUIRE(comm != nullptr && count >= 0, TC_EINVAL, "bad all-reduce arguments");
    if (count == 0) return;
    check_nccl(nccl().all_reduce(buf, buf, (size_t)count, nccl_type(dtype), nccl_op(op),
                                 reinterpret_cast<ncclComm_t>(comm), (cudaStream_t)stream),
               "ncclAllReduce");
  });
}

int tc_allreduce_u64(unsigned long long* buf, int64_t count, tc_nccl_t comm, tc_stream_t stream) {
  return tc_allreduce(buf, count, TC_DT_U64, TC_OP_SUM, comm, stream);
}

int tc_exchange(const void* send, const int64_t* send_counts, void* recv, const int64_t* recv_counts, int32_t dtype,
                int32_t nranks, tc_nccl_t comm, tc_stream_t stream) {
  return guarded([&] {
    TC_REQUIRE(comm != nullptr && send_counts && recv_counts && nranks >= 1, TC_EINVAL, "bad exchange arguments");
    const size_t eb = type_bytes(dtype);
    const ncclDataType_t t = nccl_type(dtype);
    auto* c = reinterpret_cast<ncclComm_t>(comm);
    const auto& api = nccl();
    check_nccl(api.group_start(), "ncclGroupStart");
    size_t so = 0, ro = 0;
    for (int p = 0; p < nranks; ++p) {  // all-to-all-v as grouped point-to-point
      TC_REQUIRE(send_counts[p] >= 0 && recv_counts[p] >= 0, TC_EINVAL, "negative count");
      if (send_counts[p])
        check_nccl(api.send(static_cast<const char*>(send) + so * eb, (size_t)send_counts[p], t, p, c,
                            (cudaStream_t)stream),
                   "ncclSend");
      if (recv_counts[p])
        check_nccl(api.recv(static_cast<char*>(recv) + ro * eb, (size_t)recv_counts[p], t, p, c, (cudaStream_t)stream),
                   "ncclRecv");
      so += (size_t)send_counts[p];
      ro += (size_t)recv_counts[p];
    }
    check_nccl(api.group_end(), "ncclGroupEnd");
  });
}

int tc_exchange_lists(const int32_t* send, const int64_t* send_counts, int32_t* recv, const int64_t* recv_counts,
                      int32_t nranks, tc_nccl_t comm, tc_stream_t stream) {
  return tc_exchange(send, send_counts, recv, recv_counts, TC_DT_I32, nranks, comm, stream);
}

}  // extern "C"
