// nccl_shard.cu — native NCCL transport for row sharding (pc_net_set_sharding_nccl).
//
// The sharded engine's one exchange step (all-gather of the
// refined candidate bounds before the write-back) enqueued directly as
// ncclAllGather on the engine's CUDA stream — no host callback, no Python on
// the data path; over NVLink 5 / NVSwitch on one node. libnccl.so.2 is
// loaded with dlopen (the same library torch.distributed uses when it is
// already mapped), so the product library has no link-time NCCL dependency.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

#include "../../include/polycert_b200.h"

namespace {

struct NcclApi {
  void* so = nullptr;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  std::string err;
};

NcclApi& api() {
  static NcclApi a;
  static std::once_flag once;
  std::call_once(once, [] {
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      a.so = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (a.so) break;
    }
    if (!a.so) {
      a.err = std::string("nccl: cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(a.so, "ncclGetUniqueId"));
    a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(a.so, "ncclCommInitRank"));
    a.all_gather = reinterpret_cast<decltype(a.all_gather)>(dlsym(a.so, "ncclAllGather"));
    a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(a.so, "ncclCommDestroy"));
    a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(a.so, "ncclGetErrorString"));
    if (!a.get_unique_id || !a.comm_init_rank || !a.all_gather || !a.comm_destroy)
      a.err = "nccl: libnccl.so.2 lacks the needed symbols";
  });
  return a;
}

const char* nccl_msg(ncclResult_t r) {
  return api().error_string ? api().error_string(r) : "nccl error";
}

}  // namespace

// Communicator of one sharded net (owned through pc_nccl_comm_destroy).
struct pc_nccl_comm {
  ncclComm_t comm = nullptr;
  int world = 1;
};

extern "C" {

// pc_allgather_fn over NCCL: gather `bytes` from every rank, ordered on `stream`.
int pc_nccl_allgather(void* user, const void* d_send, void* d_recv, size_t bytes, void* stream) {
  auto* c = static_cast<pc_nccl_comm*>(user);
  const ncclResult_t r = api().all_gather(d_send, d_recv, bytes, ncclUint8, c->comm,
                                          static_cast<cudaStream_t>(stream));
  return r == ncclSuccess ? 0 : 1;
}

int pc_nccl_unique_id(void* out128, char* err, int err_len) {
  NcclApi& a = api();
  if (!a.err.empty()) {
    if (err && err_len > 0) std::strncpy(err, a.err.c_str(), err_len - 1), err[err_len - 1] = 0;
    return 1;
  }
  ncclUniqueId id;
  const ncclResult_t r = a.get_unique_id(&id);
  if (r != ncclSuccess) {
    if (err && err_len > 0) std::strncpy(err, nccl_msg(r), err_len - 1), err[err_len - 1] = 0;
    return 1;
  }
  std::memcpy(out128, id.internal, NCCL_UNIQUE_ID_BYTES);
  return 0;
}

pc_nccl_comm* pc_nccl_comm_create(int device, int rank, int world, const void* id128, char* err,
                                  int err_len) {
  NcclApi& a = api();
  auto fail = [&](const std::string& m) -> pc_nccl_comm* {
    if (err && err_len > 0) std::strncpy(err, m.c_str(), err_len - 1), err[err_len - 1] = 0;
    return nullptr;
  };
  if (!a.err.empty()) return fail(a.err);
  if (cudaSetDevice(device) != cudaSuccess) return fail("nccl: cudaSetDevice failed");
  ncclUniqueId id;
  std::memcpy(id.internal, id128, NCCL_UNIQUE_ID_BYTES);
  auto* c = new pc_nccl_comm;
  c->world = world;
  const ncclResult_t r = a.comm_init_rank(&c->comm, world, id, rank);
  if (r != ncclSuccess) {
    delete c;
    return fail(std::string("nccl: ncclCommInitRank: ") + nccl_msg(r));
  }
  return c;
}

void pc_nccl_comm_destroy(pc_nccl_comm* c) {
  if (!c) return;
  if (c->comm && api().comm_destroy) api().comm_destroy(c->comm);
  delete c;
}

}  // extern "C"
