// Cross-GPU exchange of the row-sharded index (BASELINE.json north_star: "each shard produces its
// local top-K, and an NCCL allgather of K (score, item-id) pairs over NVLink feeds a final merge";
// SURVEY.md §8(a) a5, §8(e)).
//
// NCCL is loaded at run time (dlopen of libnccl.so.2; the copy PyTorch already loaded is reused),
// so liblinr.so has no link-time NCCL dependency and still loads on machines without it. One
// communicator per index handle; a search with a communicator attached is ONE collective: every
// rank packs its sorted shard-local keys [B][K] and pass counts [B] into one buffer of B*(K+1)
// u64, ncclAllGather moves G*B*(K+1)*8 bytes, and the merge kernel reduces the G lists to the
// global top-K on every rank (allgather semantics, exact by reading R13).
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

#include "internal.h"

namespace linr {

namespace {

struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  bool ok = false;
  std::string why;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);   // already in the process (torch)
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.why = std::string("dlopen libnccl.so.2 failed: ") + dlerror();
      return;
    }
    api.get_unique_id = (decltype(api.get_unique_id))dlsym(h, "ncclGetUniqueId");
    api.comm_init_rank = (decltype(api.comm_init_rank))dlsym(h, "ncclCommInitRank");
    api.all_gather = (decltype(api.all_gather))dlsym(h, "ncclAllGather");
    api.comm_destroy = (decltype(api.comm_destroy))dlsym(h, "ncclCommDestroy");
    api.error_string = (decltype(api.error_string))dlsym(h, "ncclGetErrorString");
    api.ok = api.get_unique_id && api.comm_init_rank && api.all_gather && api.comm_destroy && api.error_string;
    if (!api.ok) api.why = "libnccl.so.2 lacks a required symbol";
  });
  return api;
}

int nccl_fail(ncclResult_t r, const char* where) {
  const NcclApi& a = nccl();
  set_error(std::string(where) + ": " + (a.error_string ? a.error_string(r) : "nccl error"));
  return LINR_ENCCL;
}

}  // namespace

int comm_create(int device, const uint8_t id[128], int rank, int world, void** out) {
  const NcclApi& a = nccl();
  if (!a.ok) {
    set_error(a.why);
    return LINR_ENCCL;
  }
  ncclUniqueId uid;
  static_assert(sizeof(uid.internal) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(uid.internal, id, 128);
  int prev = -1;
  cudaGetDevice(&prev);
  if (prev != device) cudaSetDevice(device);
  ncclComm_t c = nullptr;
  const ncclResult_t r = a.comm_init_rank(&c, world, uid, rank);
  if (prev >= 0 && prev != device) cudaSetDevice(prev);
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommInitRank");
  *out = c;
  return LINR_OK;
}

void comm_destroy(void* c) {
  if (c && nccl().ok) nccl().comm_destroy((ncclComm_t)c);
}

int comm_allgather_u64(void* c, const uint64_t* send, uint64_t* recv, size_t count, cudaStream_t st) {
  const ncclResult_t r = nccl().all_gather(send, recv, count, ncclUint64, (ncclComm_t)c, st);
  if (r != ncclSuccess) return nccl_fail(r, "ncclAllGather");
  return LINR_OK;
}

}  // namespace linr

extern "C" int linr_nccl_unique_id(uint8_t* out) {
  using namespace linr;
  if (!out) {
    set_error("null out");
    return LINR_EINVAL;
  }
  const NcclApi& a = nccl();
  if (!a.ok) {
    set_error(a.why);
    return LINR_ENCCL;
  }
  ncclUniqueId uid;
  const ncclResult_t r = a.get_unique_id(&uid);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  std::memcpy(out, uid.internal, 128);
  return LINR_OK;
}
