// dist.cu — the library-owned NCCL communicator of the sharded build (
// DESIGN.md §6).
//
// One process per GPU.  Rank 0 draws an NCCL unique id (fmi_get_unique_id), the caller broadcasts the
// 128 bytes with whatever it uses for plumbing (torch.distributed), every rank calls fmi_dist_init.  A
// sharded build whose fmi_dist has no allreduce callback then sums its global-level quantities
// (partial moments, projections, octant counts and energies of the nodes above the shard depth; the
// paper's recursion P:296-313 distributed by Morton range) with ncclAllReduce IN PLACE on the device
// buffers, on the library stream: no staging copy, no host round trip, ordered with the kernels.
//
// NCCL is resolved at run time (dlopen of libnccl.so.2): in a process that imported torch this is the
// NCCL torch already loaded (same soname), so there is exactly one NCCL in the process; a host
// without NCCL gets FMI_ENCCL from fmi_dist_init instead of a library that fails to load.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

#include "../../include/fmi.h"
#include "fmi_internal.cuh"

namespace fmi {

namespace {

struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
};

NcclApi& api() {
  static NcclApi a;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      a.why = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
      return;
    }
    a.getUniqueId = reinterpret_cast<decltype(a.getUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    a.commInitRank = reinterpret_cast<decltype(a.commInitRank)>(dlsym(h, "ncclCommInitRank"));
    a.allReduce = reinterpret_cast<decltype(a.allReduce)>(dlsym(h, "ncclAllReduce"));
    a.commDestroy = reinterpret_cast<decltype(a.commDestroy)>(dlsym(h, "ncclCommDestroy"));
    a.getErrorString = reinterpret_cast<decltype(a.getErrorString)>(dlsym(h, "ncclGetErrorString"));
    a.ok = a.getUniqueId && a.commInitRank && a.allReduce && a.commDestroy && a.getErrorString;
    if (!a.ok) a.why = "libnccl.so.2 lacks a required symbol";
  });
  return a;
}

std::mutex g_comm_mu;
ncclComm_t g_comm = nullptr;
int g_rank = 0, g_world = 0;

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) fail(FMI_ENCCL, std::string(what) + ": " + api().getErrorString(r));
}

NcclApi& need_api() {
  NcclApi& a = api();
  if (!a.ok) fail(FMI_ENCCL, a.why);
  return a;
}

}  // namespace

bool dist_comm_ready(int world) {
  std::lock_guard<std::mutex> lk(g_comm_mu);
  return g_comm != nullptr && g_world == world;
}

// in-place SUM over the ranks of n elements (dtype 0 fp64, 1 int64, 2 fp32) on stream s
void dist_comm_allreduce(void* dev, int64_t n, int dtype, cudaStream_t s) {
  if (n <= 0) return;
  NcclApi& a = need_api();
  std::lock_guard<std::mutex> lk(g_comm_mu);
  if (!g_comm) fail(FMI_ENCCL, "no library communicator: call fmi_dist_init on every rank first");
  const ncclDataType_t t = dtype == 0 ? ncclFloat64 : (dtype == 1 ? ncclInt64 : ncclFloat32);
  nccl_check(a.allReduce(dev, dev, (size_t)n, t, ncclSum, g_comm, s), "ncclAllReduce");
}

void dist_nccl_unique_id(void* out128) {
  static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id is 128 bytes");
  ncclUniqueId id;
  nccl_check(need_api().getUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(out128, &id, sizeof id);
}

void dist_nccl_init(int rank, int world, const void* id128) {
  NcclApi& a = need_api();
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof id);
  std::lock_guard<std::mutex> lk(g_comm_mu);
  if (g_comm) {
    a.commDestroy(g_comm);
    g_comm = nullptr;
  }
  ncclComm_t c = nullptr;
  nccl_check(a.commInitRank(&c, world, id, rank), "ncclCommInitRank");
  g_comm = c;
  g_rank = rank;
  g_world = world;
}

void dist_nccl_finalize() {
  std::lock_guard<std::mutex> lk(g_comm_mu);
  if (g_comm) api().commDestroy(g_comm);
  g_comm = nullptr;
  g_world = 0;
}

}  // namespace fmi

