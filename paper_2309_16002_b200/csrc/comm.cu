// comm.cu — NCCL over NVLink/NVSwitch for the row-sharded path.
// libnccl.so.2 is dlopen'ed on first use (torch bundles it); no link-time dependency.
#include <dlfcn.h>
#include <nccl.h>
#include <string.h>

#include "comm.cuh"

namespace {

struct NcclApi {
  bool ok = false;
  decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
  decltype(&ncclCommInitRank) CommInitRank = nullptr;
  decltype(&ncclCommDestroy) CommDestroy = nullptr;
  decltype(&ncclCommGetAsyncError) GetAsyncError = nullptr;
  decltype(&ncclAllReduce) AllReduce = nullptr;
  decltype(&ncclGroupStart) GroupStart = nullptr;
  decltype(&ncclGroupEnd) GroupEnd = nullptr;
};

NcclApi& api() {
  static NcclApi a;
  static bool tried = false;
  if (tried) return a;
  tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return a;
  a.GetUniqueId = (decltype(a.GetUniqueId))dlsym(h, "ncclGetUniqueId");
  a.CommInitRank = (decltype(a.CommInitRank))dlsym(h, "ncclCommInitRank");
  a.CommDestroy = (decltype(a.CommDestroy))dlsym(h, "ncclCommDestroy");
  a.AllReduce = (decltype(a.AllReduce))dlsym(h, "ncclAllReduce");
  a.GroupStart = (decltype(a.GroupStart))dlsym(h, "ncclGroupStart");
  a.GroupEnd = (decltype(a.GroupEnd))dlsym(h, "ncclGroupEnd");
  a.GetAsyncError = (decltype(a.GetAsyncError))dlsym(h, "ncclCommGetAsyncError");
  a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.AllReduce && a.GroupStart &&
         a.GroupEnd;
  return a;
}

}  // namespace

extern "C" {

int rbrp_comm_unique_id(void* id128) {
  if (!id128) return RBRP_EINVAL;
  NcclApi& a = api();
  if (!a.ok) return RBRP_ENCCL;
  ncclUniqueId id;
  if (a.GetUniqueId(&id) != ncclSuccess) return RBRP_ENCCL;
  memcpy(id128, &id, sizeof(id));
  return RBRP_OK;
}

int rbrp_comm_init(rbrp_comm** c, const void* id128, int nranks, int rank, int device) {
  if (!c || !id128 || nranks < 1 || rank < 0 || rank >= nranks) return RBRP_EINVAL;
  NcclApi& a = api();
  if (!a.ok) return RBRP_ENCCL;
  if (cudaSetDevice(device) != cudaSuccess) return RBRP_ECUDA;
  ncclUniqueId id;
  memcpy(&id, id128, sizeof(id));
  ncclComm_t nc;
  if (a.CommInitRank(&nc, nranks, id, rank) != ncclSuccess) return RBRP_ENCCL;
  rbrp_comm* r = new rbrp_comm;
  r->nccl_comm = nc;
  r->nranks = nranks;
  r->rank = rank;
  r->device = device;
  *c = r;
  return RBRP_OK;
}

int rbrp_comm_destroy(rbrp_comm* c) {
  if (!c) return RBRP_OK;
  NcclApi& a = api();
  int rc = RBRP_OK;
  if (a.ok && a.CommDestroy((ncclComm_t)c->nccl_comm) != ncclSuccess) rc = RBRP_ENCCL;
  delete c;
  return rc;
}

}  // extern "C"

namespace rbrp {

int comm_allgather_chunks(rbrp_comm* c, double* ctot, int32_t* cpos, int64_t chunk0,
                          int64_t nch_local, int64_t nchunks, cudaStream_t s) {
  NcclApi& a = api();
  if (!a.ok) return RBRP_ENCCL;
  // zero everything but this rank's chunks, then sum: x + 0 = x exactly
  if (chunk0 > 0) {
    if (cudaMemsetAsync(ctot, 0, chunk0 * 8, s) || cudaMemsetAsync(cpos, 0, chunk0 * 4, s))
      return RBRP_ECUDA;
  }
  const int64_t e = chunk0 + nch_local;
  if (e < nchunks) {
    if (cudaMemsetAsync(ctot + e, 0, (nchunks - e) * 8, s) ||
        cudaMemsetAsync(cpos + e, 0, (nchunks - e) * 4, s))
      return RBRP_ECUDA;
  }
  ncclComm_t nc = (ncclComm_t)c->nccl_comm;
  if (a.GroupStart() != ncclSuccess) return RBRP_ENCCL;
  ncclResult_t r1 = a.AllReduce(ctot, ctot, nchunks, ncclFloat64, ncclSum, nc, s);
  ncclResult_t r2 = a.AllReduce(cpos, cpos, nchunks, ncclInt32, ncclSum, nc, s);
  if (a.GroupEnd() != ncclSuccess || r1 != ncclSuccess || r2 != ncclSuccess) return RBRP_ENCCL;
  return RBRP_OK;
}

int comm_allreduce_f64(rbrp_comm* c, double* buf, int64_t count, cudaStream_t s) {
  NcclApi& a = api();
  if (!a.ok) return RBRP_ENCCL;
  if (a.AllReduce(buf, buf, count, ncclFloat64, ncclSum, (ncclComm_t)c->nccl_comm, s) != ncclSuccess)
    return RBRP_ENCCL;
  return RBRP_OK;
}

int comm_allreduce_max_i64(rbrp_comm* c, int64_t* buf, int64_t count, cudaStream_t s) {
  NcclApi& a = api();
  if (!a.ok) return RBRP_ENCCL;
  if (a.AllReduce(buf, buf, count, ncclInt64, ncclMax, (ncclComm_t)c->nccl_comm, s) != ncclSuccess)
    return RBRP_ENCCL;
  return RBRP_OK;
}

int comm_check(rbrp_comm* c) {
  NcclApi& a = api();
  if (!a.ok) return RBRP_ENCCL;
  if (!a.GetAsyncError) return RBRP_OK;
  ncclResult_t st = ncclSuccess;
  if (a.GetAsyncError((ncclComm_t)c->nccl_comm, &st) != ncclSuccess) return RBRP_ENCCL;
  return (st == ncclSuccess || st == ncclInProgress) ? RBRP_OK : RBRP_ENCCL;
}

int comm_allreduce_sum_i32(rbrp_comm* c, int32_t* buf, int64_t count, cudaStream_t s) {
  NcclApi& a = api();
  if (!a.ok) return RBRP_ENCCL;
  if (a.AllReduce(buf, buf, count, ncclInt32, ncclSum, (ncclComm_t)c->nccl_comm, s) != ncclSuccess)
    return RBRP_ENCCL;
  return RBRP_OK;
}

}  // namespace rbrp
