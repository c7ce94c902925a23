// comm.cuh — NCCL plumbing of librbrp (internal).  NCCL is loaded at run time
// (dlopen "libnccl.so.2"), so the library loads and runs single-GPU without it.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/rbrp.h"

struct rbrp_comm {
  void* nccl_comm;   // ncclComm_t
  int nranks, rank, device;
};

namespace rbrp {
// Collectives used by the multi-GPU path; each returns 0 or an rbrp_status.
// chunk totals / positive counts: every rank contributes its own chunks, zeros elsewhere
// (sum of exact zeros: bitwise exact), so all ranks see identical arrays (C1).
int comm_allgather_chunks(rbrp_comm* c, double* ctot, int32_t* cpos, int64_t chunk0,
                          int64_t nch_local, int64_t nchunks, cudaStream_t s);
int comm_allreduce_f64(rbrp_comm* c, double* buf, int64_t count, cudaStream_t s);
int comm_allreduce_max_i64(rbrp_comm* c, int64_t* buf, int64_t count, cudaStream_t s);
int comm_allreduce_sum_i32(rbrp_comm* c, int32_t* buf, int64_t count, cudaStream_t s);
// ncclCommGetAsyncError: RBRP_ENCCL if a collective of this communicator failed
int comm_check(rbrp_comm* c);
}  // namespace rbrp
