// Library-owned NCCL communicator for the multi-GPU hot path (one process per
// GPU).  NCCL is resolved at run time (dlopen of libnccl.so.2, preferring the
// copy already mapped into the process, e.g. PyTorch's), so the library has
// no link-time NCCL dependency and never loads a second, different NCCL.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include "common.cuh"

namespace lc {

struct Comm {
    ncclComm_t comm = nullptr;
    int world = 1, rank = 0;
    bool ready() const { return comm != nullptr; }
};

// NCCL unique id of a new communicator (rank 0 creates it; the caller moves it
// to the other ranks by any out-of-band means).
void comm_unique_id(ncclUniqueId *id);
// Join the communicator on the calling thread's current device.
void comm_init(Comm &c, const ncclUniqueId &id, int world, int rank);
void comm_destroy(Comm &c);
// In-place int64 MAX all-reduce of n words on stream s (the partials exchange:
// items of other ranks hold INT64_MIN, the bits of -0.0).
void comm_allreduce_max_i64(Comm &c, void *buf, size_t n, cudaStream_t s);
// Loaded NCCL version (e.g. 22809), 0 if NCCL cannot be loaded.
int nccl_version();

}  // namespace lc
