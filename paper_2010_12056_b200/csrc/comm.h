// Collectives of the processor grid (Alg. 3 lines 14/17/18, Alg. 4 line 9): reduce-scatter of
// the partial MTTKRP and all-gather of factor rows within Proc-Slice(x_n), all-reduce of the
// Gram / dS / scalars over all ranks.  Two backends behind one interface:
//   * NCCL (one process per GPU, NVLink/NVSwitch) -- the product path;
//   * an in-process "local group": `world` contexts on ONE device, each driven by its own
//     host thread, exchanging through device pointers with fixed-order sums -- used to
//     verify the partitioned algorithm on a single GPU (tests).
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>
#include <stdint.h>

#include <string>

namespace cpd {

struct LocalGroup;

struct Comm {
  ncclComm_t nccl = nullptr;
  LocalGroup* lg = nullptr;
  int rank = 0, world = 1;
  cudaStream_t st = nullptr;
  bool owns_nccl = false;  // a communicator from comm_split (destroyed by comm_free)
};

// 0 = ok; otherwise 4 (CUDA) or 5 (NCCL) with a message in *msg
int comm_reduce_scatter(Comm& c, const double* send, double* recv, int64_t count, std::string* msg);
int comm_all_gather(Comm& c, const double* send, double* recv, int64_t count, std::string* msg);
int comm_all_reduce(Comm& c, double* buf, int64_t count, std::string* msg);
int comm_group_start(Comm& c, std::string* msg);
int comm_group_end(Comm& c, std::string* msg);

// sub-communicator of `parent` (N-D processor grid): NCCL ncclCommSplit or a local sub-group;
// collective over parent's ranks.  *out gets nccl/lg/rank/world of the child (st copied).
int comm_split(const Comm& parent, int color, int key, Comm* out, std::string* msg);
void comm_free(Comm& c);  // NCCL child communicators only (local sub-groups belong to the parent)

int comm_exchange_ptr(Comm& c, void* mine, void** all, std::string* msg);
// NCCL symmetric window of `bytes` (ncclMemAlloc + ncclCommWindowRegister, collective over comm)
// and the flat addresses of every rank's buffer (peers[0..nranks)); peer.cu
int nccl_window_peers(ncclComm_t comm, size_t bytes, int nranks, void** buf, void** peers, void** win,
                      cudaStream_t st, std::string* msg);
void nccl_window_free(ncclComm_t comm, void* buf, void* win);
int comm_barrier(Comm& c, double* scratch1, std::string* msg);

LocalGroup* local_group_create(int world);
int local_group_split(LocalGroup* g, int rank, int color, int key, LocalGroup** out, int* out_rank, int* out_size);
void local_group_destroy(LocalGroup* g);
int local_group_world(const LocalGroup* g);

}  // namespace cpd
