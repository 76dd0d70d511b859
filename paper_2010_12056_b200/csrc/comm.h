// Collectives of the 1-D processor grid (Alg. 3 lines 14/17/18, Alg. 4 line 9):
// reduce-scatter of the partial MTTKRP, all-gather of factor rows, all-reduce of the last
// mode's Gram / dS / scalars.  Two backends behind one interface:
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
};

// 0 = ok; otherwise 4 (CUDA) or 5 (NCCL) with a message in *msg
int comm_reduce_scatter(Comm& c, const double* send, double* recv, int64_t count, std::string* msg);
int comm_all_gather(Comm& c, const double* send, double* recv, int64_t count, std::string* msg);
int comm_all_reduce(Comm& c, double* buf, int64_t count, std::string* msg);
int comm_group_start(Comm& c, std::string* msg);
int comm_group_end(Comm& c, std::string* msg);

LocalGroup* local_group_create(int world);
void local_group_destroy(LocalGroup* g);
int local_group_world(const LocalGroup* g);

}  // namespace cpd
