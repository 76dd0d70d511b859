// Collective backends of the 1-D grid (see comm.h).
#include <algorithm>
#include <condition_variable>
#include <map>
#include <mutex>
#include <utility>
#include <vector>

#include "comm.h"
#include "kernels.h"

namespace cpd {

struct LocalGroup {
  int world;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long gen = 0;
  std::vector<const double*> src;
  std::vector<double*> dst;
  std::vector<cudaEvent_t> ev_in, ev_out;
  std::vector<double*> scratch;
  std::vector<size_t> cap;
  // sub-groups (N-D processor grid): colour/key published per rank, children by (split number, colour)
  std::vector<int> colors, keys, nsplit;
  std::map<std::pair<int, int>, LocalGroup*> children;
  explicit LocalGroup(int w)
      : world(w), src(w), dst(w), ev_in(w, nullptr), ev_out(w, nullptr), scratch(w, nullptr), cap(w, 0),
        colors(w, 0), keys(w, 0), nsplit(w, 0) {}
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    long g = gen;
    if (++arrived == world) {
      arrived = 0;
      gen++;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

namespace {

struct Ptrs {
  const double* p[8];
};

// dst[e] = Σ_{q < world} src_q[off + e]   (fixed order q = 0, 1, ...)
__global__ void local_sum_kernel(Ptrs s, int world, int64_t off, int64_t n, double* __restrict__ dst) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    double v = s.p[0][off + e];
    for (int q = 1; q < world; q++) v += s.p[q][off + e];
    dst[e] = v;
  }
}

unsigned blocks_for(int64_t n) {
  int64_t b = (n + 255) / 256;
  if (b > 148 * 8) b = 148 * 8;
  return (unsigned)(b < 1 ? 1 : b);
}

int cuda_fail(cudaError_t e, std::string* msg) {
  if (e == cudaSuccess) return 0;
  if (msg) *msg = std::string("local group: ") + cudaGetErrorString(e);
  return 4;
}

// phase 1: publish buffers, make this rank's stream wait for every rank's prior work
int local_enter(Comm& c, const double* src, double* dst, std::string* msg) {
  LocalGroup* g = c.lg;
  if (!g->ev_in[c.rank]) {
    cudaError_t e = cudaEventCreateWithFlags(&g->ev_in[c.rank], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&g->ev_out[c.rank], cudaEventDisableTiming);
    if (e != cudaSuccess) return cuda_fail(e, msg);
  }
  g->src[c.rank] = src;
  g->dst[c.rank] = dst;
  cudaError_t e = cudaEventRecord(g->ev_in[c.rank], c.st);
  if (e != cudaSuccess) return cuda_fail(e, msg);
  g->barrier();
  for (int q = 0; q < g->world; q++)
    if ((e = cudaStreamWaitEvent(c.st, g->ev_in[q], 0)) != cudaSuccess) return cuda_fail(e, msg);
  return 0;
}

// phase 2: nobody may overwrite a published buffer before every rank has read it
int local_leave(Comm& c, std::string* msg) {
  LocalGroup* g = c.lg;
  cudaError_t e = cudaEventRecord(g->ev_out[c.rank], c.st);
  if (e != cudaSuccess) return cuda_fail(e, msg);
  g->barrier();
  for (int q = 0; q < g->world; q++)
    if ((e = cudaStreamWaitEvent(c.st, g->ev_out[q], 0)) != cudaSuccess) return cuda_fail(e, msg);
  g->barrier();  // the events may be re-recorded by the next collective only after every wait is enqueued
  return 0;
}

Ptrs gather_ptrs(LocalGroup* g, bool use_dst) {
  Ptrs p{};
  for (int q = 0; q < g->world; q++) p.p[q] = use_dst ? g->dst[q] : g->src[q];
  return p;
}

int nccl_fail(ncclResult_t r, std::string* msg) {
  if (r == ncclSuccess) return 0;
  if (msg) *msg = std::string("NCCL: ") + ncclGetErrorString(r);
  return 5;
}

}  // namespace

LocalGroup* local_group_create(int world) {
  if (world < 1 || world > 8) return nullptr;
  return new LocalGroup(world);
}
void local_group_destroy(LocalGroup* g) {
  if (!g) return;
  for (auto& kv : g->children) local_group_destroy(kv.second);
  for (int q = 0; q < g->world; q++) {
    if (g->ev_in[q]) cudaEventDestroy(g->ev_in[q]);
    if (g->ev_out[q]) cudaEventDestroy(g->ev_out[q]);
    if (g->scratch[q]) cudaFree(g->scratch[q]);
  }
  delete g;
}
int local_group_world(const LocalGroup* g) { return g ? g->world : 0; }

// collective over g's ranks (each from its own thread, same call order): the ranks with equal
// `color` form one child group, ordered by (key, rank); the child is created once, owned by g
int local_group_split(LocalGroup* g, int rank, int color, int key, LocalGroup** out, int* out_rank, int* out_size) {
  g->colors[rank] = color;
  g->keys[rank] = key;
  g->barrier();
  std::vector<std::pair<int, int>> mem;
  for (int q = 0; q < g->world; q++)
    if (g->colors[q] == color) mem.push_back({g->keys[q], q});
  std::sort(mem.begin(), mem.end());
  int me = 0;
  for (int k = 0; k < (int)mem.size(); k++)
    if (mem[k].second == rank) me = k;
  const int seq = g->nsplit[rank]++;
  {
    std::lock_guard<std::mutex> lk(g->mu);
    auto& ch = g->children[{seq, color}];
    if (!ch) ch = new LocalGroup((int)mem.size());
    *out = ch;
  }
  *out_rank = me;
  *out_size = (int)mem.size();
  g->barrier();  // colours/keys may be overwritten by the next split only after every rank read them
  return 0;
}

int comm_reduce_scatter(Comm& c, const double* send, double* recv, int64_t count, std::string* msg) {
  if (c.world == 1) return 0;
  if (!c.lg) return nccl_fail(ncclReduceScatter(send, recv, count, ncclDouble, ncclSum, c.nccl, c.st), msg);
  int r;
  if ((r = local_enter(c, send, recv, msg))) return r;
  // own block of the sum; the in-place block (recv == send + rank*count) is read only here
  LocalGroup* g = c.lg;
  if (g->cap[c.rank] < (size_t)count) {
    if (g->scratch[c.rank]) cudaFree(g->scratch[c.rank]);
    cudaError_t e = cudaMalloc(&g->scratch[c.rank], sizeof(double) * count);
    if (e != cudaSuccess) return cuda_fail(e, msg);
    g->cap[c.rank] = count;
  }
  g_launches++;
  local_sum_kernel<<<blocks_for(count), 256, 0, c.st>>>(gather_ptrs(g, false), g->world, c.rank * count, count,
                                                        g->scratch[c.rank]);
  if ((r = local_leave(c, msg))) return r;
  return cuda_fail(cudaMemcpyAsync(recv, g->scratch[c.rank], sizeof(double) * count, cudaMemcpyDeviceToDevice, c.st),
                   msg);
}

int comm_all_gather(Comm& c, const double* send, double* recv, int64_t count, std::string* msg) {
  if (c.world == 1) return 0;
  if (!c.lg) return nccl_fail(ncclAllGather(send, recv, count, ncclDouble, c.nccl, c.st), msg);
  int r;
  if ((r = local_enter(c, send, recv, msg))) return r;
  LocalGroup* g = c.lg;
  for (int q = 0; q < g->world; q++) {
    double* d = recv + q * count;
    if (d == g->src[q] && q == c.rank) continue;  // in place
    cudaError_t e = cudaMemcpyAsync(d, g->src[q], sizeof(double) * count, cudaMemcpyDeviceToDevice, c.st);
    if (e != cudaSuccess) return cuda_fail(e, msg);
  }
  return local_leave(c, msg);
}

int comm_all_reduce(Comm& c, double* buf, int64_t count, std::string* msg) {
  if (c.world == 1) return 0;
  if (!c.lg) return nccl_fail(ncclAllReduce(buf, buf, count, ncclDouble, ncclSum, c.nccl, c.st), msg);
  int r;
  if ((r = local_enter(c, buf, buf, msg))) return r;
  LocalGroup* g = c.lg;
  if (g->cap[c.rank] < (size_t)count) {
    if (g->scratch[c.rank]) cudaFree(g->scratch[c.rank]);
    cudaError_t e = cudaMalloc(&g->scratch[c.rank], sizeof(double) * count);
    if (e != cudaSuccess) return cuda_fail(e, msg);
    g->cap[c.rank] = count;
  }
  g_launches++;
  local_sum_kernel<<<blocks_for(count), 256, 0, c.st>>>(gather_ptrs(g, false), g->world, 0, count,
                                                        g->scratch[c.rank]);
  if ((r = local_leave(c, msg))) return r;
  return cuda_fail(cudaMemcpyAsync(buf, g->scratch[c.rank], sizeof(double) * count, cudaMemcpyDeviceToDevice, c.st),
                   msg);
}

int comm_group_start(Comm& c, std::string* msg) {
  if (c.world == 1 || c.lg) return 0;
  return nccl_fail(ncclGroupStart(), msg);
}
int comm_group_end(Comm& c, std::string* msg) {
  if (c.world == 1 || c.lg) return 0;
  return nccl_fail(ncclGroupEnd(), msg);
}

}  // namespace cpd

namespace cpd {

int comm_split(const Comm& parent, int color, int key, Comm* out, std::string* msg) {
  *out = parent;
  if (parent.world == 1) return 0;
  if (parent.lg) {
    LocalGroup* ch = nullptr;
    int r = 0, w = 1;
    local_group_split(parent.lg, parent.rank, color, key, &ch, &r, &w);
    out->lg = ch;
    out->rank = r;
    out->world = w;
    out->nccl = nullptr;
    return 0;
  }
  ncclComm_t nc = nullptr;
  ncclResult_t e = ncclCommSplit(parent.nccl, color, key, &nc, nullptr);
  if (e != ncclSuccess) {
    if (msg) *msg = std::string("ncclCommSplit: ") + ncclGetErrorString(e);
    return 5;
  }
  int r = 0, w = 1;
  ncclCommUserRank(nc, &r);
  ncclCommCount(nc, &w);
  out->nccl = nc;
  out->lg = nullptr;
  out->rank = r;
  out->world = w;
  out->owns_nccl = true;
  return 0;
}

void comm_free(Comm& c) {
  if (c.owns_nccl && c.nccl) ncclCommDestroy(c.nccl);
  c.nccl = nullptr;
  c.owns_nccl = false;
}

}  // namespace cpd

namespace cpd {

// every rank of c learns every rank's `mine` (host pointer values; local group only)
int comm_exchange_ptr(Comm& c, void* mine, void** all, std::string* msg) {
  if (c.world == 1) {
    all[0] = mine;
    return 0;
  }
  if (!c.lg) {
    if (msg) *msg = "comm_exchange_ptr: local group only";
    return 4;
  }
  LocalGroup* g = c.lg;
  g->dst[c.rank] = static_cast<double*>(mine);
  g->barrier();
  for (int q = 0; q < g->world; q++) all[q] = g->dst[q];
  g->barrier();
  return 0;
}

// stream-ordered barrier: work enqueued on c.st before it is complete on every rank before any
// rank's later work runs (local group: events + host barrier; NCCL: a one-element all-reduce)
int comm_barrier(Comm& c, double* scratch1, std::string* msg) {
  if (c.world == 1) return 0;
  if (!c.lg) return nccl_fail(ncclAllReduce(scratch1, scratch1, 1, ncclDouble, ncclSum, c.nccl, c.st), msg);
  int r;
  if ((r = local_enter(c, nullptr, nullptr, msg))) return r;
  return local_leave(c, msg);
}

}  // namespace cpd
