// Peer addresses of a registered NCCL window (the fused reduce-scatter epilogue):
// the receive buffers of the ranks of one communicator are allocated with ncclMemAlloc and
// registered as a symmetric window; ncclGetPeerPointer (NCCL 2.28 device API, load/store
// accessible = NVLink peers of one node) gives each rank's flat address of every peer's buffer,
// which the mTTV / PP-stream epilogue then stores into directly.
#include <nccl.h>
#include <nccl_device.h>

#include "comm.h"
#include "kernels.h"

namespace cpd {
namespace {
__global__ void peer_ptrs_kernel(ncclWindow_t w, int n, void** out) {
  for (int q = threadIdx.x; q < n; q += blockDim.x) out[q] = ncclGetPeerPointer(w, 0, q);
}
}  // namespace

int nccl_window_peers(ncclComm_t comm, size_t bytes, int nranks, void** buf, void** peers, void** win_out,
                      cudaStream_t st, std::string* msg) {
  auto nf = [&](ncclResult_t r, const char* what) {
    if (r == ncclSuccess) return 0;
    if (msg) *msg = std::string(what) + ": " + ncclGetErrorString(r);
    return 5;
  };
  int r;
  if ((r = nf(ncclMemAlloc(buf, bytes), "ncclMemAlloc"))) return r;
  ncclWindow_t w = nullptr;
  if ((r = nf(ncclCommWindowRegister(comm, *buf, bytes, &w, NCCL_WIN_COLL_SYMMETRIC), "ncclCommWindowRegister")))
    return r;
  *win_out = (void*)w;
  void** d = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&d, sizeof(void*) * nranks, st);
  if (e == cudaSuccess) {
    g_launches++;
    peer_ptrs_kernel<<<1, 32, 0, st>>>(w, nranks, d);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpyAsync(peers, d, sizeof(void*) * nranks, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (d) cudaFreeAsync(d, st);
  if (e != cudaSuccess) {
    if (msg) *msg = std::string("peer pointers: ") + cudaGetErrorString(e);
    return 4;
  }
  return 0;
}

void nccl_window_free(ncclComm_t comm, void* buf, void* win) {
  if (win) ncclCommWindowDeregister(comm, (ncclWindow_t)win);
  if (buf) ncclMemFree(buf);
}

}  // namespace cpd
