// Per-device launch setup shared by the kernels' host launchers.
//
// Function attributes (the > 48 KB dynamic shared memory opt-in) and occupancy queries are
// per DEVICE, and contexts of one process may live on different GPUs and be driven from
// different threads (the Refined model's online and refining inpainters, PAPER.md P:146;
// vi_tp_local_allgather across devices).  So every launcher asks here, keyed by (kernel,
// current device), under a mutex, instead of caching in a per-process static.
#include <map>
#include <mutex>
#include <utility>

#include "kernels.h"

namespace vi {

namespace {
std::mutex g_setup_mu;
std::map<std::pair<const void*, int>, int> g_done;      // (kernel, device) -> max active clusters (or 1)
}  // namespace

cudaError_t ensure_kernel_setup(const void* fn, int smem_bytes, int cluster, int block, int* max_clusters) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(g_setup_mu);
  auto it = g_done.find({fn, dev});
  if (it != g_done.end()) {
    if (max_clusters) *max_clusters = it->second;
    return cudaSuccess;
  }
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
  if (e != cudaSuccess) return e;
  int sms = 0;
  e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return e;
  int mc = sms / (cluster > 0 ? cluster : 1);
  if (cluster > 1) {
    cudaLaunchConfig_t q = {};
    q.gridDim = dim3(cluster * mc);
    q.blockDim = dim3(block);
    q.dynamicSmemBytes = smem_bytes;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cluster; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    q.attrs = at;
    q.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, fn, &q) == cudaSuccess && n > 0) mc = n;
    cudaGetLastError();
  }
  g_done[{fn, dev}] = mc;
  if (max_clusters) *max_clusters = mc;
  return cudaSuccess;
}

}  // namespace vi
