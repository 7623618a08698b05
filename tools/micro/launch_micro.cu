#include <cstdio>
#include "../../paper_2403_16161_b200/csrc/kernels/common.cuh"
using namespace vi;
__global__ void k_empty(int* p) { if (p && threadIdx.x == 9999) *p = 1; }
__global__ void k_smem(int* p) { extern __shared__ uint8_t s[]; if (threadIdx.x == 9999) *p = s[0]; }
__global__ void k_tmem(int* p) {
  __shared__ uint32_t slot;
  if (threadIdx.x < 32) tmem_alloc(&slot, 256);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc(slot, 256);
}
template <typename F> void time(const char* name, F f) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int i = 0; i < 5; ++i) f();
  cudaEventRecord(a);
  for (int i = 0; i < 100; ++i) f();
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("%-28s %.2f us/launch (%s)\n", name, ms * 10, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  cudaFuncSetAttribute(k_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  time("empty 1x256", [] { k_empty<<<1, 256>>>(nullptr); });
  time("empty 148x256", [] { k_empty<<<148, 256>>>(nullptr); });
  time("smem200K 1x256", [] { k_smem<<<1, 256, 200 * 1024>>>(nullptr); });
  time("smem200K 148x256", [] { k_smem<<<148, 256, 200 * 1024>>>(nullptr); });
  time("tmem 148x256", [] { k_tmem<<<148, 256>>>(nullptr); });
  time("alternate empty/smem", [] { k_empty<<<148, 256>>>(nullptr); k_smem<<<148, 256, 200 * 1024>>>(nullptr); });
  // CUDA graph of 100 empty launches
  cudaStream_t st; cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  for (int variant = 0; variant < 2; ++variant) {
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < 100; ++i) {
      if (variant == 0) k_empty<<<148, 256, 0, st>>>(nullptr);
      else k_smem<<<148, 256, 200 * 1024, st>>>(nullptr);
    }
    cudaStreamEndCapture(st, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, st); cudaStreamSynchronize(st);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a, st);
    for (int r = 0; r < 10; ++r) cudaGraphLaunch(ge, st);
    cudaEventRecord(b, st); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("graph of 100 %s: %.2f us per kernel (%s)\n", variant ? "smem200K" : "empty", ms * 1000 / 1000, cudaGetErrorString(cudaGetLastError()));
  }
  // PDL: programmatic stream serialization between launches
  {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(148); cfg.blockDim = dim3(256); cfg.stream = st;
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization; at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    time("pdl empty 148x256", [&] { cudaLaunchKernelEx(&cfg, k_empty, (int*)nullptr); });
  }
  return 0;
}
