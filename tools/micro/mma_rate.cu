// Microbenchmark: back-to-back tcgen05.mma throughput (SS and TS, M=128, N in {64,128,256}, K=16 bf16).
#include <cstdio>
#include "../../paper_2403_16161_b200/csrc/kernels/common.cuh"
using namespace vi;

template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) k_mma(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (128 * 64 + N * 64) / 8; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x3f803f80u, 0, 0, 0);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc(&tslot, 512);
  fence_proxy_async_smem();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(smem), b = a + 128 * 128;
    constexpr uint32_t idesc = idesc_bf16_f32(128, N);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (TS) umma_bf16_ts(tmem, tmem + 256 + k * 8, sdesc_k_sw128(b + k * 32), idesc, 1);
        else umma_bf16_ss(tmem, sdesc_k_sw128(a + k * 32), sdesc_k_sw128(b + k * 32), idesc, 1);
      }
    }
    long long t1 = clock64();
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t2 = clock64();
    out[blockIdx.x * 2] = t1 - t0;
    out[blockIdx.x * 2 + 1] = t2 - t0;
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <int N, bool TS>
void run(int blocks) {
  long long* d; cudaMalloc(&d, 2 * 148 * sizeof(long long));
  const int smem = 128 * 128 + N * 128 + 2048;
  cudaFuncSetAttribute(k_mma<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 2000;
  k_mma<N, TS><<<blocks, 128, smem>>>(d, iters);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[2 * 148]; cudaMemcpy(h, d, sizeof(long long) * 2 * blocks, cudaMemcpyDeviceToHost);
  printf("N=%3d %s blocks=%3d: %s  issue %.1f clk/mma, complete %.1f clk/mma (nominal %d)\n", N, TS ? "TS" : "SS", blocks,
         cudaGetErrorString(e), double(h[0]) / (iters * 4), double(h[1]) / (iters * 4), 128 * N / 256);
  cudaFree(d);
}

int main() {
  run<64, false>(1); run<128, false>(1); run<256, false>(1);
  run<128, true>(1); run<64, true>(1);
  run<128, false>(148); run<128, true>(148); run<256, false>(148);
  return 0;
}
