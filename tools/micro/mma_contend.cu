// Does concurrent tcgen05.ld/st traffic from softmax-like warps slow down tcgen05.mma?
#include <cstdio>
#include "../../paper_2403_16161_b200/csrc/kernels/common.cuh"
using namespace vi;

template <bool TS, int LDMODE>   // LDMODE 0: none, 1: ld loop, 2: ld+st loop
__global__ void __launch_bounds__(384, 1) k(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  __shared__ volatile int done;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (128 * 128 * 2) / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x3f803f80u, 0, 0, 0);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); done = 0; }
  if (warp == 0) tmem_alloc(&tslot, 512);
  fence_proxy_async_smem();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp == 8 && (threadIdx.x & 31) == 0) {
    const uint32_t a = smem_u32(smem), b = a + 128 * 128;
    constexpr uint32_t idesc = idesc_bf16_f32(128, 128);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        if (TS) umma_bf16_ts(tmem, tmem + 128 + kk * 8, sdesc_k_sw128(b + kk * 32), idesc, 1);
        else umma_bf16_ss(tmem, sdesc_k_sw128(a + kk * 32), sdesc_k_sw128(b + kk * 32), idesc, 1);
      }
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t2 = clock64();
    out[0] = t2 - t0;
    done = 1;
  } else if (warp < 8 && LDMODE) {
    const uint32_t base = tmem + 256 + ((warp & 3) * 32 << 16) + (warp >> 2) * 128;
    long long n = 0;
    while (!done) {
      uint32_t r[32];
      tmem_ld32(base, r);
      tmem_wait_ld();
      if (LDMODE == 2) { tmem_st32(base + 64, r); tmem_wait_st(); }
      ++n;
    }
    if (threadIdx.x == 0) out[1] = n;
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <bool TS, int M>
void run() {
  long long* d; cudaMalloc(&d, 16 * sizeof(long long)); cudaMemset(d, 0, 16 * sizeof(long long));
  const int smem = 2 * 128 * 128 + 2048;
  cudaFuncSetAttribute(k<TS, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 2000;
  k<TS, M><<<1, 384, smem>>>(d, iters);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[2]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("%s ldmode=%d: %s  %.1f clk/mma; ld iterations per warp0 %lld (%.1f clk per 32-col ld)\n", TS ? "TS" : "SS", M,
         cudaGetErrorString(e), double(h[0]) / (iters * 4), h[1], h[1] ? double(h[0]) / h[1] : 0.0);
}
int main() { run<false, 0>(); run<false, 1>(); run<false, 2>(); run<true, 0>(); run<true, 1>(); run<true, 2>(); }
