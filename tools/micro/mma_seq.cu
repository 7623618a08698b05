// Microbenchmark: the attention kernel's tcgen05.mma sequence with DISTINCT operands per K step
// (as attn_sk2 issues it): per key tile, PV(t) = 8 TS MMAs (A = P from TMEM, B = V^T slices)
// then QK(t) = 8 SS MMAs (A = Q_t, B = K slices, 128 x 128 x 16 each), t = 0, 1; 148 CTAs.
// MODE 0: the full PV/QK sequence; 1: QK only (SS); 2: PV only (TS); 3: QK with N = 256 (SS,
// one Q tile, two key tiles at once).
#include <cstdio>
#include "../../paper_2403_16161_b200/csrc/kernels/common.cuh"
using namespace vi;

template <int MODE>
__global__ void __launch_bounds__(128, 1) k_seq(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 192 * 1024 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x3f803f80u ^ i, 0x3f80u, 0x3c00u, 0);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc(&tslot, 512);
  fence_proxy_async_smem();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint32_t q0 = smem_u32(smem), k0 = q0 + 65536, v0 = k0 + 65536;
    constexpr uint32_t is = idesc_bf16_f32(128, 128), is256 = idesc_bf16_f32(128, 256);
    const uint64_t dq = sdesc_k_sw128(q0), dk = sdesc_k_sw128(k0), dv = sdesc_k_sw128(v0);
    long long t0 = clock64();
    int n = 0;
    for (int it = 0; it < iters; ++it) {
      const int st = it & 1;
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        if (MODE == 0 || MODE == 2) {
#pragma unroll
          for (int hh = 0; hh < 2; ++hh)
#pragma unroll
            for (int k4 = 0; k4 < 4; ++k4, ++n)
              umma_bf16_ts(tmem + 256 + t * 128, tmem + t * 128 + hh * 64 + k4 * 8,
                           dv + uint64_t((st * 32768 + hh * 16384 + k4 * 32) >> 4), is, 1);
        }
        if (MODE == 0 || MODE == 1) {
#pragma unroll
          for (int kk = 0; kk < 8; ++kk, ++n) {
            const uint64_t off = uint64_t(((kk >> 2) * 16384 + (kk & 3) * 32) >> 4);
            umma_bf16_ss(tmem + t * 128, dq + uint64_t((t * 32768) >> 4) + off, dk + uint64_t((st * 32768) >> 4) + off, is,
                         kk > 0);
          }
        }
        if (MODE == 3 && t == 0) {
#pragma unroll
          for (int kk = 0; kk < 8; ++kk, n += 2) {
            const uint64_t off = uint64_t(((kk >> 2) * 16384 + (kk & 3) * 32) >> 4);
            umma_bf16_ss(tmem, dq + off, dk + off, is256, kk > 0);   // B: 256 key rows (both K stages)
          }
        }
      }
    }
    long long t1 = clock64();
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t2 = clock64();
    out[blockIdx.x * 3] = t1 - t0;
    out[blockIdx.x * 3 + 1] = t2 - t0;
    out[blockIdx.x * 3 + 2] = n;
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <int MODE>
void run(int blocks) {
  long long* d; cudaMalloc(&d, 3 * 148 * sizeof(long long));
  const int smem = 192 * 1024 + 2048;
  cudaFuncSetAttribute(k_seq<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 500;
  k_seq<MODE><<<blocks, 128, smem>>>(d, iters);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[3 * 148]; cudaMemcpy(h, d, sizeof(long long) * 3 * blocks, cudaMemcpyDeviceToHost);
  const char* nm[] = {"PV+QK seq", "QK only (SS)", "PV only (TS)", "QK N=256 (SS)"};
  printf("%-14s blocks=%3d: %s  %.1f clk per 128x128x16 MMA-equivalent (nominal 64)\n", nm[MODE], blocks,
         cudaGetErrorString(e), double(h[1]) / double(h[2]));
  cudaFree(d);
}

int main() {
  run<0>(1); run<1>(1); run<2>(1); run<3>(1);
  run<0>(148); run<1>(148); run<2>(148); run<3>(148);
  return 0;
}
