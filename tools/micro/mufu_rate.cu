// MUFU exp2 throughput on sm_100a: ex2.approx.ftz.f32 vs ex2.approx.f16x2 vs
// ex2.approx.ftz.bf16x2 (values per clock per SM), 16 warps per SM, independent chains.
#include <cstdint>
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_bf16.h>

template <int MODE>
__global__ void k(float* out, int iters) {
  uint32_t v[8];
  for (int i = 0; i < 8; ++i) v[i] = 0x3c003c00u ^ (threadIdx.x + i);
  float f[8];
  for (int i = 0; i < 8; ++i) f[i] = -0.001f * (threadIdx.x + i);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(f[i]));
      if (MODE == 1) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(v[i]));
      if (MODE == 2) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(v[i]));
    }
  }
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += f[i] + __uint_as_float(v[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    const double per_sm = 512.0 * iters * 8 * (MODE == 0 ? 1 : 2) / double(t1 - t0);
    printf("mode %d (%s): %.1f exp2 values / clk / SM\n", MODE, MODE == 0 ? "f32" : MODE == 1 ? "f16x2" : "bf16x2", per_sm);
  }
}

int main() {
  float* o;
  cudaMalloc(&o, 148 * 512 * 4);
  k<0><<<148, 512>>>(o, 4096);
  k<1><<<148, 512>>>(o, 4096);
  k<2><<<148, 512>>>(o, 4096);
  cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
