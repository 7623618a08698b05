// SIMT fp32 GEMM for the fp32 parity path (BASELINE configs[0], tolerance 1e-4):
// TF32 tensor cores would give ~5e-4 error, so this is plain FFMA with a 64x64 CTA
// tile, 16-deep K slices in shared memory and a 4x4 register tile per thread.
#include "kernels.h"

namespace vi {

__global__ void __launch_bounds__(256) gemm_simt_f32_kernel(const float* __restrict__ A, const float* __restrict__ W,
                                                           int M, int N, int K, Epi e) {
  __shared__ float As[16][64 + 4];
  __shared__ float Ws[16][64 + 4];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int m0 = blockIdx.x * 64, n0 = blockIdx.y * 64;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += 16) {
    for (int i = threadIdx.x; i < 64 * 16; i += 256) {
      const int r = i / 16, c = i % 16;
      const int m = m0 + r, n = n0 + r, k = k0 + c;
      As[c][r] = (m < M && k < K) ? A[(size_t)m * K + k] : 0.f;
      Ws[c][r] = (n < N && k < K) ? W[(size_t)n * K + k] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        a[i] = As[kk][ty * 4 + i];
        b[i] = Ws[kk][tx * 4 + i];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int m = m0 + ty * 4 + i, n = n0 + tx * 4 + j;
      if (m < M && n < N) epi_one<float>(e, m, n, acc[i][j]);
    }
}

cudaError_t launch_gemm_simt_f32(const float* A, const float* W, int M, int N, int K, const Epi& e, cudaStream_t st) {
  dim3 grid((M + 63) / 64, (N + 63) / 64);
  gemm_simt_f32_kernel<<<grid, 256, 0, st>>>(A, W, M, N, K, e);
  return cudaGetLastError();
}

}  // namespace vi
