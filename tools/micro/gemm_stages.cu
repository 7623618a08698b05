// TMA ring depth vs GEMM time on the memory-step shapes (C3: M = 3600; C3T1: M = 720).
// Each configuration is launched 50x back to back (PDL on); outputs compared with the
// 4-stage kernel's (same K order -> expected 0).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -I include -I paper_2403_16161_b200/csrc tools/micro/gemm_stages.cu -lcuda -o /tmp/gemm_stages
#include <cstdio>
#include <vector>

#include "../../paper_2403_16161_b200/csrc/kernels/gemm_tc.cu"
#include "../../paper_2403_16161_b200/csrc/kernels/setup.cu"
namespace vi { int g_pdl = 1; }
using namespace vi;

typedef CUresult (*PFN)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static PFN enc() {
  void* p; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  return (PFN)p;
}
static CUtensorMap tmap(void* base, uint64_t inner, uint64_t outer, uint32_t bi, uint32_t bo, bool f32 = false) {
  CUtensorMap m; cuuint64_t d[2] = {inner, outer}; cuuint64_t s[1] = {inner * (f32 ? 4 : 2)};
  cuuint32_t b[2] = {bi, bo}, e[2] = {1, 1};
  enc()(&m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, d, s, b, e,
        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return m;
}

__global__ void fill_kernel(uint16_t* p, size_t n, uint32_t seed) {
  for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    uint32_t h = uint32_t(i) * 2654435761u ^ seed;
    h ^= h >> 15; h *= 2246822519u; h ^= h >> 13;
    __nv_bfloat16 b = __float2bfloat16((float(h & 0xffff) / 65536.f - 0.5f) * 0.25f);
    p[i] = *reinterpret_cast<uint16_t*>(&b);
  }
}
__global__ void maxdiff_kernel(const float* a, const float* b, size_t n, float* out) {
  float m = 0.f;
  for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) m = fmaxf(m, fabsf(a[i] - b[i]));
  atomicMax(reinterpret_cast<int*>(out), __float_as_int(m));
}

typedef cudaError_t (*LFN)(const CUtensorMap&, const CUtensorMap&, int, int, int, int, const Epi&, cudaStream_t,
                           const CUtensorMap*, const CUtensorMap*, const CUtensorMap*);

static float* g_ref = nullptr;

static void run(const char* name, const char* cfgname, LFN fn, int M, int N, int K, int bn, int pair, int kind, bool ref) {
  uint16_t *A, *W; float *O, *bias, *x;
  cudaMalloc(&A, (size_t)M * K * 2); cudaMalloc(&W, (size_t)N * K * 2); cudaMalloc(&O, (size_t)M * N * 4);
  cudaMalloc(&bias, N * 4); cudaMalloc(&x, (size_t)M * N * 4);
  fill_kernel<<<512, 256>>>(A, (size_t)M * K, 1);
  fill_kernel<<<512, 256>>>(W, (size_t)N * K, 2);
  cudaMemset(bias, 0, N * 4); cudaMemset(x, 0, (size_t)M * N * 4); cudaMemset(O, 0, (size_t)M * N * 4);
  CUtensorMap ta = tmap(A, K, M, 64, 128), tb = tmap(W, K, N, 64, pair ? bn / 2 : bn);
  CUtensorMap to = tmap(O, N, M, 32, 32, true), tx = tmap(x, N, M, 32, 32, true);
  Epi e; memset(&e, 0, sizeof(e));
  e.kind = kind; e.M = M; e.N = N; e.bias = bias; e.out = O; e.ldo = N; e.out_f32 = 1; e.P = 1; e.S = 1;
  e.x_in = x; e.x_out = kind == EPI_RESID ? O : x;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaError_t err = fn(ta, tb, 0, M, N, K, e, 0, &to, kind == EPI_RESID ? &tx : nullptr, nullptr);
  cudaDeviceSynchronize();
  float diff = -1.f;
  if (err == cudaSuccess) {
    if (ref) {
      if (!g_ref) cudaMalloc(&g_ref, (size_t)M * N * 4);
      cudaMemcpy(g_ref, O, (size_t)M * N * 4, cudaMemcpyDeviceToDevice);
    }
    float* d; cudaMalloc(&d, 4); cudaMemset(d, 0, 4);
    maxdiff_kernel<<<256, 256>>>(O, g_ref, (size_t)M * N, d);
    cudaMemcpy(&diff, d, 4, cudaMemcpyDeviceToHost);
    cudaFree(d);
  }
  for (int i = 0; i < 3; ++i) fn(ta, tb, 0, M, N, K, e, 0, &to, kind == EPI_RESID ? &tx : nullptr, nullptr);
  const int it = 50;
  cudaEventRecord(a);
  for (int i = 0; i < it; ++i) fn(ta, tb, 0, M, N, K, e, 0, &to, kind == EPI_RESID ? &tx : nullptr, nullptr);
  cudaEventRecord(b);
  cudaError_t err2 = cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double us = ms * 1000 / it, tf = 2.0 * M * N * K / (us * 1e-6) / 1e12;
  printf("%-6s M=%-4d N=%-4d K=%-4d %-14s: %s/%s %7.2f us %5.0f TFLOP/s  maxdiff %g\n", name, M, N, K, cfgname,
         cudaGetErrorString(err), cudaGetErrorString(err2), us, tf, diff);
  fflush(stdout);
  cudaFree(A); cudaFree(W); cudaFree(O); cudaFree(bias); cudaFree(x);
}

int main() {
  struct S { const char* name; int M, N, K, kind; } shapes[] = {
      {"qkv", 3600, 1536, 512, EPI_STORE}, {"oproj", 3600, 512, 512, EPI_RESID}, {"ffn1", 3600, 1960, 512, EPI_STORE},
      {"ffn2", 3600, 512, 1960, EPI_RESID}, {"embed", 3600, 512, 6272, EPI_STORE}, {"back", 3600, 6272, 1024, EPI_STORE},
      {"qkv", 720, 1536, 512, EPI_STORE}, {"ffn1", 720, 1960, 512, EPI_STORE}, {"back", 720, 6272, 1024, EPI_STORE}};
  for (auto& s : shapes) {
    run(s.name, "128x128 s4", launch_cfg<128, 4, false, true>, s.M, s.N, s.K, 128, 0, s.kind, true);
    run(s.name, "128x128 s5", launch_cfg<128, 5, false, true>, s.M, s.N, s.K, 128, 0, s.kind, false);
    run(s.name, "128x256 s3", launch_cfg<256, 3, false, true>, s.M, s.N, s.K, 256, 0, s.kind, false);
    run(s.name, "pair256x128 s6", launch_cfg<128, 6, true, true>, s.M, s.N, s.K, 128, 1, s.kind, false);
    run(s.name, "pair256x256 s4", launch_cfg<256, 4, true, true>, s.M, s.N, s.K, 256, 1, s.kind, false);
    run(s.name, "pair256x256 s5", launch_cfg<256, 5, true, true>, s.M, s.N, s.K, 256, 1, s.kind, false);
    cudaFree(g_ref);
    g_ref = nullptr;
  }
  return 0;
}
