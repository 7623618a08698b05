// Standalone timing + cross-check of the tcgen05 GEMM kernel (gemm_tc.cu) on the memory-step
// shapes: single-CTA vs CTA-pair (2-SM MMA) tiles, register-direct vs TMA-store epilogue.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -I include -I paper_2403_16161_b200/csrc tools/micro/gemm_micro.cu -lcuda -o /tmp/gemm_micro
//
// Every configuration's fp32 output (EPI_STORE, random bf16 operands) is compared with the
// single-CTA BN=128 kernel's (max |diff|; identical K order -> expected 0).
#include <cstdio>
#include <vector>

#include "../../paper_2403_16161_b200/csrc/kernels/gemm_tc.cu"
namespace vi { int g_pdl = 1; }
using namespace vi;
#ifdef VI_GEMM_TRACE
static void* g_gemm_trace_ptr() { void* p; cudaGetSymbolAddress(&p, g_gemm_trace); return p; }
#endif

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

static float* g_ref = nullptr;

// te: TMA-store epilogue (fp32 output map); pair: CTA-pair tiles
static void run(const char* name, int M, int N, int K, int bn, int kind, int pair, bool te, bool ref = false) {
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
  const CUtensorMap* pto = te ? &to : nullptr;
  const CUtensorMap* ptx = (te && kind == EPI_RESID) ? &tx : nullptr;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaError_t err = launch_gemm_tc(ta, tb, 0, M, N, K, bn, e, 0, pair, pto, ptx);
  cudaDeviceSynchronize();
  float diff = -1.f;
  if (err == cudaSuccess && kind == EPI_STORE) {
    if (ref) {
      if (!g_ref) cudaMalloc(&g_ref, (size_t)M * N * 4);
      cudaMemcpy(g_ref, O, (size_t)M * N * 4, cudaMemcpyDeviceToDevice);
    }
    float* d; cudaMalloc(&d, 4); cudaMemset(d, 0, 4);
    maxdiff_kernel<<<256, 256>>>(O, g_ref, (size_t)M * N, d);
    cudaMemcpy(&diff, d, 4, cudaMemcpyDeviceToHost);
    cudaFree(d);
  }
  for (int i = 0; i < 3; ++i) launch_gemm_tc(ta, tb, 0, M, N, K, bn, e, 0, pair, pto, ptx);
  const int it = 50;
  cudaEventRecord(a);
  for (int i = 0; i < it; ++i) launch_gemm_tc(ta, tb, 0, M, N, K, bn, e, 0, pair, pto, ptx);
  cudaEventRecord(b);
  cudaError_t err2 = cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double us = ms * 1000 / it, tf = 2.0 * M * N * K / (us * 1e-6) / 1e12;
  printf("%-6s M=%d N=%d K=%d BN=%d epi=%d pair=%d te=%d: %s/%s %.2f us %5.0f TFLOP/s  maxdiff vs single-128 %g\n", name, M,
         N, K, bn, kind, pair, int(te), cudaGetErrorString(err), cudaGetErrorString(err2), us, tf, diff);
  fflush(stdout);
#ifdef VI_GEMM_TRACE
  long long tr[64];
  cudaMemcpyFromSymbol(tr, g_gemm_trace, sizeof(tr));
  printf("   CTA0 (ns from start): setup %lld first-data %lld | mma-done", tr[1] - tr[0], tr[2] - tr[0]);
  for (int i = 0; i < 4; ++i) printf(" %lld", tr[3 + i] > tr[0] ? tr[3 + i] - tr[0] : -1);
  printf(" | epi end");
  for (int i = 0; i < 4; ++i) printf(" %lld", tr[11 + i] > tr[0] ? tr[11 + i] - tr[0] : -1);
  printf(" | exit %lld\n", tr[15] - tr[0]);
  printf("   epilogue warp 0, tile 0 chunks (start / tmem ld / smem written / store issued):");
  for (int k = 0; k < 8 && tr[16 + 4 * k]; ++k)
    printf(" [%lld %lld %lld %lld]", tr[16 + 4 * k] - tr[0], tr[17 + 4 * k] - tr[0], tr[18 + 4 * k] - tr[0], tr[19 + 4 * k] - tr[0]);
  printf("\n");
  cudaMemset(g_gemm_trace_ptr(), 0, sizeof(tr));
#endif
  cudaFree(A); cudaFree(W); cudaFree(O); cudaFree(bias); cudaFree(x);
}

int main(int argc, char** argv) {
  // the memory step's GEMMs at C3 (M = 3600 rows = 5 frames x 720 tokens)
  struct S { const char* name; int N, K, kind; } shapes[] = {
      {"qkv", 1536, 512, EPI_STORE}, {"oproj", 512, 512, EPI_RESID}, {"ffn1", 1960, 512, EPI_STORE},
      {"ffn2", 512, 1960, EPI_RESID}, {"embed", 512, 6272, EPI_STORE}, {"back", 6272, 1024, EPI_STORE}};
  for (auto& sh : shapes) {
    run(sh.name, 3600, sh.N, sh.K, 128, EPI_STORE, 0, true, true);     // reference output
    run(sh.name, 3600, sh.N, sh.K, 256, EPI_STORE, 0, true);
    run(sh.name, 3600, sh.N, sh.K, 128, EPI_STORE, 1, true);
    run(sh.name, 3600, sh.N, sh.K, 256, EPI_STORE, 1, true);
    run(sh.name, 3600, sh.N, sh.K, 256, EPI_STORE, 1, false);
    if (sh.kind == EPI_RESID) {
      run(sh.name, 3600, sh.N, sh.K, 128, EPI_RESID, 0, true);
      run(sh.name, 3600, sh.N, sh.K, 128, EPI_RESID, 1, true);
      run(sh.name, 3600, sh.N, sh.K, 256, EPI_RESID, 1, true);
    }
    cudaFree(g_ref);
    g_ref = nullptr;
  }
  return 0;
}
