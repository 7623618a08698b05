// Standalone timing of the tcgen05 GEMM kernel (gemm_tc.cu) on the memory-step shapes.
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
static CUtensorMap tmap(void* base, uint64_t inner, uint64_t outer, uint32_t bi, uint32_t bo) {
  CUtensorMap m; cuuint64_t d[2] = {inner, outer}; cuuint64_t s[1] = {inner * 2}; cuuint32_t b[2] = {bi, bo}, e[2] = {1, 1};
  enc()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, d, s, b, e, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return m;
}

static void run(const char* name, int M, int N, int K, int bn, int kind, int cl = 0) {
  void *A, *W, *O; float *bias, *x;
  cudaMalloc(&A, (size_t)M * K * 2); cudaMalloc(&W, (size_t)N * K * 2); cudaMalloc(&O, (size_t)M * N * 4);
  cudaMalloc(&bias, N * 4); cudaMalloc(&x, (size_t)M * N * 4);
  cudaMemset(A, 0, (size_t)M * K * 2); cudaMemset(W, 0, (size_t)N * K * 2); cudaMemset(bias, 0, N * 4); cudaMemset(x, 0, (size_t)M * N * 4);
  const int CMs[8] = {1, 2, 1, 2, 1, 2, 1, 4}, CNs[8] = {1, 1, 2, 2, 4, 4, 8, 2};
  const int CM = CMs[cl], CN = CNs[cl];
  CUtensorMap ta = tmap(A, K, M, 64, 128 / CN), tb = tmap(W, K, N, 64, bn / CM);
  Epi e; memset(&e, 0, sizeof(e));
  e.kind = kind; e.M = M; e.N = N; e.bias = bias; e.out = O; e.ldo = N; e.P = 1; e.S = 1; e.x_in = x; e.x_out = x;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) launch_gemm_tc(ta, tb, 0, M, N, K, bn, e, 0, cl);
  const int it = 50;
  cudaEventRecord(a);
  for (int i = 0; i < it; ++i) launch_gemm_tc(ta, tb, 0, M, N, K, bn, e, 0, cl);
  cudaEventRecord(b);
  cudaError_t err = cudaEventSynchronize(b);

  float ms; cudaEventElapsedTime(&ms, a, b);
  const double us = ms * 1000 / it, tf = 2.0 * M * N * K / (us * 1e-6) / 1e12;
  printf("%-8s M=%d N=%d K=%d BN=%d epi=%d cl=%d: %s %.2f us  %.0f TFLOP/s\n", name, M, N, K, bn, kind, cl, cudaGetErrorString(err), us, tf);
#ifdef VI_GEMM_TRACE
  long long tr[24];
  cudaMemcpyFromSymbol(tr, g_gemm_trace, sizeof(tr));
  printf("   CTA0 (ns from start): setup %lld first-data %lld | mma-done", tr[1] - tr[0], tr[2] - tr[0]);
  for (int i = 0; i < 4; ++i) printf(" %lld", tr[3 + i] > tr[0] ? tr[3 + i] - tr[0] : -1);
  printf(" | epi start");
  for (int i = 0; i < 4; ++i) printf(" %lld", tr[7 + i] > tr[0] ? tr[7 + i] - tr[0] : -1);
  printf(" | epi end");
  for (int i = 0; i < 4; ++i) printf(" %lld", tr[11 + i] > tr[0] ? tr[11 + i] - tr[0] : -1);
  printf(" | exit %lld\n", tr[15] - tr[0]);
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
    for (int bn : {128, 256}) {
      run(sh.name, 3600, sh.N, sh.K, bn, EPI_NONE, 0);
      run(sh.name, 3600, sh.N, sh.K, bn, sh.kind, 0);
      for (int cl : {1, 2, 3})
        run(sh.name, 3600, sh.N, sh.K, bn, sh.kind, cl);
    }
  }
  return 0;
}
