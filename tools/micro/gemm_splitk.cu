// Residual GEMM + LayerNorm at the C3 shapes, two ways, each launched 50x back to back (PDL on):
//   fused   : residual TMA-store epilogue (x_out = x_in + bias + A W^T), then layernorm_v4_kernel
//   split-K : ks fp32 partials (TMA store), then splitk_resid_kernel (sum in split order + bias
//             + x_in, LayerNorm written in the same pass)
// x_out and h of both ways are compared (max |diff|).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -I include -I paper_2403_16161_b200/csrc tools/micro/gemm_splitk.cu -lcuda -o /tmp/gemm_splitk
#include <cstdio>
#include <vector>

#include "../../paper_2403_16161_b200/csrc/kernels/gemm_tc.cu"
#include "../../paper_2403_16161_b200/csrc/kernels/rows.cu"
#include "../../paper_2403_16161_b200/csrc/kernels/setup.cu"
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
__global__ void fillf_kernel(float* p, size_t n, uint32_t seed) {
  for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    uint32_t h = uint32_t(i) * 2654435761u ^ seed;
    h ^= h >> 15; h *= 2246822519u; h ^= h >> 13;
    p[i] = float(h & 0xffff) / 65536.f - 0.5f;
  }
}
__global__ void maxdiff_kernel(const float* a, const float* b, size_t n, float* out) {
  float m = 0.f;
  for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) m = fmaxf(m, fabsf(a[i] - b[i]));
  atomicMax(reinterpret_cast<int*>(out), __float_as_int(m));
}
static float maxdiff(const float* a, const float* b, size_t n) {
  float* d; cudaMalloc(&d, 4); cudaMemset(d, 0, 4);
  maxdiff_kernel<<<256, 256>>>(a, b, n, d);
  float r; cudaMemcpy(&r, d, 4, cudaMemcpyDeviceToHost); cudaFree(d);
  return r;
}

typedef cudaError_t (*LFN)(const CUtensorMap&, const CUtensorMap&, int, int, int, int, const Epi&, cudaStream_t,
                           const CUtensorMap*, const CUtensorMap*, const CUtensorMap*);

struct Bufs {
  int M, N, K;
  uint16_t *A, *W, *W2;
  float *bias, *x0, *x, *ws, *g, *b, *h;
};

// one residual step + LN: x = x0 + bias + A W^T; h = LN(x) (fp32 h here, to compare exactly)
static float time_seq(const char* name, const char* cfg, Bufs& B, LFN fn, int bn, int pair, int ks, float* xref, float* href) {
  const int M = B.M, N = B.N, K = B.K, TM = pair ? 256 : 128, kpad = (M + 255) / 256 * 256;
  CUtensorMap ta = tmap(B.A, K, M, 64, 128), tb = tmap(B.W, K, N, 64, pair ? bn / 2 : bn);
  CUtensorMap tx0 = tmap(B.x0, N, M, 32, 32, true), tx = tmap(B.x, N, M, 32, 32, true);
  CUtensorMap tws = tmap(B.ws, N, (uint64_t)(ks > 1 ? ks : 1) * kpad, 32, 32, true);
  Epi e; memset(&e, 0, sizeof(e));
  e.M = M; e.N = N; e.P = 1; e.S = 1; e.out_f32 = 1;
  if (ks > 1) {
    e.kind = EPI_STORE; e.out = B.ws; e.ldo = N; e.ksplit = ks; e.kpad_rows = kpad;
  } else {
    e.kind = EPI_RESID; e.bias = B.bias; e.x_in = B.x0; e.x_out = B.x;
  }
  (void)TM;
  auto once = [&]() -> cudaError_t {
    cudaError_t err;
    if (ks > 1) {
      err = fn(ta, tb, 0, M, N, K, e, 0, &tws, nullptr, nullptr);
      if (err != cudaSuccess) return err;
      return launch_splitk_resid(B.ws, ks, (size_t)kpad * N, B.bias, B.x0, B.x, nullptr, 1, B.g, B.b, B.h, 1, M, N, 0, nullptr);
    }
    err = fn(ta, tb, 0, M, N, K, e, 0, &tx, &tx0, nullptr);   // residual: output map x, x_in map x0
    if (err != cudaSuccess) return err;
    return launch_layernorm(B.x, B.g, B.b, B.h, 1, M, N, 0);
  };
  cudaError_t err = once();
  cudaDeviceSynchronize();
  float dx = -1, dh = -1;
  if (xref) {
    if (!href) {
    } else {
      dx = maxdiff(B.x, xref, (size_t)M * N);
      dh = maxdiff(B.h, href, (size_t)M * N);
    }
  }
  for (int i = 0; i < 3; ++i) once();
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int it = 50;
  cudaEventRecord(a);
  for (int i = 0; i < it; ++i) once();
  cudaEventRecord(b);
  cudaError_t err2 = cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double us = ms * 1000 / it;
  printf("%-6s M=%-4d N=%-4d K=%-4d %-22s: %s/%s %7.2f us (GEMM + LN)  maxdiff x %g h %g\n", name, M, N, K, cfg,
         cudaGetErrorString(err), cudaGetErrorString(err2), us, dx, dh);
  fflush(stdout);
  return float(us);
}

int main() {
  struct S { const char* name; int M, N, K; } shapes[] = {
      {"oproj", 3600, 512, 512}, {"ffn2", 3600, 512, 1960}, {"embed", 3600, 512, 6272},
      {"oproj", 720, 512, 512}, {"ffn2", 720, 512, 1960}};
  for (auto& s : shapes) {
    Bufs B; B.M = s.M; B.N = s.N; B.K = s.K;
    const size_t MN = (size_t)s.M * s.N;
    cudaMalloc(&B.A, (size_t)s.M * s.K * 2); cudaMalloc(&B.W, (size_t)s.N * s.K * 2);
    cudaMalloc(&B.bias, s.N * 4); cudaMalloc(&B.x0, MN * 4); cudaMalloc(&B.x, MN * 4);
    cudaMalloc(&B.ws, 8 * (size_t)((s.M + 255) / 256 * 256) * s.N * 4);
    cudaMalloc(&B.g, s.N * 4); cudaMalloc(&B.b, s.N * 4); cudaMalloc(&B.h, MN * 4);
    fill_kernel<<<512, 256>>>(B.A, (size_t)s.M * s.K, 1);
    fill_kernel<<<512, 256>>>(B.W, (size_t)s.N * s.K, 2);
    fillf_kernel<<<512, 256>>>(B.x0, MN, 3);
    fillf_kernel<<<64, 256>>>(B.bias, s.N, 4);
    fillf_kernel<<<64, 256>>>(B.g, s.N, 5);
    fillf_kernel<<<64, 256>>>(B.b, s.N, 6);
    float *xr, *hr; cudaMalloc(&xr, MN * 4); cudaMalloc(&hr, MN * 4);
    time_seq(s.name, "128x128 resid (ref)", B, launch_cfg<128, 4, false, true>, 128, 0, 1, nullptr, nullptr);
    cudaMemcpy(xr, B.x, MN * 4, cudaMemcpyDeviceToDevice); cudaMemcpy(hr, B.h, MN * 4, cudaMemcpyDeviceToDevice);
    time_seq(s.name, "pair256x128 resid", B, launch_cfg<128, 6, true, true>, 128, 1, 1, xr, hr);
    for (int ks = 2; ks <= 4; ++ks) {
      char nm[64];
      snprintf(nm, sizeof nm, "128x128 splitK %d", ks);
      time_seq(s.name, nm, B, launch_cfg<128, 4, false, true>, 128, 0, ks, xr, hr);
      snprintf(nm, sizeof nm, "pair256x128 splitK %d", ks);
      time_seq(s.name, nm, B, launch_cfg<128, 6, true, true>, 128, 1, ks, xr, hr);
      snprintf(nm, sizeof nm, "pair256x256 splitK %d", ks);
      time_seq(s.name, nm, B, launch_cfg<256, 4, true, true>, 256, 1, ks, xr, hr);
    }
    cudaFree(B.A); cudaFree(B.W); cudaFree(B.bias); cudaFree(B.x0); cudaFree(B.x); cudaFree(B.ws);
    cudaFree(B.g); cudaFree(B.b); cudaFree(B.h); cudaFree(xr); cudaFree(hr);
  }
  return 0;
}
