// Standalone timing of the small-chunk attention (attn.cu: attn_tc2 KV split + combine) at
// the C3T1 shape: 720 queries (one frame) x 7920 keys (11 ring slots of 720 tokens), 4 heads,
// d = 128, the engine's split (11 splits of 6 key tiles).  Prints the mean time of the split
// kernel alone, the combine alone and the pair, back-to-back launches (L2 warm).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo --expt-relaxed-constexpr \
//        -I include -I paper_2403_16161_b200/csrc -I paper_2403_16161_b200/csrc/kernels \
//        tools/micro/tc2_micro.cu -lcuda -o /tmp/tc2_micro
//   /tmp/tc2_micro [iters] [nsplit (0 = engine's)]
#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#define TC2_TRACE 1

#ifndef TC2_SRC
#define TC2_SRC "../../paper_2403_16161_b200/csrc/kernels/attn.cu"
#endif
#include TC2_SRC
#include "../../paper_2403_16161_b200/csrc/kernels/setup.cu"
namespace vi {
int g_pdl = 1;
}
using namespace vi;

typedef CUresult (*PFN)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static PFN enc() {
  void* p;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  return (PFN)p;
}
static CUtensorMap tmap(void* base, uint64_t inner, uint64_t outer, uint32_t bi, uint32_t bo) {
  CUtensorMap m;
  cuuint64_t d[2] = {inner, outer};
  cuuint64_t s[1] = {inner * 2};
  cuuint32_t b[2] = {bi, bo}, e[2] = {1, 1};
  enc()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, d, s, b, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return m;
}

__global__ void fill_kernel(uint16_t* p, size_t n, uint32_t seed, float scale) {
  for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    uint32_t h = uint32_t(i) * 2654435761u ^ seed;
    h ^= h >> 15; h *= 2246822519u; h ^= h >> 13;
    const float f = (float(h & 0xffff) / 65536.f - 0.5f) * scale;
    __nv_bfloat16 b = __float2bfloat16(f);
    p[i] = *reinterpret_cast<uint16_t*>(&b);
  }
}

// L2 read-bandwidth probe: sum of n float4 (grid-stride), one value per block written
__global__ void read_probe(const float4* __restrict__ p, size_t n, float* out) {
  float acc = 0.f;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const float4 v = __ldcg(p + i);
    acc += v.x + v.y + v.z + v.w;
  }
  if (acc == 12345.f) out[blockIdx.x] = acc;
}

int main(int argc, char** argv) {
  const int iters = argc > 1 ? atoi(argv[1]) : 200;
  const int force_split = argc > 2 ? atoi(argv[2]) : 0;
  const int Nq = 720, H = 4, HD = 128, D = H * HD, SP = 11 * 720, vt_ld = (SP + 63) / 64 * 64;
  uint16_t *q, *k, *vt, *o;
  cudaMalloc(&q, (size_t)Nq * D * 2);
  cudaMalloc(&k, (size_t)SP * D * 2);
  cudaMalloc(&vt, (size_t)D * vt_ld * 2);
  cudaMalloc(&o, (size_t)Nq * D * 2);
  fill_kernel<<<1024, 256>>>(q, (size_t)Nq * D, 1, 4.f);
  fill_kernel<<<1024, 256>>>(k, (size_t)SP * D, 2, 4.f);
  fill_kernel<<<1024, 256>>>(vt, (size_t)D * vt_ld, 3, 2.f);
  CUtensorMap tq = tmap(q, D, Nq, 64, 128), tk = tmap(k, D, SP, 64, 128), tv = tmap(vt, vt_ld, D, 64, HD);
  AttnTC a;
  memset(&a, 0, sizeof(a));
  a.Nq = Nq; a.hd = HD; a.D = D; a.H = H;
  a.scale_log2 = 1.4426950408889634f / sqrtf(float(HD));
  a.segs.n = 1; a.segs.len[0] = SP; a.segs.tile0[1] = (SP + 127) / 128;
  a.o = reinterpret_cast<bf16*>(o); a.o_ld = D; a.o_hs = HD;
  const int ntiles = a.segs.tile0[1], units = ((Nq + 255) / 256) * H;
  // engine.cu choose_split
  double best = 1e30;
  int ns = 1, tps = ntiles;
  for (int s = 1; s <= 16 && s <= ntiles; ++s) {
    const int t = (ntiles + s - 1) / s;
    const int waves = (units * s + 147) / 148;
    const double cost = double(waves) * (t + 4.0) + (s > 1 ? 1.0 + 0.3 * s : 0.0);
    if (cost < best - 1e-9) { best = cost; ns = s; tps = t; }
  }
  if (force_split > 0) { ns = force_split; tps = (ntiles + ns - 1) / ns; }
  a.tiles_per_split = tps;
  a.nsplit = (ntiles + tps - 1) / tps;
  cudaMalloc(&a.opart, (size_t)16 * Nq * D * 2);
  cudaMalloc(&a.lse, (size_t)16 * H * Nq * 4);
  cudaStream_t st;
  cudaStreamCreate(&st);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](int which) {
    for (int i = 0; i < 5; ++i) {
      if (which & 1) launch_attn_tc2(tq, tk, tv, a, st);
      if (which & 2) launch_attn_combine(a, st);
    }
    cudaEventRecord(e0, st);
    for (int i = 0; i < iters; ++i) {
      if (which & 1) launch_attn_tc2(tq, tk, tv, a, st);
      if (which & 2) launch_attn_combine(a, st);
    }
    cudaEventRecord(e1, st);
    cudaError_t err = cudaStreamSynchronize(st);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    return std::make_pair(1e3 * ms / iters, err);
  };
  const double flop = 4.0 * Nq * SP * D;
  const char* nm[4] = {"", "tc2", "combine", "tc2+combine"};
  for (int w = 1; w <= 3; ++w) {
    auto r = run(w);
    printf("C3T1 nsplit %d x %d tiles, grid %d: %-12s %7.2f us  (%.0f TFLOP/s on the pair) %s\n", a.nsplit,
           a.tiles_per_split, units * a.nsplit, nm[w], r.first, w == 3 ? flop / (r.first * 1e-6) / 1e12 : 0.0,
           cudaGetErrorString(r.second));
  }
  {   // L2 read probe over the partials (nsplit x Nq x D bf16)
    float* dummy;
    cudaMalloc(&dummy, 1 << 20);
    const size_t n4 = (size_t)a.nsplit * Nq * D / 8;   // bf16 partials
    for (int blocks : {148, 296, 592, 1184}) {
      for (int i = 0; i < 3; ++i) read_probe<<<blocks, 512, 0, st>>>((const float4*)a.opart, n4, dummy);
      cudaEventRecord(e0, st);
      for (int i = 0; i < 100; ++i) read_probe<<<blocks, 512, 0, st>>>((const float4*)a.opart, n4, dummy);
      cudaEventRecord(e1, st);
      cudaStreamSynchronize(st);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("read probe %d x 512: %.2f us for %.1f MB (%.0f GB/s)\n", blocks, ms * 10.f, n4 * 16 / 1e6,
             n4 * 16 / (ms * 1e-5) / 1e9);
    }
  }
  {   // checksum of the merged output
    std::vector<uint16_t> ho((size_t)Nq * D);
    cudaMemcpy(ho.data(), o, ho.size() * 2, cudaMemcpyDeviceToHost);
    unsigned long long hs = 1469598103934665603ull;
    for (uint16_t x : ho) hs = (hs ^ x) * 1099511628211ull;
    printf("output hash %016llx\n", hs);
  }
  if (getenv("CTA_TRACE")) {   // per-CTA stamps of one launch (after a warm launch)
    const int grid = units * a.nsplit;
    long long* ctb;
    cudaMalloc(&ctb, (size_t)grid * 8 * 8);
    cudaMemset(ctb, 0, (size_t)grid * 8 * 8);
    launch_attn_tc2(tq, tk, tv, a, st);
    a.cta_trace = ctb;
    launch_attn_tc2(tq, tk, tv, a, st);
    cudaStreamSynchronize(st);
    a.cta_trace = nullptr;
    std::vector<long long> h((size_t)grid * 8);
    cudaMemcpy(h.data(), ctb, h.size() * 8, cudaMemcpyDeviceToHost);
    long long t0 = LLONG_MAX;
    for (int c = 0; c < grid; ++c) t0 = std::min(t0, h[c * 8]);
    printf("cta: entry waited firstS ofinal epi_done exit spun (ns from the first entry)\n");
    double acc[7] = {0, 0, 0, 0, 0, 0, 0};
    for (int c = 0; c < grid; ++c) {
      const long long* e = &h[c * 8];
      if (c < 24 || c % 16 == 0) {
        printf("%3d:", c);
        for (int i = 0; i < 7; ++i) printf(" %6lld", e[i] ? e[i] - t0 : -1);
        printf("\n");
      }
      for (int i = 0; i < 7; ++i) acc[i] += double(e[i] ? e[i] - t0 : 0) / grid;
    }
    printf("mean:");
    for (int i = 0; i < 7; ++i) printf(" %6.0f", acc[i]);
    printf("\n");
  }
  return 0;
}
