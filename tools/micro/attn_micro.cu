// Standalone timing of the stream-K memory attention (attn_sk2.cu) at the C3 shape:
// 3600 queries x 10800 keys (15 full ring slots of 720 tokens), 4 heads, d = 128.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo --expt-relaxed-constexpr \
//        -I include -I paper_2403_16161_b200/csrc [-DATTN_SRC='"/path/attn_sk2.cu"'] \
//        tools/micro/attn_micro.cu -lcuda -o /tmp/attn_micro
//   /tmp/attn_micro [iters] [t(race)|x] [grid (0 = auto)] [2] [w(indow shape)] [s(ingle-tile window units)]
// (tools/micro/ab_attn.sh builds two sources and alternates them on one GPU)
//
// Prints the mean launch time, TFLOP/s (4 Nq Nk D valid-key FLOPs) and, with `trace`, the
// clock64 timeline of CTA 0's first key tiles (the kernel's VI_SK_TRACE stamps).
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <vector>

#ifndef SK2_TRACE
#define SK2_TRACE 1   // per-CTA / per-tile stamps compiled in (-DSK2_TRACE=0 for the library's code)
#endif
#ifndef ATTN_SRC
#define ATTN_SRC "../../paper_2403_16161_b200/csrc/kernels/attn_sk2.cu"
#endif
#ifndef SETUP_SRC
#define SETUP_SRC "../../paper_2403_16161_b200/csrc/kernels/setup.cu"
#endif
#include ATTN_SRC
#include SETUP_SRC
namespace vi {
int g_pdl = 1;   // (rows.cu's definition in the library)
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

int main(int argc, char** argv) {
  const int iters = argc > 1 ? atoi(argv[1]) : 50;
  const bool trace = argc > 2 && argv[2][0] == 't';
  const int grid_override = argc > 3 ? atoi(argv[3]) : 0;
  const int ver = 2;
  // argv[5] == 'w': the C4 window shape (16 windows of 5 x 9 tokens, window-major rows,
  // 225 queries and 675 keys per window, key regions padded to 680 rows)
  const bool win = argc > 5 && argv[5][0] == 'w';
  const int WN = 16, WREAL = 45, WKS = (15 * WREAL + 7) / 8 * 8;
  const int Nq = 3600, H = 4, HD = 128, D = H * HD, P = 720, S = 15, SP = win ? WN * WKS : S * P,
            vt_ld = (SP + 63) / 64 * 64;
  uint16_t *q, *k, *vt, *o;
  cudaMalloc(&q, (size_t)Nq * D * 2);
  cudaMalloc(&k, (size_t)SP * D * 2);
  cudaMalloc(&vt, (size_t)D * vt_ld * 2);
  cudaMalloc(&o, (size_t)Nq * D * 2);
  fill_kernel<<<1024, 256>>>(q, (size_t)Nq * D, 1, 4.f);
  fill_kernel<<<1024, 256>>>(k, (size_t)SP * D, 2, 4.f);
  fill_kernel<<<1024, 256>>>(vt, (size_t)D * vt_ld, 3, 2.f);
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  CUtensorMap tq = tmap(q, D, Nq, 64, 128), tk = tmap(k, D, SP, 64, 128), tv = tmap(vt, vt_ld, D, 64, HD);
  CUtensorMap to = tmap(o, D, Nq, 64, 32);     // output rows (TMA-store epilogue)
  auto launch = [&](const AttnTC& aa, int gr, cudaStream_t s_) {
#ifdef VI_SK2_HAS_OUT_MAP
    return launch_attn_sk2(tq, tk, tv, aa, gr, s_, &to);
#else
    return launch_attn_sk2(tq, tk, tv, aa, gr, s_);
#endif
  };
  AttnTC a;
  memset(&a, 0, sizeof(a));
  a.Nq = Nq; a.hd = HD; a.D = D; a.H = H; a.krow_base = 0; a.vrow_base = 0;
  a.scale_log2 = 1.4426950408889634f / sqrtf(float(HD));
  a.segs.n = 1; a.segs.row0[0] = 0; a.segs.lead[0] = 0; a.segs.len[0] = SP; a.segs.tile0[0] = 0;
  a.segs.tile0[1] = (SP + 127) / 128;
  a.o = reinterpret_cast<bf16*>(o); a.o_ld = D; a.o_hs = HD; a.q_row0 = 0;
#ifdef VI_SK2_HAS_OUT_MAP
  a.o_tma = (argc > 5 && argv[5][0] == 'w') ? 0 : 1;
#endif
  a.npairs = (Nq + 255) / 256;
  a.units = a.npairs * H;
  if (win) {
    a.win_n = WN; a.win_pad = WREAL; a.win_real = WREAL; a.win_h = 5; a.win_w = 9; a.win_cols = 4;
    a.ow = 36; a.P = P; a.win_nq = 5 * WREAL; a.win_qstride = 5 * WREAL; a.win_kstride = WKS;
    a.win_npw = 1;
    a.segs.len[0] = 15 * WREAL;
    a.segs.tile0[1] = (15 * WREAL + 127) / 128;
    a.npairs = 1;
    a.units = WN * H;
#ifndef VI_SK2_NO_SINGLE
    if (argc > 6 && argv[6][0] == 's') {   // single 128-query tiles per unit (the engine's C4 default)
      a.sk_single = 1;
      a.win_npw = 2;
      a.npairs = 2;
      a.units = WN * 2 * H;
    }
#endif
  }
  cudaMalloc(&a.spart, (size_t)nsm * 2 * 256 * HD * 4);
  cudaMalloc(&a.slse, (size_t)nsm * 2 * 256 * 4);
  cudaMalloc(&a.sflag, (size_t)(nsm * 2 + a.units + 8) * 4);
  cudaMemset(a.sflag, 0, (size_t)(nsm * 2 + a.units + 8) * 4);
#ifndef VI_SK2_BASE
  a.uparts = a.sflag;   // (2 x units ints fit in the flag buffer)
#endif
  const long long work = (long long)a.units * a.segs.tile0[1];
  // sk2 tail ordering (engine.cu): the last pair of each head has an empty second tile
  const int rem = Nq % 256;
  a.sk_tail = (ver == 2 && rem > 0 && rem <= 128 && !win) ? 1 : 0;
  a.sk_tail_w = a.sk_tail && getenv("VI_SK_TAIL_W") ? atoi(getenv("VI_SK_TAIL_W")) : 16;
  a.sk_wfull = (long long)(a.npairs - a.sk_tail) * H * a.segs.tile0[1];
  a.sk_ucost = getenv("VI_SK_UNIT_COST") ? atoi(getenv("VI_SK_UNIT_COST")) : (win ? 0 : 56);
  int grid = int(work < nsm ? work : nsm);
  if (grid_override > 0) grid = grid_override;
  cudaStream_t st;
  cudaStreamCreate(&st);
  for (int i = 0; i < 3; ++i) launch(a, grid, st);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, st);
  for (int i = 0; i < iters; ++i) launch(a, grid, st);
  cudaEventRecord(e1, st);
  cudaError_t err = cudaStreamSynchronize(st);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flop = 4.0 * Nq * (win ? 15.0 * WREAL : double(SP)) * D, us = 1e3 * ms / iters;
  printf("attn_sk%d C3: grid %d, %.2f us/launch, %.1f TFLOP/s (%s)\n", ver, grid, us, flop / (us * 1e-6) / 1e12,
         cudaGetErrorString(err));
#ifndef VI_SK2_BASE
  if (getenv("COMB_ONLY") && !win) {   // the split-unit combine kernel alone, back to back
    cudaEventRecord(e0, st);
    for (int i = 0; i < iters; ++i) sk2_combine_kernel<128, false><<<dim3(a.units, 8, 2), 256, 0, st>>>(a);
    cudaEventRecord(e1, st);
    cudaStreamSynchronize(st);
    float cms = 0.f;
    cudaEventElapsedTime(&cms, e0, e1);
    printf("combine alone: %.2f us/launch (%s)\n", 1e3 * cms / iters, cudaGetErrorString(cudaGetLastError()));
  }
#endif
  if (getenv("CTA_TRACE")) {   // per-CTA globaltimer stamps of one launch
    long long* ctb;
    cudaMalloc(&ctb, (size_t)grid * 24 * 8);
    cudaMemset(ctb, 0, (size_t)grid * 24 * 8);
    a.cta_trace = ctb;
    launch(a, grid, st);
    cudaStreamSynchronize(st);
    a.cta_trace = nullptr;
    std::vector<long long> h((size_t)grid * 24);
    cudaMemcpy(h.data(), ctb, h.size() * 8, cudaMemcpyDeviceToHost);
    long long t0 = LLONG_MAX;
    for (int c = 0; c < grid; ++c) t0 = std::min(t0, h[c * 24]);
    printf("cta: entry setup firstQK lastOfinal lastEpi ownerFlags exit nseg | segment o_final (ns from first entry)\n");
    for (int c = 0; c < grid; ++c) {
      const long long* e = &h[c * 24];
      printf("%3d:", c);
      for (int i = 0; i < 7; ++i) printf(" %6lld", e[i] ? e[i] - t0 : -1);
      printf(" %lld |", e[7]);
      for (int i = 0; i < e[7] && i < 4; ++i) printf(" %6lld", e[8 + i] - t0);
      printf(" | piece published %6lld merged %6lld | lastflag %6lld lastland %6lld | go %6lld flag0 %6lld land0 %6lld merged0 %6lld",
             e[12] ? e[12] - t0 : -1, e[13] ? e[13] - t0 : -1, e[14] ? e[14] - t0 : -1, e[15] ? e[15] - t0 : -1,
             e[16] ? e[16] - t0 : -1, e[17] ? e[17] - t0 : -1, e[18] ? e[18] - t0 : -1, e[19] ? e[19] - t0 : -1);
      printf("\n");
    }
  }
  if (trace) {
    long long* tb;
    cudaMalloc(&tb, 32 * 32 * sizeof(long long));
    cudaMemset(tb, 0, 32 * 32 * sizeof(long long));
    a.trace = tb;
    launch(a, grid, st);
    cudaStreamSynchronize(st);
    std::vector<long long> h(32 * 32);
    cudaMemcpy(h.data(), tb, h.size() * 8, cudaMemcpyDeviceToHost);
    const long long t0 = h[24];
    printf("per key tile j and Q tile t: S ready | row max exchanged | P written (half0 min..max, half1 min..max) | "
           "PV issue (half0, half1) | QK issued   (clk relative to the first QK)\n");
    for (int j = 0; j < 32 && (h[j * 32 + 24] || h[j * 32 + 25]); ++j) {
      printf("%2d", j);
      for (int t = 0; t < 2; ++t) {
        const long long* e = &h[j * 32];
        if (!e[24 + t]) continue;          // (single-tile units: tile j on warpgroup j % 2 only)
        long long pm[2][2];
        for (int hf = 0; hf < 2; ++hf) {
          pm[hf][0] = LLONG_MAX;
          pm[hf][1] = 0;
          for (int qd = 0; qd < 4; ++qd) {
            pm[hf][0] = std::min(pm[hf][0], e[4 + t * 8 + hf * 4 + qd]);
            pm[hf][1] = std::max(pm[hf][1], e[4 + t * 8 + hf * 4 + qd]);
          }
        }
        printf(" | t%d S %6lld ld %+4lld mx %+4lld e0 %+4lld P0 %+4lld..%+4lld e1 %+4lld P1 %+4lld..%+4lld PV %+4lld %+4lld QK %6lld",
               t, e[t] - t0, e[22 + t] - e[t], e[2 + t] - e[t], e[28 + t] - e[t], pm[0][0] - e[t], pm[0][1] - e[t],
               e[30 + t] - e[t], pm[1][0] - e[t], pm[1][1] - e[t], e[20 + t] - e[t], e[26 + t] - e[t], e[24 + t] - t0);
      }
      printf("\n");
    }
  }
  return 0;
}
