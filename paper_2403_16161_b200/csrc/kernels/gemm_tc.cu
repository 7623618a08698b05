// tcgen05 GEMM with fused epilogues: C[M][N] = A[M][K] * W[N][K]^T (bf16 in, fp32 acc).
//
// Persistent, warp-specialised, in clusters of CM x CN CTAs: a cluster owns CM x CN
// adjacent 128 x BN output tiles (a "super-tile") and walks super-tiles cid, cid + #clusters,
// ...  The A tile (128 rows x 64 k) of a cluster row is loaded in CN slices, each CTA of the
// row loading one slice and TMA-multicasting it to the row; the W tile of a cluster column
// likewise in CM slices.  At M = 3600 the operands are re-read once per tile from L2, so
// multicast is what keeps these GEMMs off the L2 bandwidth ceiling.  A stage is refilled
// only after every CTA of the cluster has consumed it (tcgen05.commit multicast to all).
// Warp roles (384 threads):
//   warp 0, lane 0 : TMA producer  (A box 64x128, W box 64xBN, 128-byte swizzle), an
//                    STAGES-deep smem ring that keeps streaming across tile boundaries
//   warp 1, lane 0 : MMA issuer    (tcgen05.mma kind::f16, M=128, N=BN, K=16 per instr)
//   warp 2         : TMEM allocator (2 x BN fp32 columns: double-buffered accumulator)
//   warps 4..11    : epilogue      (tcgen05.ld 32x32b, thread = accumulator row; warps w and
//                    w+4 share a TMEM lane quadrant and split the tile's columns in half)
// With two accumulators the epilogue of tile i overlaps the mainloop of tile i+1.  The
// bias of a tile is staged in shared memory (broadcast reads) and residual rows are
// loaded before the TMEM load is waited on, so the epilogue keeps pace with the MMAs.
#include "epilogue.cuh"
#include "kernels.h"

namespace vi {

__device__ __forceinline__ void gemm_named_bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

template <int BN, int STAGES, bool TE = false>
struct GemmSmem {  // (cluster shape does not change the layout)
  static constexpr int A_BYTES = 128 * 64 * 2;
  static constexpr int B_BYTES = BN * 64 * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  // TMA-store epilogue: per epilogue warp two 32-row x 128-byte staging buffers (1 KB aligned
  // for the 128-byte swizzle of the output tensor maps)
  static constexpr int STG_OFF = STAGES * STAGE_BYTES;
  static constexpr int STG_BYTES = TE ? 8 * 2 * 4096 : 0;
  static constexpr int BAR_OFF = STG_OFF + STG_BYTES;
  static constexpr int NBAR = 2 * STAGES + 4 + 8;                          // + [8] x_in tile loads
  static constexpr int BIAS_OFF = BAR_OFF + NBAR * 8 + 16;                 // [2][BN] fp32
  static constexpr int TOTAL = BIAS_OFF + 2 * BN * 4 + 1024;              // +1024 alignment slack
};

#ifdef VI_GEMM_TRACE
__device__ long long g_gemm_trace[24];
#define GTR(i) do { if (blockIdx.x == 0) g_gemm_trace[i] = (long long)globaltimer(); } while (0)
#else
#define GTR(i) do { } while (0)
#endif

template <int BN, int STAGES, int CM, int CN, bool TE>
__global__ void __launch_bounds__(384, 1)
gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
               const __grid_constant__ CUtensorMap tmO, const __grid_constant__ CUtensorMap tmX, int K, int brow0,
               Epi epi) {
  using L = GemmSmem<BN, STAGES, TE>;
  constexpr int CS = CM * CN;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // 1 KB aligned, stays in .shared
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::BAR_OFF);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;     // [2] accumulator ready for the epilogue
  uint64_t* tempty = tfull + 2;         // [2] accumulator drained by the epilogue
  uint64_t* xbar = tempty + 2;          // [8] per epilogue warp: x_in tile landed (TE, EPI_RESID)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(xbar + 8);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) GTR(0);
  const int rank = CS > 1 ? int(cluster_ctarank()) : 0;
  const int cx = rank % CN, cy = rank / CN;           // position inside the cluster
  const int cid = blockIdx.x / CS, ncl = gridDim.x / CS;
  const int tiles_m = (epi.M + 127) / 128, tiles_n = (epi.N + BN - 1) / BN;
  const int super_m = (tiles_m + CM - 1) / CM, super_n = (tiles_n + CN - 1) / CN;
  const int nsuper = super_m * super_n;
  const int nk = (K + 63) / 64;
  constexpr uint32_t TMEM_COLS = 2 * BN < 32 ? 32 : 2 * BN;
  constexpr int A_SLICE = L::A_BYTES / CN, B_SLICE = L::B_BYTES / CM;
  const uint16_t row_mask = uint16_t(((1u << CN) - 1) << (cy * CN));
  uint16_t col_mask = 0;
#pragma unroll
  for (int y = 0; y < CM; ++y) col_mask |= uint16_t(1u << (y * CN + cx));
  const uint16_t all_mask = uint16_t((1u << CS) - 1);

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    if (TE) {
      tma_prefetch(&tmO);
      if (epi.kind == EPI_RESID) tma_prefetch(&tmX);
    }
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CS);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 256);
    }
    for (int w = 0; w < 8; ++w) mbar_init(&xbar[w], 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, TMEM_COLS);
  tc_fence_before();
  if (CS > 1) cluster_sync_all();   // peers' barriers initialised before any multicast
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // everything above overlaps the previous kernel's tail (programmatic dependent launch)
  griddep_wait();
  griddep_launch();
  if (threadIdx.x == 0) GTR(1);
  if (threadIdx.x == 0) time_begin(epi.timing);

  if (warp == 0) {
    if (lane == 0) {
      int it = 0;                               // global k-block counter (ring position)
      for (int st = cid; st < nsuper; st += ncl) {
        const int m0 = ((st % super_m) * CM + cy) * 128, n0 = ((st / super_m) * CN + cx) * BN;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % STAGES;
          if (it >= STAGES) mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
          uint8_t* sa = smem + s * L::STAGE_BYTES;
          mbar_arrive_expect_tx(&full[s], L::STAGE_BYTES);
          int ak = kb * 64, am = m0;
          if (epi.a_hs > 0) {                   // head-major A: K-block kb of head kb / a_kpb
            const int hh = kb / epi.a_kpb;
            ak = (kb - hh * epi.a_kpb) * 64;
            am = hh * epi.a_hs + m0;
          }
          if (CN > 1)
            tma_load_2d_mc(sa + cx * A_SLICE, &tmA, &full[s], ak, am + cx * (128 / CN), row_mask);
          else
            tma_load_2d(sa, &tmA, &full[s], ak, am);
          if (CM > 1)
            tma_load_2d_mc(sa + L::A_BYTES + cy * B_SLICE, &tmB, &full[s], kb * 64, brow0 + n0 + cy * (BN / CM),
                           col_mask);
          else
            tma_load_2d(sa + L::A_BYTES, &tmB, &full[s], kb * 64, brow0 + n0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16_f32(128, BN);
      int it = 0, lt = 0;
      for (int st = cid; st < nsuper; st += ncl, ++lt) {
        const int acc = lt & 1;
        if (lt >= 2) mbar_wait(&tempty[acc], ((lt >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * BN;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % STAGES;
          mbar_wait(&full[s], (it / STAGES) & 1);
          if (it == 0) GTR(2);
          tc_fence_after();
          const uint32_t a = smem_u32(smem + s * L::STAGE_BYTES);
          const uint32_t b = a + L::A_BYTES;
#pragma unroll
          for (int k = 0; k < 4; ++k)
            umma_bf16_ss(d, sdesc_k_sw128(a + k * 32), sdesc_k_sw128(b + k * 32), idesc, (kb | k) != 0);
          if (CS > 1)
            umma_commit_mc(&empty[s], all_mask);    // stage free in every CTA that shares it
          else
            umma_commit(&empty[s]);
        }
        umma_commit(&tfull[acc]);
        if (lt < 4) GTR(3 + lt);
      }
    }
  } else if (warp >= 4) {
    const int ew = warp - 4;                     // 0..7
    const int q = ew & 3, hc = ew >> 2;          // TMEM lane quadrant, column half
    const int etid = ew * 32 + lane;             // 0..255
    float* bias_s = reinterpret_cast<float*>(smem + L::BIAS_OFF);
    uint8_t* stg = smem + L::STG_OFF + ew * 8192;
    int nchunk = 0;
    uint32_t xphase = 0;
    int lt = 0;
    for (int st = cid; st < nsuper; st += ncl, ++lt) {
      const int acc = lt & 1;
      const int m0 = ((st % super_m) * CM + cy) * 128, n0 = ((st / super_m) * CN + cx) * BN;
      float* bs = bias_s + acc * BN;
      if (epi.bias) {
        for (int i = etid; i < BN; i += 256) bs[i] = n0 + i < epi.N ? __ldg(epi.bias + n0 + i) : 0.f;
      }
      gemm_named_bar_sync(1, 256);
      mbar_wait(&tfull[acc], (lt >> 1) & 1);
      if (lt < 4 && ew == 0 && lane == 0) GTR(7 + lt);
      tc_fence_after();
      const int m = m0 + q * 32 + lane;
      if constexpr (TE) {
        // TMA-store epilogue: the warp's 32 rows x (128 B of output) go through a swizzled
        // staging buffer and leave as one bulk tensor store (coalesced, asynchronous); a
        // residual tile arrives the same way (TMA load into the buffer it is stored from).
        const bool resid = epi.kind == EPI_RESID;
        const int cw = (resid || epi.out_f32) ? 32 : 64;           // columns per 128-byte row
        const int sw = lane & 7;                                  // 128-byte swizzle phase of this row
#pragma unroll 1
        for (int c = hc * (BN / 2); c < (hc + 1) * (BN / 2); c += cw, ++nchunk) {
          if (n0 + c >= epi.N) break;
          uint8_t* buf = stg + (nchunk & 1) * 4096;
          if (nchunk >= 2) {                    // the store that used this buffer has read it
            if (lane == 0) bulk_wait_read<1>();
            __syncwarp();
          }
          if (resid && lane == 0) {
            mbar_arrive_expect_tx(&xbar[ew], 4096);
            tma_load_2d(buf, &tmX, &xbar[ew], n0 + c, m0 + q * 32);
          }
#pragma unroll 1
          for (int h2 = 0; h2 < cw; h2 += 32) {
            float v[32];
            tmem_ld32(tmem + acc * BN + (uint32_t(q * 32) << 16) + c + h2, reinterpret_cast<uint32_t*>(v));
            tmem_wait_ld();
            if (epi.bias) {
#pragma unroll
              for (int i = 0; i < 32; ++i) v[i] += bs[c + h2 + i];
            }
            if (epi.kind == EPI_GELU) {
#pragma unroll
              for (int i = 0; i < 32; ++i) v[i] = gelu_erf(v[i]);
            } else if (epi.kind == EPI_STORE && epi.pos && m < epi.M) {
              const float* pr = epi.pos + (size_t)(m % epi.P) * epi.N + n0 + c + h2;
#pragma unroll
              for (int i = 0; i < 32; ++i) v[i] += (n0 + c + h2 + i < epi.N) ? __ldg(pr + i) : 0.f;
            }
            uint8_t* row = buf + lane * 128;
            if (resid || epi.out_f32) {
              if (resid) {
                mbar_wait(&xbar[ew], xphase);
                xphase ^= 1u;
              }
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                float4* p4 = reinterpret_cast<float4*>(row + ((j ^ sw) << 4));
                float4 o = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
                if (resid) {
                  const float4 xi = *p4;
                  o.x += xi.x; o.y += xi.y; o.z += xi.z; o.w += xi.w;
                }
                *p4 = o;
              }
            } else {
#pragma unroll
              for (int j = 0; j < 4; ++j)
                *reinterpret_cast<uint4*>(row + (((h2 / 8 + j) ^ sw) << 4)) =
                    make_uint4(pack_bf16(v[8 * j], v[8 * j + 1]), pack_bf16(v[8 * j + 2], v[8 * j + 3]),
                               pack_bf16(v[8 * j + 4], v[8 * j + 5]), pack_bf16(v[8 * j + 6], v[8 * j + 7]));
            }
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&tmO, buf, n0 + c, m0 + q * 32);
            bulk_commit();
          }
        }
        tc_fence_before();
        mbar_arrive(&tempty[acc]);
        if (lt < 4 && ew == 0 && lane == 0) GTR(11 + lt);
        continue;
      }
#pragma unroll 1
      for (int c = hc * (BN / 2); c < (hc + 1) * (BN / 2); c += 32) {
        if (n0 + c >= epi.N) break;
        uint32_t r[32];
        tmem_ld32(tmem + acc * BN + (uint32_t(q * 32) << 16) + c, r);
        float4 xin[8];
        if (epi.kind == EPI_RESID && m < epi.M && n0 + c + 32 <= epi.N) {
          const float4* xi = reinterpret_cast<const float4*>(epi.x_in + (size_t)m * epi.N + n0 + c);
#pragma unroll
          for (int i = 0; i < 8; ++i) xin[i] = xi[i];
        }
        tmem_wait_ld();
        epi_row32_bf16(epi, m, n0 + c, reinterpret_cast<float*>(r), epi.bias ? bs + c : nullptr, xin);
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      if (lt < 4 && ew == 0 && lane == 0) GTR(11 + lt);
    }
    if (TE && lane == 0) bulk_wait<0>();        // staging buffers stay valid until stored
  }
  tc_fence_before();
  if (CS > 1) cluster_sync_all();   // no CTA leaves while peers may still multicast into it
  else __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, TMEM_COLS);
  }
  if (threadIdx.x == 0) GTR(15);
  if (threadIdx.x == 0) time_end(epi.timing, gridDim.x);
}

static int g_num_sms = 0;

template <int BN, int STAGES, int CM, int CN, bool TE = false>
static cudaError_t launch_cfg(const CUtensorMap& a, const CUtensorMap& b, int brow0, int M, int N, int K,
                              const Epi& e, cudaStream_t st, const CUtensorMap* tmo = nullptr,
                              const CUtensorMap* tmx = nullptr) {
  using L = GemmSmem<BN, STAGES, TE>;
  constexpr int CS = CM * CN;
  auto kfn = gemm_tc_kernel<BN, STAGES, CM, CN, TE>;
  static int max_clusters = 0;
  if (!max_clusters) {
    cudaError_t err = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, L::TOTAL);
    if (err != cudaSuccess) return err;
    if (CS > 1) cudaFuncSetAttribute(kfn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    max_clusters = g_num_sms / CS;
    if (CS > 1) {
      cudaLaunchConfig_t q = {};
      q.gridDim = dim3(CS * max_clusters);
      q.blockDim = dim3(384);
      q.dynamicSmemBytes = L::TOTAL;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = CS; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      q.attrs = at;
      q.numAttrs = 1;
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, kfn, &q) == cudaSuccess && n > 0) max_clusters = n;
      cudaGetLastError();
    }
  }
  const int tiles_m = (M + 127) / 128, tiles_n = (N + BN - 1) / BN;
  const int nsuper = ((tiles_m + CM - 1) / CM) * ((tiles_n + CN - 1) / CN);
  const int ncl = nsuper < max_clusters ? nsuper : max_clusters;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ncl * CS);
  cfg.blockDim = dim3(384);
  cfg.dynamicSmemBytes = L::TOTAL;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CS; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = g_pdl;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  // unused output maps are passed as copies of the A map (never dereferenced)
  return cudaLaunchKernelEx(&cfg, kfn, a, b, tmo ? *tmo : a, tmx ? *tmx : a, K, brow0, e);
}

// cluster (CM x CN): 0 = 1x1, 1 = 2x1 (W tile multicast), 2 = 1x2 (A multicast), 3 = 2x2,
// 4 = 1x4, 5 = 2x4, 6 = 1x8, 7 = 4x2.  The A map's box must be 64 x (128 / CN), the W map's
// 64 x (BN / CM).
cudaError_t launch_gemm_tc(const CUtensorMap& a, const CUtensorMap& b, int brow0, int M, int N, int K, int bn,
                           const Epi& e, cudaStream_t st, int cluster, const CUtensorMap* tmo,
                           const CUtensorMap* tmx) {
  if (tmo) {   // TMA-store epilogue (EPI_STORE / EPI_GELU / EPI_RESID), no clusters
    if (e.kind != EPI_STORE && e.kind != EPI_GELU && e.kind != EPI_RESID) return cudaErrorInvalidValue;
    if (e.kind == EPI_RESID && !tmx) return cudaErrorInvalidValue;
    switch (bn) {
      case 64: return launch_cfg<64, 6, 1, 1, true>(a, b, brow0, M, N, K, e, st, tmo, tmx);
      case 128: return launch_cfg<128, 4, 1, 1, true>(a, b, brow0, M, N, K, e, st, tmo, tmx);
      case 256: return launch_cfg<256, 3, 1, 1, true>(a, b, brow0, M, N, K, e, st, tmo, tmx);
      default: return cudaErrorInvalidValue;
    }
  }
#define CASES(BN, ST)                                                              \
  switch (cluster) {                                                               \
    case 0: return launch_cfg<BN, ST, 1, 1>(a, b, brow0, M, N, K, e, st);          \
    case 1: return launch_cfg<BN, ST, 2, 1>(a, b, brow0, M, N, K, e, st);          \
    case 2: return launch_cfg<BN, ST, 1, 2>(a, b, brow0, M, N, K, e, st);          \
    case 3: return launch_cfg<BN, ST, 2, 2>(a, b, brow0, M, N, K, e, st);          \
    case 4: return launch_cfg<BN, ST, 1, 4>(a, b, brow0, M, N, K, e, st);          \
    case 5: return launch_cfg<BN, ST, 2, 4>(a, b, brow0, M, N, K, e, st);          \
    case 6: return launch_cfg<BN, ST, 1, 8>(a, b, brow0, M, N, K, e, st);          \
    case 7: return launch_cfg<BN, ST, 4, 2>(a, b, brow0, M, N, K, e, st);          \
    default: return cudaErrorInvalidValue;                                         \
  }
  switch (bn) {
    case 64: CASES(64, 8)
    case 128: CASES(128, 6)
    case 256: CASES(256, 4)
    default: return cudaErrorInvalidValue;
  }
#undef CASES
}

}  // namespace vi
