// tcgen05 GEMM with fused epilogues: C[M][N] = A[M][K] * W[N][K]^T (bf16 in, fp32 acc).
//
// Persistent, warp-specialised: grid = min(#tiles, #SMs) CTAs, each walks the 128 x BN
// output tiles blockIdx.x, blockIdx.x + gridDim.x, ... (m fastest, so CTAs running at
// the same time share the weight block in L2).  Warp roles (384 threads):
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

template <int BN, int STAGES>
struct GemmSmem {
  static constexpr int A_BYTES = 128 * 64 * 2;
  static constexpr int B_BYTES = BN * 64 * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int BAR_OFF = STAGES * STAGE_BYTES;
  static constexpr int BIAS_OFF = BAR_OFF + (2 * STAGES + 4) * 8 + 16;   // [2][BN] fp32
  static constexpr int TOTAL = BIAS_OFF + 2 * BN * 4 + 1024;              // +1024 alignment slack
};

template <int BN, int STAGES>
__global__ void __launch_bounds__(384, 1)
gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int K, int brow0,
               Epi epi) {
  using L = GemmSmem<BN, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::BAR_OFF);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;     // [2] accumulator ready for the epilogue
  uint64_t* tempty = tfull + 2;         // [2] accumulator drained by the epilogue
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tiles_m = (epi.M + 127) / 128, tiles_n = (epi.N + BN - 1) / BN;
  const int ntiles = tiles_m * tiles_n;
  const int nk = (K + 63) / 64;
  constexpr uint32_t TMEM_COLS = 2 * BN < 32 ? 32 : 2 * BN;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 256);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int it = 0;                               // global k-block counter (ring position)
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int m0 = (tile % tiles_m) * 128, n0 = (tile / tiles_m) * BN;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % STAGES;
          if (it >= STAGES) mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
          uint8_t* sa = smem + s * L::STAGE_BYTES;
          mbar_arrive_expect_tx(&full[s], L::STAGE_BYTES);
          tma_load_2d(sa, &tmA, &full[s], kb * 64, m0);
          tma_load_2d(sa + L::A_BYTES, &tmB, &full[s], kb * 64, brow0 + n0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16_f32(128, BN);
      int it = 0, lt = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++lt) {
        const int acc = lt & 1;
        if (lt >= 2) mbar_wait(&tempty[acc], ((lt >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * BN;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % STAGES;
          mbar_wait(&full[s], (it / STAGES) & 1);
          tc_fence_after();
          const uint32_t a = smem_u32(smem + s * L::STAGE_BYTES);
          const uint32_t b = a + L::A_BYTES;
#pragma unroll
          for (int k = 0; k < 4; ++k)
            umma_bf16_ss(d, sdesc_k_sw128(a + k * 32), sdesc_k_sw128(b + k * 32), idesc, (kb | k) != 0);
          umma_commit(&empty[s]);
        }
        umma_commit(&tfull[acc]);
      }
    }
  } else if (warp >= 4) {
    const int ew = warp - 4;                     // 0..7
    const int q = ew & 3, hc = ew >> 2;          // TMEM lane quadrant, column half
    const int etid = ew * 32 + lane;             // 0..255
    float* bias_s = reinterpret_cast<float*>(smem + L::BIAS_OFF);
    int lt = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++lt) {
      const int acc = lt & 1;
      const int m0 = (tile % tiles_m) * 128, n0 = (tile / tiles_m) * BN;
      float* bs = bias_s + acc * BN;
      if (epi.bias) {
        for (int i = etid; i < BN; i += 256) bs[i] = n0 + i < epi.N ? __ldg(epi.bias + n0 + i) : 0.f;
      }
      gemm_named_bar_sync(1, 256);
      mbar_wait(&tfull[acc], (lt >> 1) & 1);
      tc_fence_after();
      const int m = m0 + q * 32 + lane;
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
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, TMEM_COLS);
  }
}

static int g_num_sms = 0;

template <int BN, int STAGES>
static cudaError_t launch_bn(const CUtensorMap& a, const CUtensorMap& b, int brow0, int M, int N, int K,
                             const Epi& e, cudaStream_t st) {
  using L = GemmSmem<BN, STAGES>;
  auto kfn = gemm_tc_kernel<BN, STAGES>;
  static bool configured = false;
  if (!configured) {
    cudaError_t err = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, L::TOTAL);
    if (err != cudaSuccess) return err;
    configured = true;
  }
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int tiles = ((M + 127) / 128) * ((N + BN - 1) / BN);
  const int grid = tiles < g_num_sms ? tiles : g_num_sms;
  kfn<<<grid, 384, L::TOTAL, st>>>(a, b, K, brow0, e);
  return cudaGetLastError();
}

cudaError_t launch_gemm_tc(const CUtensorMap& a, const CUtensorMap& b, int brow0, int M, int N, int K, int bn,
                           const Epi& e, cudaStream_t st) {
  switch (bn) {
    case 64: return launch_bn<64, 8>(a, b, brow0, M, N, K, e, st);
    case 128: return launch_bn<128, 6>(a, b, brow0, M, N, K, e, st);
    case 256: return launch_bn<256, 4>(a, b, brow0, M, N, K, e, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace vi
