// tcgen05 GEMM with fused epilogues: C[M][N] = A[M][K] * W[N][K]^T (bf16 in, fp32 acc).
//
// Persistent and warp-specialised, in two modes:
//   single CTA   : a CTA owns 128 x BN output tiles and walks tiles blockIdx.x, +gridDim.x, ...
//   CTA pair     : a cluster of 2 CTAs owns 256 x BN tiles and computes them with the 2-SM
//                  MMA (tcgen05.mma.cta_group::2, M = 256): each CTA loads its 128 rows of A
//                  and HALF of the BN rows of W into its own shared memory, the leader (rank
//                  0) issues the MMAs, each CTA's TMEM receives its 128 accumulator rows.
//                  Per SM the operand bytes per MMA cycle drop from (128 + BN)/(2 BN) x 128 B
//                  to (128 + BN/2)/(2 BN) x 128 B -- the per-SM ingress (~60-80 B/clk
//                  measured, tools/micro/gemm_micro) bounds the single-CTA K = 512 GEMMs.
// Warp roles (384 threads per CTA):
//   warp 0, lane 0 : TMA producer  (A box 64x128, W box 64x(BN or BN/2), 128-byte swizzle),
//                    a STAGES-deep smem ring that keeps streaming across tile boundaries;
//                    in pair mode both CTAs load, completion counted on the leader's barrier
//   warp 1, lane 0 : MMA issuer    (tcgen05.mma kind::f16, M = 128 or 256, N = BN, K = 16)
//   warp 2         : TMEM allocator (2 x BN fp32 columns: double-buffered accumulator)
//   warps 4..11    : epilogue      (tcgen05.ld 32x32b, thread = accumulator row; warps w and
//                    w+4 share a TMEM lane quadrant and split the tile's columns in half)
// With two accumulators the epilogue of tile i overlaps the mainloop of tile i+1.  TE: the
// STORE / GELU / RESID epilogues leave through per-warp swizzled staging buffers and TMA
// bulk tensor stores (residual tiles arrive by TMA loads); otherwise (the QKV memory
// scatter) from registers (epilogue.cuh).
#include "epilogue.cuh"
#include "kernels.h"

namespace vi {

__device__ __forceinline__ void gemm_named_bar_sync(int id, int n) {   // (.aligned: converged warps)
  __syncwarp();
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

template <int BN, int STAGES, bool PAIR, bool TE>
struct GemmSmem {
  static constexpr int A_BYTES = 128 * 64 * 2;
  static constexpr int B_BYTES = (PAIR ? BN / 2 : BN) * 64 * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  // TMA-store epilogue: per epilogue warp two 32-row x 128-byte staging buffers (1 KB aligned
  // for the 128-byte swizzle of the output tensor maps)
  static constexpr int STG_OFF = STAGES * STAGE_BYTES;
  static constexpr int STG_BYTES = TE ? 8 * 2 * 4096 : 0;
  static constexpr int BAR_OFF = STG_OFF + STG_BYTES;
  static constexpr int NBAR = 2 * STAGES + 4 + 16;                         // + [8 warps][2 buffers] x_in tile loads
  static constexpr int BIAS_OFF = BAR_OFF + NBAR * 8 + 16;                 // [2][BN] fp32
  static constexpr int TOTAL = BIAS_OFF + 2 * BN * 4 + 1024;              // +1024 alignment slack
};

#ifdef VI_GEMM_TRACE
__device__ long long g_gemm_trace[64];
#define GTR(i) do { if (blockIdx.x == 0) g_gemm_trace[i] = (long long)globaltimer(); } while (0)
#else
#define GTR(i) do { } while (0)
#endif

template <int BN, int STAGES, bool PAIR, bool TE>
__global__ void __launch_bounds__(384, 1)
gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
               const __grid_constant__ CUtensorMap tmO, const __grid_constant__ CUtensorMap tmX,
               const __grid_constant__ CUtensorMap tmV, int K, int brow0, Epi epi) {
  using L = GemmSmem<BN, STAGES, PAIR, TE>;
  constexpr int TM = PAIR ? 256 : 128;                 // rows of a (pair) tile
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // 1 KB aligned, stays in .shared
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::BAR_OFF);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;     // [2] accumulator ready for the epilogue
  uint64_t* tempty = tfull + 2;         // [2] accumulator drained by the epilogue (leader's counts both CTAs)
  uint64_t* xbar = tempty + 2;          // [8 warps][2 staging buffers]: x_in tile landed (TE, EPI_RESID)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(xbar + 16);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) GTR(0);
  const int rank = PAIR ? int(cluster_ctarank()) : 0;
  const bool leader = rank == 0;
  const int cid = PAIR ? blockIdx.x / 2 : blockIdx.x, ncl = PAIR ? gridDim.x / 2 : gridDim.x;
  const int tiles_m = (epi.M + TM - 1) / TM, tiles_n = (epi.N + BN - 1) / BN;
  const int ks = epi.ksplit > 1 ? epi.ksplit : 1;
  const int nout = tiles_m * tiles_n;          // output tiles
  const int ntiles = nout * ks;                // work items: (split, tile), tile fastest
  const int nk_all = (K + 63) / 64;
  const int kper = (nk_all + ks - 1) / ks;     // k-blocks per split
  constexpr uint32_t TMEM_COLS = 2 * BN < 32 ? 32 : 2 * BN;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    if (TE) {
      tma_prefetch(&tmO);
      if (epi.kind == EPI_RESID || epi.kind == EPI_QKV) tma_prefetch(&tmX);
      if (epi.kind == EPI_QKV) tma_prefetch(&tmV);
    }
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], PAIR ? 16 : 8);     // one elected arrive per epilogue warp (of both CTAs)
    }
    for (int w = 0; w < 16; ++w) mbar_init(&xbar[w], 1);
    fence_barrier_init();
  }
  if (warp == 2) {
    if (PAIR) tmem_alloc_pair(tmem_slot, TMEM_COLS);
    else tmem_alloc(tmem_slot, TMEM_COLS);
  }
  tc_fence_before();
  if (PAIR) cluster_sync_all();   // both CTAs' barriers initialised and TMEM allocated
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // B is always a weight matrix (constant during a step): the producer requests the first
  // work item's first stages of B before waiting for the previous kernel, so those loads and
  // everything above overlap its tail (programmatic dependent launch)
  int npre = 0;
  if (warp == 0 && lane == 0 && cid < ntiles) {
    const int ot = cid % nout, kb0 = (cid / nout) * kper;
    const int kb1 = kb0 + kper < nk_all ? kb0 + kper : nk_all;
    const int bn0 = brow0 + (ot / tiles_m) * BN + (PAIR ? rank * (BN / 2) : 0);
    npre = kb1 - kb0 < STAGES ? kb1 - kb0 : STAGES;
    for (int j = 0; j < npre; ++j) {
      uint8_t* sa = smem + j * L::STAGE_BYTES;
      if (PAIR) {
        if (leader) mbar_arrive_expect_tx(&full[j], 2 * L::STAGE_BYTES);   // both CTAs' A and B bytes
        tma_load_2d_pair(sa + L::A_BYTES, &tmB, &full[j], (kb0 + j) * 64, bn0);
      } else {
        mbar_arrive_expect_tx(&full[j], L::STAGE_BYTES);
        tma_load_2d(sa + L::A_BYTES, &tmB, &full[j], (kb0 + j) * 64, bn0);
      }
    }
  }
  griddep_wait();
  griddep_launch();
  if (threadIdx.x == 0) GTR(1);
  if (threadIdx.x == 0) time_begin(epi.timing);

  if (warp == 0) {
    if (lane == 0) {
      int it = 0;                               // global k-block counter (ring position)
      for (int st = cid; st < ntiles; st += ncl) {
        const int ot = st % nout, kb0 = (st / nout) * kper;
        const int kb1 = kb0 + kper < nk_all ? kb0 + kper : nk_all;
        const int m0 = (ot % tiles_m) * TM + rank * 128, n0 = (ot / tiles_m) * BN;
        const int bn0 = brow0 + n0 + (PAIR ? rank * (BN / 2) : 0);
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % STAGES;
          if (it >= STAGES) mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
          uint8_t* sa = smem + s * L::STAGE_BYTES;
          int ak = kb * 64, am = m0;
          if (epi.a_hs > 0) {                   // head-major A: K-block kb of head kb / a_kpb
            const int hh = kb / epi.a_kpb;
            ak = (kb - hh * epi.a_kpb) * 64;
            am = hh * epi.a_hs + m0;
          }
          if (it < npre) {            // B of this stage was requested before the wait
            if (PAIR) tma_load_2d_pair(sa, &tmA, &full[s], ak, am);
            else tma_load_2d(sa, &tmA, &full[s], ak, am);
          } else if (PAIR) {
            if (leader) mbar_arrive_expect_tx(&full[s], 2 * L::STAGE_BYTES);   // both CTAs' bytes
            tma_load_2d_pair(sa, &tmA, &full[s], ak, am);
            tma_load_2d_pair(sa + L::A_BYTES, &tmB, &full[s], kb * 64, bn0);
          } else {
            mbar_arrive_expect_tx(&full[s], L::STAGE_BYTES);
            tma_load_2d(sa, &tmA, &full[s], ak, am);
            tma_load_2d(sa + L::A_BYTES, &tmB, &full[s], kb * 64, bn0);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      constexpr uint32_t idesc = idesc_bf16_f32(TM, BN);
      int it = 0, lt = 0;
      for (int st = cid; st < ntiles; st += ncl, ++lt) {
        const int acc = lt & 1;
        const int kb0 = (st / nout) * kper;
        const int kb1 = kb0 + kper < nk_all ? kb0 + kper : nk_all;
        if (lt >= 2) mbar_wait(&tempty[acc], ((lt >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % STAGES;
          mbar_wait(&full[s], (it / STAGES) & 1);
          if (it == 0) GTR(2);
          tc_fence_after();
          const uint32_t a = smem_u32(smem + s * L::STAGE_BYTES);
          const uint32_t b = a + L::A_BYTES;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (PAIR)
              umma_bf16_ss_pair(d, sdesc_k_sw128(a + k * 32), sdesc_k_sw128(b + k * 32), idesc, (kb != kb0) || k);
            else
              umma_bf16_ss(d, sdesc_k_sw128(a + k * 32), sdesc_k_sw128(b + k * 32), idesc, (kb != kb0) || k);
          }
          if (PAIR) umma_commit_pair(&empty[s]);    // the stage is free in both CTAs
          else umma_commit(&empty[s]);
        }
        if (PAIR) umma_commit_pair(&tfull[acc]);
        else umma_commit(&tfull[acc]);
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
    uint32_t xphase = 0;   // bit b: parity of staging buffer b's next x_in load
    int lt = 0;
    for (int st = cid; st < ntiles; st += ncl, ++lt) {
      const int acc = lt & 1;
      const int ot = st % nout;
      const int m0 = (ot % tiles_m) * TM + rank * 128, n0 = (ot / tiles_m) * BN;
      const int srow0 = (st / nout) * epi.kpad_rows;   // split-K: this split's workspace rows
      float* bs = bias_s + acc * BN;
      if (epi.bias) {
        for (int i = etid; i < BN; i += 256) bs[i] = n0 + i < epi.N ? __ldg(epi.bias + n0 + i) : 0.f;
      }
      gemm_named_bar_sync(1, 256);
      // residual epilogue: the x_in tiles of this warp's first two chunks are requested now,
      // while the accumulator is still being computed (both staging buffers free: every
      // earlier store has read them), so their latency overlaps the mainloop
      const bool pre_x = TE && epi.kind == EPI_RESID;
      if (pre_x) {
        if (lane == 0) {
          bulk_wait_read<0>();
          for (int k = 0; k < 2; ++k) {
            const int c = hc * (BN / 2) + k * 32;
            if (c < (hc + 1) * (BN / 2) && n0 + c < epi.N) {
              const int b = (nchunk + k) & 1;
              mbar_arrive_expect_tx(&xbar[2 * ew + b], 4096);
              tma_load_2d(stg + b * 4096, &tmX, &xbar[2 * ew + b], n0 + c, m0 + q * 32);
            }
          }
        }
        __syncwarp();
      }
      mbar_wait_warp(&tfull[acc], (lt >> 1) & 1);
      if (lt < 4 && ew == 0 && lane == 0) GTR(7 + lt);
      tc_fence_after();
      const int m = m0 + q * 32 + lane;
      if constexpr (TE) {
        // TMA-store epilogue: the warp's 32 rows x (128 B of output) go through a swizzled
        // staging buffer and leave as one bulk tensor store (coalesced, asynchronous); a
        // residual tile arrives the same way (TMA load into the buffer it is stored from).
        const bool resid = epi.kind == EPI_RESID, qkv = epi.kind == EPI_QKV;
        const int cw = (resid || epi.out_f32) ? 32 : 64;           // columns per 128-byte row
        const int sw = lane & 7;                                  // 128-byte swizzle phase of this row
        int kc = 0;                             // chunk index within this tile
#pragma unroll 1
        for (int c = hc * (BN / 2); c < (hc + 1) * (BN / 2); c += cw, ++nchunk, ++kc) {
          if (n0 + c >= epi.N) break;
          const int bi = nchunk & 1;
          uint8_t* buf = stg + bi * 4096;
          const bool gtr_c = lt == 0 && ew == 0 && lane == 0 && kc < 8;
          if (gtr_c) GTR(16 + kc * 4);
          if (nchunk >= 2 && !(pre_x && kc < 2)) {   // the store that used this buffer has read it
            if (lane == 0) bulk_wait_read<1>();
            __syncwarp();
          }
          if (resid && kc >= 2 && lane == 0) {  // (chunks 0, 1 were requested before the mainloop ended)
            mbar_arrive_expect_tx(&xbar[2 * ew + bi], 4096);
            tma_load_2d(buf, &tmX, &xbar[2 * ew + bi], n0 + c, m0 + q * 32);
          }
          // QKV: a 64-column chunk lies in one of Q / K / V (D % 64 == 0); V leaves transposed
          const int region = qkv ? (n0 + c) / epi.D : 0;
#pragma unroll 1
          for (int h2 = 0; h2 < cw; h2 += 32) {
            float v[32];
            tmem_ld32(tmem + acc * BN + (uint32_t(q * 32) << 16) + c + h2, reinterpret_cast<uint32_t*>(v));
            tmem_wait_ld();
            if (gtr_c && h2 == 0) GTR(17 + kc * 4);
            if (epi.bias) {
              const float4* b4 = reinterpret_cast<const float4*>(bs + c + h2);
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                const float4 bb = b4[i];
                v[4 * i] += bb.x; v[4 * i + 1] += bb.y; v[4 * i + 2] += bb.z; v[4 * i + 3] += bb.w;
              }
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
            if (region == 2) {
              // Vt boxes: 4 x [64 d][8 tokens] (1 KB each, token group lane / 8)
              uint8_t* vb = buf + (lane >> 3) * 1024 + (lane & 7) * 2;
#pragma unroll
              for (int i = 0; i < 32; ++i)
                *reinterpret_cast<bf16*>(vb + (h2 + i) * 16) = __float2bfloat16_rn(v[i]);
            } else if (resid || epi.out_f32) {
              if (resid) {
                mbar_wait_warp(&xbar[2 * ew + bi], (xphase >> bi) & 1u);
                xphase ^= 1u << bi;
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
          if (gtr_c) GTR(18 + kc * 4);
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            if (region == 0) {
              tma_store_2d(&tmO, buf, n0 + c, srow0 + m0 + q * 32);
            } else {
              // K rows / Vt columns of the frame's memory slot, 8 tokens at a time (P % 8 == 0:
              // a group never straddles two frames); rows past the chunk are not stored
              for (int g8 = 0; g8 < 4; ++g8) {
                const int r0 = m0 + q * 32 + g8 * 8;
                if (r0 >= epi.M) break;
                const int t = r0 / epi.P, p = r0 - t * epi.P;
                const int krow = ((epi.first_slot + t) % epi.S) * epi.P + p;
                if (region == 1)
                  tma_store_2d(&tmX, buf + g8 * 1024, n0 + c - epi.D, epi.qkv_krow0 + krow);
                else
                  tma_store_2d(&tmV, buf + g8 * 1024, krow, epi.qkv_vrow0 + n0 + c - 2 * epi.D);
              }
            }
            bulk_commit();
            if (gtr_c) GTR(19 + kc * 4);
          }
        }
      } else {
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
      }
      // accumulator drained: one arrive per warp on the (leader's) barrier
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (PAIR) mbar_arrive_cluster(&tempty[acc], 0);
        else mbar_arrive(&tempty[acc]);
      }
      if (lt < 4 && ew == 0 && lane == 0) GTR(11 + lt);
    }
    if (TE && lane == 0) bulk_wait<0>();        // staging buffers stay valid until stored
  }
  tc_fence_before();
  if (PAIR) cluster_sync_all();   // no CTA leaves while its peer may still use its smem / TMEM
  else __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    if (PAIR) tmem_dealloc_pair(tmem, TMEM_COLS);
    else tmem_dealloc(tmem, TMEM_COLS);
  }
  if (threadIdx.x == 0) GTR(15);
  if (threadIdx.x == 0) time_end(epi.timing, gridDim.x);
}

template <int BN, int STAGES, bool PAIR, bool TE>
static cudaError_t launch_cfg(const CUtensorMap& a, const CUtensorMap& b, int brow0, int M, int N, int K,
                              const Epi& e, cudaStream_t st, const CUtensorMap* tmo, const CUtensorMap* tmx,
                              const CUtensorMap* tmv = nullptr) {
  using L = GemmSmem<BN, STAGES, PAIR, TE>;
  constexpr int CS = PAIR ? 2 : 1;
  auto kfn = gemm_tc_kernel<BN, STAGES, PAIR, TE>;
  int max_clusters = 0;
  cudaError_t err = ensure_kernel_setup(reinterpret_cast<const void*>(kfn), L::TOTAL, CS, 384, &max_clusters);
  if (err != cudaSuccess) return err;
  const int TM = PAIR ? 256 : 128;
  const int ntiles = ((M + TM - 1) / TM) * ((N + BN - 1) / BN) * (e.ksplit > 1 ? e.ksplit : 1);
  const int ncl = ntiles < max_clusters ? ntiles : max_clusters;
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
  return cudaLaunchKernelEx(&cfg, kfn, a, b, tmo ? *tmo : a, tmx ? *tmx : a, tmv ? *tmv : a, K, brow0, e);
}

// pair = 1: the CTA-pair kernel (M = 256 tiles; the W map's box must be 64 x BN/2).
cudaError_t launch_gemm_tc(const CUtensorMap& a, const CUtensorMap& b, int brow0, int M, int N, int K, int bn,
                           const Epi& e, cudaStream_t st, int pair, const CUtensorMap* tmo,
                           const CUtensorMap* tmx, const CUtensorMap* tmv) {
  if (tmo) {   // TMA-store epilogue (EPI_STORE / EPI_GELU / EPI_RESID / EPI_QKV)
    if (e.kind == EPI_NONE) return cudaErrorInvalidValue;
    if ((e.kind == EPI_RESID || e.kind == EPI_QKV) && !tmx) return cudaErrorInvalidValue;
    if (e.kind == EPI_QKV && (!tmv || e.out_f32 || e.win_pad || e.P % 8 || e.D % 64)) return cudaErrorInvalidValue;
    if (e.ksplit > 1) {   // split-K partials: raw fp32 stores, every split non-empty, whole tiles per split
      const int TM = pair ? 256 : 128, nk = (K + 63) / 64, kper = (nk + e.ksplit - 1) / e.ksplit;
      if (e.kind != EPI_STORE || !e.out_f32 || e.bias || e.pos || e.win_pad || (e.ksplit - 1) * kper >= nk ||
          e.kpad_rows < (M + TM - 1) / TM * TM)
        return cudaErrorInvalidValue;
    }
    if (pair) {
      switch (bn) {
        case 128: return launch_cfg<128, 6, true, true>(a, b, brow0, M, N, K, e, st, tmo, tmx, tmv);
        case 256: return launch_cfg<256, 4, true, true>(a, b, brow0, M, N, K, e, st, tmo, tmx, tmv);
        default: return cudaErrorInvalidValue;
      }
    }
    switch (bn) {
      case 64: return launch_cfg<64, 6, false, true>(a, b, brow0, M, N, K, e, st, tmo, tmx, tmv);
      case 128: return launch_cfg<128, 4, false, true>(a, b, brow0, M, N, K, e, st, tmo, tmx, tmv);
      case 256: return launch_cfg<256, 3, false, true>(a, b, brow0, M, N, K, e, st, tmo, tmx, tmv);
      default: return cudaErrorInvalidValue;
    }
  }
  if (pair) {
    switch (bn) {
      case 128: return launch_cfg<128, 8, true, false>(a, b, brow0, M, N, K, e, st, nullptr, nullptr);
      case 256: return launch_cfg<256, 6, true, false>(a, b, brow0, M, N, K, e, st, nullptr, nullptr);
      default: return cudaErrorInvalidValue;
    }
  }
  switch (bn) {
    case 64: return launch_cfg<64, 8, false, false>(a, b, brow0, M, N, K, e, st, nullptr, nullptr);
    case 128: return launch_cfg<128, 6, false, false>(a, b, brow0, M, N, K, e, st, nullptr, nullptr);
    case 256: return launch_cfg<256, 4, false, false>(a, b, brow0, M, N, K, e, st, nullptr, nullptr);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace vi
