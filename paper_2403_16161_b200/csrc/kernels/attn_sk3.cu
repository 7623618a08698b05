// Memory attention, persistent stream-K, 16 softmax warps in the 16x256b TMEM layout (the
// VI_ATTN_SK=3 variant; attn_sk2 stays the default: measured 2-5 % faster).
//
// attn_sk2.cu's schedule (two 128-query tiles per CTA, S/P and O in TMEM, P as the TMEM A
// operand of the PV MMA, per-key-half P hand-off, stream-K work split with owner merge)
// with a different softmax-thread mapping: each softmax warp owns 16 rows of a Q tile and
// all 128 keys of every key tile, read with tcgen05.ld.16x256b so that a row lives in 4
// lanes of the warp.  The row max and row sum are then two xor-shuffles instead of
// attn_sk2's exchange of row maxima between two warps through shared memory plus a named
// barrier, which sat on the per-Q-tile critical path S ready -> P written (measured with
// tools/micro/attn_micro: 456 of ~1720 clk).  Partial outputs of split units go through a
// thread-private, coalesced slot layout (no shared-memory staging in the merge).
// 576 threads: warps 0-15 softmax (Q tile = w / 8, TMEM lanes (w % 4) * 32 + ((w / 4) % 2)
// * 16 + [0, 16)), warp 16 TMA producer, warp 17 TMEM allocator + MMA issuer.
#include "kernels.h"

namespace vi {

// which of the 8 key groups of a half take exp2 by polynomial on the FMA pipe instead of
// MUFU.EX2 (MUFU: 16 lanes/clk/SM; the rest of the softmax issues on the FMA/ALU pipes)
#ifndef SK3_POLY_MASK
#define SK3_POLY_MASK 0x88
#endif
constexpr unsigned kSk3PolyMask = SK3_POLY_MASK;

template <int HD>
struct AttnSk3Smem {
  static constexpr int ST = 2;
  static constexpr int QB = 128 * HD * 2;
  static constexpr int KB = 128 * HD * 2;
  static constexpr int VB = HD * 128 * 2;
  static constexpr int Q_OFF = 0;
  static constexpr int K_OFF = 2 * QB;
  static constexpr int V_OFF = K_OFF + ST * KB;
  static constexpr int BAR_OFF = V_OFF + ST * VB;
  static constexpr int NBAR = 2 + 4 * ST + 2 + 4 + 2 + 2;
  static constexpr int STG_ROW = 80;                          // 64 B of bf16 + pad (conflict-free rows)
  static constexpr int STG_WARP = 16 * STG_ROW;
  static constexpr int STG_OFF = BAR_OFF + NBAR * 8 + 16;      // [16 warps][16 rows][80 B] output staging
  static constexpr int TOTAL = STG_OFF + 16 * STG_WARP + 1024;
};

__device__ __forceinline__ void sk3_key_tile(const KeySegs& s, int g, int& row0, int& nvalid, int& nskip) {
  int i = 0;
  while (i + 1 < s.n && g >= s.tile0[i + 1]) ++i;
  const int off = (g - s.tile0[i]) * 128;
  row0 = s.row0[i] + off;
  const int rem = s.len[i] - off;
  nvalid = rem < 128 ? rem : 128;
  nskip = off == 0 ? s.lead[i] : 0;
}

__device__ __forceinline__ void sk3_named_bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void sk3_bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// slice of the flattened work [0, W) owned by CTA c of G
__device__ __forceinline__ long long sk3_begin(long long W, int G, int c) { return W * c / G; }

template <int HD>
__global__ void __launch_bounds__(576, 1)
attn_sk3_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
               const __grid_constant__ CUtensorMap tvt, const AttnTC a) {
  using L = AttnSk3Smem<HD>;
  constexpr int ST = L::ST;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // 1 KB aligned, stays in .shared
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR_OFF);
  uint64_t* q_full = bars;
  uint64_t* q_empty = bars + 1;
  uint64_t* k_full = bars + 2;
  uint64_t* k_empty = k_full + ST;
  uint64_t* v_full = k_empty + ST;
  uint64_t* v_empty = v_full + ST;
  uint64_t* s_full = v_empty + ST;    // [2] per Q tile
  uint64_t* p_full = s_full + 2;      // [2 tiles][2 key halves]
  uint64_t* o_final = p_full + 4;     // [2] all PV of a segment done
  uint64_t* o_free = o_final + 2;     // [2] O read out by the epilogue
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_free + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int NT = a.segs.tile0[a.segs.n];
  const long long W = (long long)a.units * NT;
  const int G = gridDim.x, cta = blockIdx.x;
  const long long w_begin = sk3_begin(W, G, cta), w_end = sk3_begin(W, G, cta + 1);

  if (warp == 16 && lane == 0) {
    tma_prefetch(&tq);
    tma_prefetch(&tk);
    tma_prefetch(&tvt);
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int s = 0; s < ST; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(&s_full[t], 1);
      mbar_init(&p_full[2 * t], 8);                // one elected arrive per softmax warp of the tile
      mbar_init(&p_full[2 * t + 1], 8);
      mbar_init(&o_final[t], 1);
      mbar_init(&o_free[t], 256);
    }
    fence_barrier_init();
  }
  if (warp == 17) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) time_begin(a.timing);
  // debug timeline (VI_SK_TRACE): CTA 0, first segment's first 32 key tiles, 32 clock64 stamps per tile
  long long* const trc = (a.trace && cta == 0) ? a.trace : nullptr;

  if (warp == 16) {
    // TMA producer: the whole warp walks the schedule, one elected lane issues
    int jg = 0, sg = 0;
    for (long long w = w_begin; w < w_end; ++sg) {
      const int u = int(w / NT), ta = int(w - (long long)u * NT);
      const int tb = (int)((long long)NT < ta + (w_end - w) ? NT : ta + (w_end - w));
      const int h = u / a.npairs, q0 = (u - h * a.npairs) * 256;
      if (sg > 0) mbar_wait(q_empty, (sg - 1) & 1);
      if (elect_one()) {
        mbar_arrive_expect_tx(q_full, 2 * L::QB);
#pragma unroll
        for (int t = 0; t < 2; ++t)
#pragma unroll
          for (int at = 0; at < HD / 64; ++at)
            tma_load_2d(smem + L::Q_OFF + t * L::QB + at * 16384, &tq, q_full, h * HD + at * 64, a.q_row0 + q0 + t * 128);
      }
      __syncwarp();
      for (int j = ta; j < tb; ++j, ++jg) {
        int row0, nv, nskip;
        sk3_key_tile(a.segs, j, row0, nv, nskip);
        const int st = jg % ST;
        const uint32_t par = ((jg / ST) & 1) ^ 1;
        if (jg >= ST) mbar_wait(&k_empty[st], par);
        if (elect_one()) {
          uint8_t* sk = smem + L::K_OFF + st * L::KB;
          mbar_arrive_expect_tx(&k_full[st], L::KB);
#pragma unroll
          for (int at = 0; at < HD / 64; ++at)
            tma_load_2d(sk + at * 16384, &tk, &k_full[st], h * HD + at * 64, a.krow_base + row0);
        }
        __syncwarp();
        if (jg >= ST) mbar_wait(&v_empty[st], par);
        if (elect_one()) {
          uint8_t* sv = smem + L::V_OFF + st * L::VB;
          mbar_arrive_expect_tx(&v_full[st], L::VB);
#pragma unroll
          for (int at = 0; at < 2; ++at)
            tma_load_2d(sv + at * (HD * 128), &tvt, &v_full[st], row0 + at * 64, a.vrow_base + h * HD);
        }
        __syncwarp();
      }
      w += tb - ta;
    }
  } else if (warp == 17) {
    // The whole warp walks the schedule (warp-uniform control flow keeps the descriptors in
    // uniform registers); one elected lane issues each group of MMAs and commits.
    constexpr uint32_t idesc_s = idesc_bf16_f32(128, 128);
    constexpr uint32_t idesc_o = idesc_bf16_f32(128, HD);
    const uint64_t dq0 = sdesc_k_sw128(smem_u32(smem + L::Q_OFF));
    const uint64_t dk0 = sdesc_k_sw128(smem_u32(smem + L::K_OFF));
    const uint64_t dv0 = sdesc_k_sw128(smem_u32(smem + L::V_OFF));
    int jg = 0, sg = 0;
    for (long long w = w_begin; w < w_end; ++sg) {
      const int u = int(w / NT), ta = int(w - (long long)u * NT);
      const int tb = (int)((long long)NT < ta + (w_end - w) ? NT : ta + (w_end - w));
      const int n = tb - ta;
      mbar_wait(q_full, sg & 1);
      auto issue_pv = [&](int t, int j) {          // O_t (+)= P_t(j) V(j), j local to the segment
        const int g = jg + j, st = g % ST;
        if (t == 0) mbar_wait(&v_full[st], (g / ST) & 1);
        if (j == 0 && sg > 0) mbar_wait(&o_free[t], (sg - 1) & 1);   // previous segment's O read out
        const uint64_t dv = dv0 + uint64_t((st * L::VB) >> 4);
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          mbar_wait(&p_full[2 * t + hh], g & 1);
          tc_fence_after();
          if (elect_one()) {
            if (trc && g < 32) trc[g * 32 + 20 + hh * 6 + t] = clock64();
#pragma unroll
            for (int k4 = 0; k4 < 4; ++k4)
              umma_bf16_ts(tmem + 256 + t * 128, tmem + t * 128 + hh * 64 + k4 * 8,
                           dv + uint64_t((hh * (HD * 128) + k4 * 32) >> 4), idesc_o, (j | hh | k4) != 0);
            if (hh == 1 && t == 1) umma_commit(&v_empty[st]);
          }
          __syncwarp();
        }
      };
      auto issue_qk = [&](int t, int j) {          // S_t = Q_t K(j)^T
        const int g = jg + j, st = g % ST;
        if (t == 0) {
          mbar_wait(&k_full[st], (g / ST) & 1);
          tc_fence_after();
        }
        const uint64_t dk = dk0 + uint64_t((st * L::KB) >> 4), dq = dq0 + uint64_t((t * L::QB) >> 4);
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk) {
            const uint64_t off = uint64_t(((kk >> 2) * 16384 + (kk & 3) * 32) >> 4);
            umma_bf16_ss(tmem + t * 128, dq + off, dk + off, idesc_s, kk > 0);
          }
          umma_commit(&s_full[t]);
          if (trc && g < 32) trc[g * 32 + 24 + t] = clock64();
          if (t == 1) umma_commit(&k_empty[st]);
        }
        __syncwarp();
      };
      for (int j = 0; j < n; ++j)
        for (int t = 0; t < 2; ++t) {
          if (j > 0) issue_pv(t, j - 1);
          issue_qk(t, j);
        }
      if (elect_one()) umma_commit(q_empty);       // all QK of the segment issued: Q smem free when done
      __syncwarp();
      for (int t = 0; t < 2; ++t) {
        issue_pv(t, n - 1);
        if (elect_one()) umma_commit(&o_final[t]);
        __syncwarp();
      }
      jg += n;
      w += n;
    }
  } else if (warp < 16) {
    // Softmax warps: warp w handles Q tile t = w / 8 and TMEM lanes qd*32 + hf*16 + [0,16)
    // (qd = w % 4 is the warp's hardware lane quadrant), all 128 keys of every key tile.
    // With the 16x256b TMEM shape, thread (g = lane/4, c = lane%4) holds rows g and g+8 of
    // that 16-lane slab and keys 8k + 2c + {0,1}, k = 0..15: a row lives in 4 lanes of one
    // warp, so the row max and row sum are two xor-shuffles -- no shared memory, no barrier.
    const int t = warp >> 3;
    const int qd = warp & 3, hf = (warp >> 2) & 1;
    const int g4 = lane >> 2, c4 = lane & 3;
    const int rowA = qd * 32 + hf * 16 + g4;        // row within the Q tile; rowB = rowA + 8
    const uint32_t lane_off = uint32_t(qd * 32 + hf * 16) << 16;
    const uint32_t TS = tmem + t * 128 + lane_off, TO = tmem + 256 + t * 128 + lane_off;
    const int sid = warp * 32 + lane;               // 0..511
    const float2 cc = make_float2(a.scale_log2, a.scale_log2);
    uint8_t* stg = smem + L::STG_OFF + warp * L::STG_WARP;
    int jg = 0, sg = 0;
    for (long long w = w_begin; w < w_end; ++sg) {
      const int u = int(w / NT), ta = int(w - (long long)u * NT);
      const int tb = (int)((long long)NT < ta + (w_end - w) ? NT : ta + (w_end - w));
      const int n = tb - ta;
      const int h = u / a.npairs, q0 = (u - h * a.npairs) * 256;
      float mA = -INFINITY, mB = -INFINITY, lA = 0.f, lB = 0.f;   // lA/lB: this thread's keys only
      for (int j = 0; j < n; ++j) {
        const int g = jg + j;
        int row0, nv, nskip;
        sk3_key_tile(a.segs, ta + j, row0, nv, nskip);
        mbar_wait(&s_full[t], g & 1);
        tc_fence_after();
        const bool tr = trc && lane == 0 && g < 32;
        if (tr && warp == 8 * t) trc[g * 32 + 0 + t] = clock64();
        float s[64];                                // s[4k+i]: key 8k + 2c + (i&1), row A (i<2) / B
        tmem_ld_16x256b_x8(TS, reinterpret_cast<uint32_t*>(s));
        tmem_ld_16x256b_x8(TS + 64, reinterpret_cast<uint32_t*>(s + 32));
        tmem_wait_ld();
        if (tr && warp == 8 * t) trc[g * 32 + 22 + t] = clock64();
        if (nskip > 0 || nv < 128) {
#pragma unroll
          for (int i = 0; i < 64; ++i) {
            const int key = 8 * (i >> 2) + 2 * c4 + (i & 1);
            if (key < nskip || key >= nv) s[i] = -INFINITY;
          }
        }
        float xa[2] = {-INFINITY, -INFINITY}, xb[2] = {-INFINITY, -INFINITY};
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          xa[k & 1] = fmaxf(xa[k & 1], fmaxf(s[4 * k], s[4 * k + 1]));
          xb[k & 1] = fmaxf(xb[k & 1], fmaxf(s[4 * k + 2], s[4 * k + 3]));
        }
        float mxA = fmaxf(xa[0], xa[1]), mxB = fmaxf(xb[0], xb[1]);
        mxA = fmaxf(mxA, __shfl_xor_sync(0xffffffffu, mxA, 1));
        mxB = fmaxf(mxB, __shfl_xor_sync(0xffffffffu, mxB, 1));
        mxA = fmaxf(mxA, __shfl_xor_sync(0xffffffffu, mxA, 2));
        mxB = fmaxf(mxB, __shfl_xor_sync(0xffffffffu, mxB, 2));
        if (tr && warp == 8 * t) trc[g * 32 + 2 + t] = clock64();
        // lazy rescale: the reference max only moves when the row max grows by > 2^8
        const float rA = mxA * a.scale_log2, rB = mxB * a.scale_log2;
        const bool growA = rA > mA + 8.f, growB = rB > mB + 8.f;
        float alphaA = 1.f, alphaB = 1.f;
        if (growA) {
          alphaA = ex2(mA - rA);
          mA = rA;
        }
        if (growB) {
          alphaB = ex2(mB - rB);
          mB = rB;
        }
        const float2 nA = make_float2(-mA, -mA), nB = make_float2(-mB, -mB);
        float2 sumA = make_float2(0.f, 0.f), sumB = make_float2(0.f, 0.f);
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          uint32_t pk[16];                          // 16x128b layout: packed column 4k + c
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const int k = hh * 8 + kk;
            const float2 x0 = ffma2(make_float2(s[4 * k], s[4 * k + 1]), cc, nA);
            const float2 x1 = ffma2(make_float2(s[4 * k + 2], s[4 * k + 3]), cc, nB);
            float2 p0, p1;
            if ((kSk3PolyMask >> kk) & 1) {         // part of the exponentials on the FMA pipe
#ifdef SK3_POLY_DEG2
              p0 = exp2_poly2_deg2(x0);
              p1 = exp2_poly2_deg2(x1);
#else
              p0 = exp2_poly2(x0);
              p1 = exp2_poly2(x1);
#endif
            } else {
              p0.x = ex2(x0.x); p0.y = ex2(x0.y);
              p1.x = ex2(x1.x); p1.y = ex2(x1.y);
            }
            __nv_bfloat162 b0 = __floats2bfloat162_rn(p0.x, p0.y), b1 = __floats2bfloat162_rn(p1.x, p1.y);
            pk[2 * kk] = *reinterpret_cast<uint32_t*>(&b0);
            pk[2 * kk + 1] = *reinterpret_cast<uint32_t*>(&b1);
            sumA = fadd2(sumA, p0);
            sumB = fadd2(sumB, p1);
          }
          if (tr && warp == 8 * t) trc[g * 32 + 28 + 2 * hh + t] = clock64();
          tmem_st_16x128b_x8(TS + hh * 64, pk);     // P keys [hh*64, +64) -> packed cols [hh*64, +32)
          if (hh == 0 && j > 0 && __any_sync(0xffffffffu, growA || growB)) {
            // O rescale before PV(j) may start; PV(j-1) is complete (s_full(j) implies it)
#pragma unroll 1
            for (int cb = 0; cb < HD; cb += 32) {
              float o[16];
              tmem_ld_16x256b_x4(TO + cb, reinterpret_cast<uint32_t*>(o));
              tmem_wait_ld();
#pragma unroll
              for (int i = 0; i < 16; ++i) o[i] *= (i & 2) ? alphaB : alphaA;
              tmem_st_16x256b_x4(TO + cb, reinterpret_cast<uint32_t*>(o));
            }
          }
          tmem_wait_st();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&p_full[2 * t + hh]);
          if (tr) trc[g * 32 + 4 + t * 8 + hh * 4 + (warp & 3)] = clock64();
        }
        lA = lA * alphaA + (sumA.x + sumA.y);
        lB = lB * alphaB + (sumB.x + sumB.y);
      }
      // ---- segment epilogue: rows A/B of this warp's 16-lane slab, all HD columns
      mbar_wait(&o_final[t], sg & 1);
      tc_fence_after();
      lA += __shfl_xor_sync(0xffffffffu, lA, 1);
      lB += __shfl_xor_sync(0xffffffffu, lB, 1);
      lA += __shfl_xor_sync(0xffffffffu, lA, 2);
      lB += __shfl_xor_sync(0xffffffffu, lB, 2);
      const float lseA = mA + __log2f(lA), lseB = mB + __log2f(lB);
      const int rA256 = t * 128 + rowA, rB256 = rA256 + 8;     // rows in the CTA's 256-row slot
      const int rbase = q0 + t * 128 + qd * 32 + hf * 16;      // first output row of the slab
      // 32 O columns [cb, cb+32) (registers of tmem_ld_16x256b_x4) -> bf16 rows of the output
      auto write_out32 = [&](int cb, const float* f, float sa, float sb) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int col = 8 * k + 2 * c4;
          *reinterpret_cast<uint32_t*>(stg + g4 * L::STG_ROW + col * 2) = pack_bf16(f[4 * k] * sa, f[4 * k + 1] * sa);
          *reinterpret_cast<uint32_t*>(stg + (g4 + 8) * L::STG_ROW + col * 2) =
              pack_bf16(f[4 * k + 2] * sb, f[4 * k + 3] * sb);
        }
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 2; ++i) {              // 16 rows x 64 B: 4 lanes per row, 16 B each
          const int rr = i * 8 + (lane >> 2), part = lane & 3;
          const uint4 v = *reinterpret_cast<const uint4*>(stg + rr * L::STG_ROW + part * 16);
          if (rbase + rr < a.Nq)
            *reinterpret_cast<uint4*>(a.o + (size_t)(rbase + rr) * a.o_ld + (size_t)h * a.o_hs + cb + part * 8) = v;
        }
        __syncwarp();
      };
      float4* const slot = reinterpret_cast<float4*>(a.spart);
      if (ta > 0) {
        // continuation piece: normalised partial O -> this CTA's slot (thread-private,
        // interleaved for coalescing), log2-sum-exp per row, then raise the flag
        const float iA = 1.f / lA, iB = 1.f / lB;
#pragma unroll 1
        for (int cb = 0; cb < HD; cb += 32) {
          float f[16];
          tmem_ld_16x256b_x4(TO + cb, reinterpret_cast<uint32_t*>(f));
          tmem_wait_ld();
#pragma unroll
          for (int q = 0; q < 4; ++q)
            slot[((size_t)cta * (HD / 8) + (cb / 8 + q)) * 512 + sid] =
                make_float4(f[4 * q] * iA, f[4 * q + 1] * iA, f[4 * q + 2] * iB, f[4 * q + 3] * iB);
        }
        tc_fence_before();
        mbar_arrive(&o_free[t]);
        if (c4 == 0) {
          a.slse[(size_t)cta * 256 + rA256] = lseA;
          a.slse[(size_t)cta * 256 + rB256] = lseB;
        }
        sk3_bar_sync(9, 512);                         // every row of the slot written (CTA scope) ...
        if (threadIdx.x == 0) {                      // ... then one cumulative gpu-scope release
          __threadfence();
          atomicExch(&a.sflag[cta], 1);
        }
      } else if (tb < NT) {
        // owner of a split unit (always the last segment of this CTA): merge the pieces of
        // CTAs cta+1 .. (the unit's last tile) in CTA order
        const long long unit_end = (long long)(u + 1) * NT;
        int last = cta + 1;
        while (last + 1 < G && sk3_begin(W, G, last + 1) < unit_end) ++last;
        const int np = last - cta;
        for (int k = lane; k < np; k += 32) {
          const int* fl = a.sflag + cta + 1 + k;
          while (*reinterpret_cast<const volatile int*>(fl) == 0) __nanosleep(32);
        }
        __syncwarp();
        __threadfence();
        float mxA2 = lseA, mxB2 = lseB;
        for (int k = 0; k < np; ++k) {
          mxA2 = fmaxf(mxA2, __ldcg(a.slse + (size_t)(cta + 1 + k) * 256 + rA256));
          mxB2 = fmaxf(mxB2, __ldcg(a.slse + (size_t)(cta + 1 + k) * 256 + rB256));
        }
        const float woA = ex2(lseA - mxA2), woB = ex2(lseB - mxB2);
        float wsA = woA, wsB = woB;
        for (int k = 0; k < np; ++k) {
          wsA += ex2(__ldcg(a.slse + (size_t)(cta + 1 + k) * 256 + rA256) - mxA2);
          wsB += ex2(__ldcg(a.slse + (size_t)(cta + 1 + k) * 256 + rB256) - mxB2);
        }
        const float sA = woA / lA / wsA, sB = woB / lB / wsB;     // own (unnormalised) O weight
#pragma unroll 1
        for (int cb = 0; cb < HD; cb += 32) {
          float f[16];
          tmem_ld_16x256b_x4(TO + cb, reinterpret_cast<uint32_t*>(f));
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; ++i) f[i] *= (i & 2) ? sB : sA;
#pragma unroll 1
          for (int k = 0; k < np; ++k) {
            const int pc = cta + 1 + k;
            const float wA = ex2(__ldcg(a.slse + (size_t)pc * 256 + rA256) - mxA2) / wsA;
            const float wB = ex2(__ldcg(a.slse + (size_t)pc * 256 + rB256) - mxB2) / wsB;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const float4 v = __ldcg(slot + ((size_t)pc * (HD / 8) + (cb / 8 + q)) * 512 + sid);
              f[4 * q] += wA * v.x;
              f[4 * q + 1] += wA * v.y;
              f[4 * q + 2] += wB * v.z;
              f[4 * q + 3] += wB * v.w;
            }
          }
          write_out32(cb, f, 1.f, 1.f);
        }
        tc_fence_before();
        mbar_arrive(&o_free[t]);
        sk3_bar_sync(11, 512);                       // every row has read the slots
        for (int k = threadIdx.x; k < np; k += 512) a.sflag[cta + 1 + k] = 0;
      } else {
        const float iA = 1.f / lA, iB = 1.f / lB;
#pragma unroll 1
        for (int cb = 0; cb < HD; cb += 32) {
          float f[16];
          tmem_ld_16x256b_x4(TO + cb, reinterpret_cast<uint32_t*>(f));
          tmem_wait_ld();
          write_out32(cb, f, iA, iB);
        }
        tc_fence_before();
        mbar_arrive(&o_free[t]);
      }
      jg += n;
      w += n;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) time_end(a.timing, gridDim.x);
  if (warp == 17) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int HD>
static cudaError_t launch_sk3_hd(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tvt,
                                const AttnTC& a, int grid, cudaStream_t st) {
  using L = AttnSk3Smem<HD>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(attn_sk3_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::TOTAL);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(576);
  cfg.dynamicSmemBytes = L::TOTAL;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;     // owners wait on other CTAs: all must be resident
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, attn_sk3_kernel<HD>, tq, tk, tvt, a);
}

cudaError_t launch_attn_sk3(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tvt, const AttnTC& a,
                           int grid, cudaStream_t st) {
  if (a.hd == 128) return launch_sk3_hd<128>(tq, tk, tvt, a, grid, st);
  if (a.hd == 64) return launch_sk3_hd<64>(tq, tk, tvt, a, grid, st);
  return cudaErrorInvalidValue;
}

}  // namespace vi
