// Memory attention: per head h,
//   O_h = softmax(Q_h K_h^T / sqrt(d)) V_h
// where the queries are the new frames only and the keys/values are the rows
// of every VALID slot of the layer's ring-buffer memory: the chunk itself plus the
// resident frames f-M .. f-1 (Eq. 3).  Softmax is exact (max-subtracted,
// online over key tiles; reading Q14), key order = slot order (permutation invariant).
//
// Kernels here: the fp32 SIMT path (attn_simt_f32_kernel, BASELINE configs[0]) and the
// small-chunk tensor-core path (attn_tc2_kernel: fixed KV split, partials merged by
// attn_combine_kernel in a fixed order -- deterministic, no atomics).  The large-chunk
// default is the persistent stream-K kernel of attn_sk2.cu.
#include "kernels.h"

namespace vi {

// ------------------------------------------------------------------ SIMT fp32 path
__global__ void attn_simt_f32_kernel(AttnArgs a) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= a.Nq * a.H) return;
  const int q = warp / a.H, h = warp - q * a.H;
  const int R = a.hd / 32;                    // hd % 32 == 0, hd <= 128
  const float* Q = reinterpret_cast<const float*>(a.q) + (size_t)q * a.D + h * a.hd;
  const float* K = reinterpret_cast<const float*>(a.kslab);
  const float* Vt = reinterpret_cast<const float*>(a.vtslab);
  const size_t ld = (size_t)a.vt_ld;
  float qv[4], acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int i = 0; i < R; ++i) qv[i] = Q[lane + 32 * i];
  float m = -INFINITY, l = 0.f;
  for (int s = 0; s < a.S; ++s) {
    if (!((a.valid >> s) & 1ull)) continue;
    for (int p = 0; p < a.P; ++p) {
      const size_t row = (size_t)s * a.P + p;
      const float* kr = K + row * a.D + h * a.hd;
      float dot = 0.f;
      for (int i = 0; i < R; ++i) dot = fmaf(qv[i], kr[lane + 32 * i], dot);
#pragma unroll
      for (int o = 16; o; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
      const float sc = dot * a.scale_log2;
      const float mn = fmaxf(m, sc);
      const float alpha = exp2f(m - mn), pe = exp2f(sc - mn);
      l = l * alpha + pe;
      for (int i = 0; i < R; ++i) acc[i] = acc[i] * alpha + pe * Vt[(size_t)(h * a.hd + lane + 32 * i) * ld + row];
      m = mn;
    }
  }
  float* O = reinterpret_cast<float*>(a.o) + (size_t)q * a.D + h * a.hd;
  for (int i = 0; i < R; ++i) O[lane + 32 * i] = acc[i] / l;
}

cudaError_t launch_attn_simt_f32(const AttnArgs& a, cudaStream_t st) {
  const int warps = a.Nq * a.H;
  attn_simt_f32_kernel<<<(warps * 32 + 255) / 256, 256, 0, st>>>(a);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ tcgen05 bf16 path

// Tile g of the valid key space: keys row0 .. row0+127 of the slab, of which
// [nskip, nvalid) belong to valid slots (the rest is masked to -inf).
// window attention: output token row of local query q of window w, or -1 for padding /
// rows beyond the chunk
__device__ __forceinline__ int win_out_row(const AttnTC& a, int w, int q) {
  if (q >= a.win_nq) return -1;
  const int t = q / a.win_pad, i = q - t * a.win_pad;
  if (i >= a.win_real) return -1;
  const int oy = (w / a.win_cols) * a.win_h + i / a.win_w, ox = (w % a.win_cols) * a.win_w + i % a.win_w;
  const int tok = oy * a.ow + ox;
  return a.win_split_rows ? t * a.win_split_rows + tok - a.win_part * a.win_split_rows : t * a.P + tok;
}

__device__ __forceinline__ void key_tile(const KeySegs& s, int g, int& row0, int& nvalid, int& nskip) {
  int i = 0;
  while (i + 1 < s.n && g >= s.tile0[i + 1]) ++i;
  const int off = (g - s.tile0[i]) * 128;
  row0 = s.row0[i] + off;
  const int rem = s.len[i] - off;
  nvalid = rem < 128 ? rem : 128;
  nskip = off == 0 ? s.lead[i] : 0;
}


// ------------------------------------------------------------------ v2: two Q tiles per CTA
// attn_tc2_kernel: one CTA = (pair of 128-query tiles, head, KV split), 384 threads:
//   warps 0-3 : softmax of Q tile 0 (thread = query row = TMEM lane)
//   warps 4-7 : softmax of Q tile 1
//   warp 8    : TMA producer (Q tiles once; K / transposed-V tiles, 2-stage ring)
//   warp 9    : MMA issuer
//   warp 10   : TMEM allocator (512 cols: S0/P0 | S1/P1 | O0 | O1)
// Each K/V tile fetched once serves 256 queries.  P is written back into the TMEM
// columns of its own S tile (bf16 pairs) and is the A operand (from TMEM) of O += P V.
// Tensor-core order per KV tile j:  PV(0,j-1) QK(0,j) PV(1,j-1) QK(1,j), so while one
// softmax warpgroup works on tile j the tensor core runs the other tile's MMAs.
// tcgen05 ops of one thread complete in order, so the commit of QK(t,j) also proves
// PV(t,j-1) finished: the softmax may then overwrite P(t) and rescale O(t) safely.
// Running max update is lazy (only when it grows by > 8 in log2 units), exact either way.
template <int HD>
struct Attn2Smem {
  static constexpr int ST = 2;
  static constexpr int QB = 128 * HD * 2;
  static constexpr int KB = 128 * HD * 2;
  static constexpr int VB = HD * 128 * 2;
  static constexpr int Q_OFF = 0;
  static constexpr int K_OFF = 2 * QB;
  static constexpr int V_OFF = K_OFF + ST * KB;
  static constexpr int BAR_OFF = V_OFF + ST * VB;
  static constexpr int NBAR = 1 + 4 * ST + 2 + 4 + 2;
  static constexpr int TOTAL = BAR_OFF + NBAR * 8 + 16 + 1024;
};

// One softmax warpgroup per Q tile (thread = row, all 128 keys).
#ifndef TC2_TRACE
#define TC2_TRACE 0   // per-CTA globaltimer stamps into AttnTC::cta_trace (micro-benchmarks only)
#endif
template <int HD>
__global__ void __launch_bounds__(384, 1)
attn_tc2_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                const __grid_constant__ CUtensorMap tvt, const AttnTC a) {
  using L = Attn2Smem<HD>;
  constexpr int ST = L::ST;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // 1 KB aligned, stays in .shared
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR_OFF);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;
  uint64_t* k_empty = k_full + ST;
  uint64_t* v_full = k_empty + ST;
  uint64_t* v_empty = v_full + ST;
  uint64_t* s_full = v_empty + ST;    // [2] per Q tile
  uint64_t* p_full = s_full + 2;      // [2 tiles][2 key halves]
  uint64_t* o_final = p_full + 4;     // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_final + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int win_l = a.win_n ? int(blockIdx.x) / a.win_npw : 0;                 // window of this launch's range
  const int win = a.win0 + win_l;                                                // window (0 if global)
  const int q0 = (a.win_n ? int(blockIdx.x) % a.win_npw : int(blockIdx.x)) * 256, h = blockIdx.y, z = blockIdx.z;
  const int wq = win * a.win_qstride, wk = win * a.win_kstride;                  // window row offsets
  const int ntiles = a.segs.tile0[a.segs.n];
  const int t_begin = z * a.tiles_per_split;
  int t_end = t_begin + a.tiles_per_split;
  if (t_end > ntiles) t_end = ntiles;
  const int n = t_end > t_begin ? t_end - t_begin : 0;
  long long* const ct =
      (TC2_TRACE && a.cta_trace)
          ? a.cta_trace + (size_t)((blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x) * 8
          : nullptr;
  if (ct && threadIdx.x == 0) ct[0] = (long long)globaltimer();

  if (warp == 8 && lane == 0) {
    tma_prefetch(&tq);
    tma_prefetch(&tk);
    tma_prefetch(&tvt);
    mbar_init(q_full, 1);
    for (int s = 0; s < ST; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(&s_full[t], 1);
      mbar_init(&p_full[2 * t], 128);
      mbar_init(&p_full[2 * t + 1], 128);
      mbar_init(&o_final[t], 1);
    }
    fence_barrier_init();
  }
  if (warp == 10) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // the set-up above overlaps the previous kernel's tail (programmatic dependent launch); the
  // combine kernel may launch now (it waits for this grid's completion before reading)
  griddep_wait();
  griddep_launch();
  if (threadIdx.x == 0) time_begin(a.timing);
  if (ct && threadIdx.x == 0) ct[1] = (long long)globaltimer();

  if (warp == 8) {
    if (lane == 0 && n > 0) {
      mbar_arrive_expect_tx(q_full, 2 * L::QB);
#pragma unroll
      for (int t = 0; t < 2; ++t)
#pragma unroll
        for (int at = 0; at < HD / 64; ++at)
          tma_load_2d(smem + L::Q_OFF + t * L::QB + at * 16384, &tq, q_full, h * HD + at * 64,
                      a.q_row0 + wq + q0 + t * 128);
      for (int jj = 0; jj < n; ++jj) {
        int row0, nv, nskip;
        key_tile(a.segs, t_begin + jj, row0, nv, nskip);
        const int st = jj % ST;
        const uint32_t par = ((jj / ST) & 1) ^ 1;
        if (jj >= ST) mbar_wait(&k_empty[st], par);
        uint8_t* sk = smem + L::K_OFF + st * L::KB;
        mbar_arrive_expect_tx(&k_full[st], L::KB);
#pragma unroll
        for (int at = 0; at < HD / 64; ++at)
          tma_load_2d(sk + at * 16384, &tk, &k_full[st], h * HD + at * 64, a.krow_base + wk + row0);
        if (jj >= ST) mbar_wait(&v_empty[st], par);
        uint8_t* sv = smem + L::V_OFF + st * L::VB;
        mbar_arrive_expect_tx(&v_full[st], L::VB);
#pragma unroll
        for (int at = 0; at < 2; ++at)
          tma_load_2d(sv + at * (HD * 128), &tvt, &v_full[st], wk + row0 + at * 64, a.vrow_base + h * HD);
      }
    }
  } else if (warp == 9) {
    if (lane == 0 && n > 0) {
      constexpr uint32_t idesc_s = idesc_bf16_f32(128, 128);
      constexpr uint32_t idesc_o = idesc_bf16_f32(128, HD);
      const uint32_t sq = smem_u32(smem + L::Q_OFF);
      mbar_wait(q_full, 0);
      const bool trm = a.trace && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0;
      auto issue_pv = [&](int t, int j) {            // O_t (+)= P_t(j) V(j), one key half at a time
        const int st = j % ST;
        if (trm && j < 32) a.trace[j * 32 + 24 + t * 4] = clock64();
        if (t == 0) mbar_wait(&v_full[st], (j / ST) & 1);
        const uint32_t sv = smem_u32(smem + L::V_OFF + st * L::VB);
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          mbar_wait(&p_full[2 * t + hh], j & 1);
          if (trm && j < 32) a.trace[j * 32 + 25 + t * 4 + hh] = clock64();
          tc_fence_after();
#pragma unroll
          for (int k4 = 0; k4 < 4; ++k4) {
            const int kk = hh * 4 + k4;
            const uint32_t offv = hh * (HD * 128) + k4 * 32;
            umma_bf16_ts(tmem + 256 + t * 128, tmem + t * 128 + kk * 8, sdesc_k_sw128(sv + offv), idesc_o,
                         (j | kk) != 0);
          }
        }
        if (t == 1) umma_commit(&v_empty[st]);
      };
      auto issue_qk = [&](int t, int j) {            // S_t = Q_t K(j)^T
        const int st = j % ST;
        if (t == 0) {
          mbar_wait(&k_full[st], (j / ST) & 1);
          tc_fence_after();
        }
        const uint32_t sk = smem_u32(smem + L::K_OFF + st * L::KB);
        const uint32_t sqt = sq + t * L::QB;
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          umma_bf16_ss(tmem + t * 128, sdesc_k_sw128(sqt + off), sdesc_k_sw128(sk + off), idesc_s, kk > 0);
        }
        umma_commit(&s_full[t]);
        if (t == 1) umma_commit(&k_empty[st]);
        if (trm && j > 0 && j <= 32) a.trace[(j - 1) * 32 + 27 + t * 4] = clock64();
      };
      for (int j = 0; j < n; ++j) {
        for (int t = 0; t < 2; ++t) {
          if (j > 0) issue_pv(t, j - 1);
          issue_qk(t, j);
        }
      }
      for (int t = 0; t < 2; ++t) {
        issue_pv(t, n - 1);
        umma_commit(&o_final[t]);
      }
    }
  } else if (warp < 8) {
    const int t = warp >> 2;                          // Q tile of this warpgroup
    const int qd = warp & 3;                          // TMEM lane quadrant
    const uint32_t lane_off = uint32_t(qd * 32) << 16;
    const uint32_t TS = tmem + t * 128 + lane_off, TO = tmem + 256 + t * 128 + lane_off;
    float m_use = -INFINITY, l = 0.f;
    for (int jj = 0; jj < n; ++jj) {
      int row0, nv, nskip;
      key_tile(a.segs, t_begin + jj, row0, nv, nskip);
      const bool tr = a.trace && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && lane == 0 && jj < 32;
      mbar_wait_warp(&s_full[t], jj & 1);
      if (ct && jj == 0 && threadIdx.x == 0) ct[2] = (long long)globaltimer();
      if (tr) a.trace[jj * 32 + t * 12 + qd] = clock64();
      tc_fence_after();
      float s[128];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld32(TS + c * 32, reinterpret_cast<uint32_t*>(s + c * 32));
      tmem_wait_ld();
      float mx[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) mx[i] = -INFINITY;
      if (nv < 128 || nskip > 0) {
#pragma unroll
        for (int i = 0; i < 128; ++i)
          if (i >= nv || i < nskip) s[i] = -INFINITY;
      }
      if (a.win_pad > a.win_real) {                   // window padding keys (index % pad >= real)
        uint32_t pm[4] = {0u, 0u, 0u, 0u};
        for (int k = a.win_real - row0 % a.win_pad; k < 128; k += a.win_pad)
          for (int e = k < 0 ? 0 : k; e < k + a.win_pad - a.win_real && e < 128; ++e) pm[e >> 5] |= 1u << (e & 31);
#pragma unroll
        for (int i = 0; i < 128; ++i)
          if ((pm[i >> 5] >> (i & 31)) & 1u) s[i] = -INFINITY;
      }
#pragma unroll
      for (int i = 0; i < 128; ++i) mx[i & 7] = fmaxf(mx[i & 7], s[i]);
      const float rmax = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])),
                               fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7]))) * a.scale_log2;
      // lazy rescale: keep the old reference max unless the row max grew by > 8 (x256)
      const bool grow = rmax > m_use + 8.f;
      float alpha = 1.f;
      if (grow) {
        alpha = ex2(m_use - rmax);
        m_use = rmax;
      }
      if (__any_sync(0xffffffffu, grow) && jj > 0) {  // O(t) is idle here (see above)
#pragma unroll 1
        for (int c = 0; c < HD; c += 32) {
          uint32_t r[32];
          tmem_ld32(TO + c, r);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
          tmem_st32(TO + c, r);
        }
      }
      // p = 2^(s c - m): 10 of every 16 pairs on the MUFU (ex2), 6 by polynomial on the FMA
      // pipe (balances MUFU time and issue slots); packed FFMA2 / FADD2.  P goes back to
      // TMEM 32 keys (16 packed columns) at a time and each key half is handed to the MMA
      // warp as soon as it is written, so PV on keys 0-63 overlaps the exps of 64-127.
      const float2 cc = make_float2(a.scale_log2, a.scale_log2), mm = make_float2(-m_use, -m_use);
      float2 sum[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) sum[i] = make_float2(0.f, 0.f);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t pk[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const int i = c * 16 + k;
          const float2 x = ffma2(make_float2(s[2 * i], s[2 * i + 1]), cc, mm);
          float2 p;
          if (k % 5 >= 3) {
            p = exp2_poly2(x);
          } else {
            p.x = ex2(x.x);
            p.y = ex2(x.y);
          }
          __nv_bfloat162 b = __floats2bfloat162_rn(p.x, p.y);
          pk[k] = *reinterpret_cast<uint32_t*>(&b);
          sum[k & 3] = fadd2(sum[k & 3], p);
        }
        tmem_st16(TS + c * 16, pk);
        if (c & 1) {
          tmem_wait_st();
          tc_fence_before();
          if (tr) a.trace[jj * 32 + t * 12 + 4 + (c >> 1) * 4 + qd] = clock64();
          mbar_arrive(&p_full[2 * t + (c >> 1)]);
        }
      }
      const float2 s01 = fadd2(fadd2(sum[0], sum[1]), fadd2(sum[2], sum[3]));
      l = l * alpha + (s01.x + s01.y);
    }
    // epilogue
    const int q = q0 + t * 128 + qd * 32 + lane;
    // output row (global: q itself; windows: the token row of (frame, window index), -1 = none)
    const int orow = a.win_n ? win_out_row(a, win, q) : (q < a.Nq ? q : -1);
    const int qp = win_l * a.win_qstride + q;         // row of the KV-split partials (launch-local windows)
    if (n > 0) {
      mbar_wait_warp(&o_final[t], 0);
      tc_fence_after();
    }
    if (ct && threadIdx.x == 0) ct[3] = (long long)globaltimer();
    const float inv = n > 0 ? 1.f / l : 0.f;
    if (a.nsplit == 1) {
#pragma unroll 1
      for (int c = 0; c < HD; c += 32) {
        uint32_t r[32];
        tmem_ld32(TO + c, r);
        tmem_wait_ld();
        if (orow >= 0) {
          const float* f = reinterpret_cast<const float*>(r);
          uint4* dst = reinterpret_cast<uint4*>(a.o + (size_t)orow * a.o_ld + (size_t)h * a.o_hs + c);
#pragma unroll
          for (int i = 0; i < 4; ++i)
            dst[i] = make_uint4(pack_bf16(f[8 * i] * inv, f[8 * i + 1] * inv), pack_bf16(f[8 * i + 2] * inv, f[8 * i + 3] * inv),
                                pack_bf16(f[8 * i + 4] * inv, f[8 * i + 5] * inv), pack_bf16(f[8 * i + 6] * inv, f[8 * i + 7] * inv));
        }
      }
    } else {
      // the normalised partial row (bf16, as attn_sk2's pieces) leaves through shared memory as
      // one bulk copy (direct stores put 32 rows in every warp instruction and ran at one L2
      // sector per clock: 4.5 us per CTA for fp32 rows).  Staging: tile t's rows at a padded
      // pitch (a warp's 16-B stores cover 8 bank groups) in the Q / K buffers, free once
      // o_final[t] is seen (the MMAs complete in issue order and QK(1, n-1) precedes the commit
      // of O(0)).
      constexpr int PITCH = HD * 2 + 16;
      static_assert(2 * 128 * PITCH <= L::V_OFF, "partial staging exceeds the Q / K buffers");
      uint8_t* srow = smem + (size_t)(t * 128 + qd * 32 + lane) * PITCH;
#pragma unroll 1
      for (int c = 0; c < HD; c += 32) {
        uint32_t r[32];
        if (n > 0) {
          tmem_ld32(TO + c, r);
          tmem_wait_ld();
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) r[i] = 0u;
        }
        const float* f = reinterpret_cast<const float*>(r);
        uint4* dst = reinterpret_cast<uint4*>(srow + c * 2);
#pragma unroll
        for (int i = 0; i < 4; ++i)
          dst[i] = make_uint4(pack_bf16(f[8 * i] * inv, f[8 * i + 1] * inv), pack_bf16(f[8 * i + 2] * inv, f[8 * i + 3] * inv),
                              pack_bf16(f[8 * i + 4] * inv, f[8 * i + 5] * inv), pack_bf16(f[8 * i + 6] * inv, f[8 * i + 7] * inv));
      }
      if (orow >= 0) {
        fence_proxy_async_smem();
        bulk_s2g(a.opart + ((size_t)z * a.Nq + qp) * a.D + h * HD, srow, HD * 2);
        bulk_commit();
        a.lse[((size_t)z * a.H + h) * a.Nq + qp] = n > 0 ? m_use + __log2f(l) : -INFINITY;
        bulk_wait_read<0>();
      }
    }
    if (ct && threadIdx.x == 0) ct[4] = (long long)globaltimer();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 10) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
  if (ct && threadIdx.x == 0) ct[5] = (long long)globaltimer();
  if (threadIdx.x == 0) time_end(a.timing, gridDim.x * gridDim.y * gridDim.z);
}

template <int HD>
static cudaError_t launch2_hd(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tvt, const AttnTC& a,
                              cudaStream_t st) {
  using L = Attn2Smem<HD>;
  cudaError_t e = ensure_kernel_setup(reinterpret_cast<const void*>(attn_tc2_kernel<HD>), L::TOTAL);
  if (e != cudaSuccess) return e;
  dim3 grid(a.win_n ? a.win_n * a.win_npw : (a.Nq + 255) / 256, a.H, a.nsplit);
  return pdl_launch(attn_tc2_kernel<HD>, grid, dim3(384), L::TOTAL, st, tq, tk, tvt, a);
}

cudaError_t launch_attn_tc2(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tvt, const AttnTC& a,
                            cudaStream_t st) {
  if (a.hd == 128) return launch2_hd<128>(tq, tk, tvt, a, st);
  if (a.hd == 64) return launch2_hd<64>(tq, tk, tvt, a, st);
  return cudaErrorInvalidValue;
}

// Merge of the KV-split partials: O = sum_z 2^(lse_z - M) O_z / sum_z 2^(lse_z - M), z in
// split order (deterministic).  A group of hd / 4 lanes per (query row, head): lane z of the
// group loads lse_z (broadcast by shuffles), every lane issues its <= kMaxZ partial loads
// (4 bf16 columns each) before the sums.  Partial rows are window-major for windows.
constexpr int kMaxZ = 16;
__global__ void __launch_bounds__(256) attn_combine_kernel(const AttnTC a) {
  griddep_wait();
  if (threadIdx.x == 0) time_begin(a.combine_timing);
  griddep_launch();
  const int G = a.hd / 4;                                   // lanes per row: 32 (d 128) or 16 (d 64)
  const int sub = (threadIdx.x & 31) % G;
  const int r = (blockIdx.x * blockDim.x + threadIdx.x) / G;
  const bool live = r < a.Nq * a.H;
  const int h = live ? r % a.H : 0, q = live ? r / a.H : 0;
  const float lme = (live && sub < a.nsplit) ? __ldcg(a.lse + ((size_t)sub * a.H + h) * a.Nq + q) : -INFINITY;
  const uint2* src = reinterpret_cast<const uint2*>(a.opart + (size_t)q * a.D + h * a.hd) + sub;
  const size_t zstride = (size_t)a.Nq * a.D / 4;            // one split's partials, in uint2
  uint2 u[kMaxZ];
#pragma unroll
  for (int z = 0; z < kMaxZ; ++z) u[z] = (live && z < a.nsplit) ? __ldcg(src + z * zstride) : make_uint2(0u, 0u);
  float mx = lme;
  for (int o = G / 2; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o, G));
  float acc[4] = {0.f, 0.f, 0.f, 0.f}, wsum = 0.f;
#pragma unroll
  for (int z = 0; z < kMaxZ; ++z) {
    const float lz = __shfl_sync(0xffffffffu, lme, z, G);
    if (lz == -INFINITY) continue;
    const float w = exp2f(lz - mx);
    const float2 v01 = unpack_bf16x2(u[z].x), v23 = unpack_bf16x2(u[z].y);
    wsum += w;
    acc[0] += w * v01.x; acc[1] += w * v01.y; acc[2] += w * v23.x; acc[3] += w * v23.y;
  }
  const int orow = !live ? -1 : a.win_n ? win_out_row(a, a.win0 + q / a.win_qstride, q % a.win_qstride) : q;
  if (orow >= 0) {
    const float inv = 1.f / wsum;
    *reinterpret_cast<uint2*>(a.o + (size_t)orow * a.o_ld + (size_t)h * a.o_hs + sub * 4) =
        make_uint2(pack_bf16(acc[0] * inv, acc[1] * inv), pack_bf16(acc[2] * inv, acc[3] * inv));
  }
  if (a.combine_timing) {
    __syncthreads();
    if (threadIdx.x == 0) time_end(a.combine_timing, gridDim.x);
  }
}

cudaError_t launch_attn_combine(const AttnTC& a, cudaStream_t st) {
  if (a.nsplit > kMaxZ || (a.hd != 128 && a.hd != 64)) return cudaErrorInvalidValue;
  const size_t threads = (size_t)a.Nq * a.H * (a.hd / 4);
  const unsigned blocks = unsigned((threads + 255) / 256);
  return pdl_launch(attn_combine_kernel, dim3(blocks ? blocks : 1), dim3(256), 0, st, a);
}

}  // namespace vi
