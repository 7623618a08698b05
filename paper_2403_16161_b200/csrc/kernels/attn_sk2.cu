// Memory attention, persistent stream-K, COLUMN-SPLIT softmax (the default bf16 kernel).
//
// attn_sk.cu's design (two 128-query tiles per CTA, S/P and O in TMEM, P as the TMEM A
// operand, stream-K work split with owner merge) with 16 softmax warps instead of 8: for
// each Q tile, warps w and w+4 own the same 32 rows and keys [0,64) / [64,128) of every
// key tile (and O columns [0,64) / [64,128)).  The row max of a tile is exchanged through
// shared memory between the two warps (one named barrier per warp pair); everything else
// (exponentials, P halves, row sums, O rescale, epilogue columns) is per half.  This halves
// the softmax latency that sits on the per-Q-tile chain softmax -> PV -> QK -> softmax.
// 576 threads: warps 0-15 softmax (tile t = w / 8, key half = (w / 4) % 2, lane quadrant
// = w % 4), warp 16 TMA producer, warp 17 TMEM allocator + MMA issuer.
#include "kernels.h"

// SK2_EXPERIMENT (micro-benchmark builds only): 1 = softmax warps skip the math (MMA + TMA
// pipeline alone), 2 = no MMAs issued (softmax chain alone), 3 = no K / V loads, 4 = 1 + 3
#ifndef SK2_EXPERIMENT
#define SK2_EXPERIMENT 0
#endif
// SK2_TRACE=1 (micro-benchmark builds): compile in the clock64 / globaltimer stamps of
// AttnTC::trace and ::cta_trace; the library's kernel carries none of that code
#ifndef SK2_TRACE
#define SK2_TRACE 0
#endif
// exp2 pairs k with k % MOD >= GE go to the degree-3 polynomial on the FMA pipe (max rel.
// error 7.5e-5, far below the bf16 rounding of P), the rest to MUFU.  Round 2 A/B (C3 micro,
// one box, 3 alternations): 5 of 16 pairs (3/2) 80.7 us, 4/16 (4/3) 81.2, 6/16 (8/5) 83.3,
// none 83.0 (profiles/r02_attn_ab.md)
#ifndef SK2_POLY_MOD
#define SK2_POLY_MOD 3
#endif
#ifndef SK2_POLY_GE
#define SK2_POLY_GE 2
#endif

namespace vi {

template <int HD>
struct AttnSk2Smem {
  static constexpr int ST = 2;
  static constexpr int QB = 128 * HD * 2;
  static constexpr int KB = 128 * HD * 2;
  static constexpr int VB = HD * 128 * 2;
  static constexpr int Q_OFF = 0;
  static constexpr int K_OFF = 2 * QB;
  static constexpr int V_OFF = K_OFF + ST * KB;
  static constexpr int BAR_OFF = V_OFF + ST * VB;
  static constexpr int NBAR = 2 + 4 * ST + 2 + 4 + 2 + 2;
  static constexpr int STG_OFF = (BAR_OFF + NBAR * 8 + 16 + 127) / 128 * 128;   // [16 warps][32 rows][48 B] output staging
  static constexpr int XCH_OFF = STG_OFF + 16 * 32 * 48;        // [2 phases][2 tiles][2 halves][128] fp32
  static constexpr int TOTAL = XCH_OFF + 2 * 2 * 2 * 128 * 4 + 1024;
};

__device__ __forceinline__ void sk2_key_tile(const KeySegs& s, int g, int& row0, int& nvalid, int& nskip) {
  int i = 0;
  while (i + 1 < s.n && g >= s.tile0[i + 1]) ++i;
  const int off = (g - s.tile0[i]) * 128;
  row0 = s.row0[i] + off;
  const int rem = s.len[i] - off;
  nvalid = rem < 128 ? rem : 128;
  nskip = off == 0 ? s.lead[i] : 0;
}

// (bar.sync is .aligned: callers are converged -- every wait ends in a full-warp meeting)
__device__ __forceinline__ void sk2_named_bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// slice of the flattened work [0, W) owned by CTA c of G: an even split of the COST, where
// a unit costs sk_ucost (its start: the owner's segment switch and merge) + 16 per key tile,
// and the key tiles of the tail units (ordered last) sk_tail_w each
__device__ __forceinline__ long long sk2_begin(const AttnTC& a, long long W, int G, int c) {
  if (c >= G) return W;
  const long long NT = W / a.units, B = a.sk_ucost, tw = a.sk_tail_w;
  const long long uf = a.sk_wfull / NT;                 // full units
  const long long ucf = B + 16 * NT, uct = B + tw * NT;
  const long long cf = uf * ucf;
  const long long x = (cf + (a.units - uf) * uct) * c / G;
  if (x < cf) {
    const long long u = x / ucf, r = x - u * ucf;
    return u * NT + (r <= B ? 0 : (r - B) / 16);
  }
  const long long u = (x - cf) / uct, r = x - cf - u * uct;
  return (uf + u) * NT + (r <= B ? 0 : (r - B) / tw);
}

// unit u -> (head, first query row of its pair, window); tail units (if any) are the last H.
// Window attention (win_n > 0): units = (head, window, query pair of the window), one CTA per
// unit (the launch never splits them); query / key rows are offsets into the window-major
// buffers (win_qstride / win_kstride rows per window).
template <bool WIN>
__device__ __forceinline__ void sk2_unit(const AttnTC& a, int u, int& h, int& q0, int& win) {
  win = 0;
  if (WIN) {
    const int per_h = a.win_n * a.win_npw;
    h = u / per_h;
    const int r = u - h * per_h;
    const int wl = r / a.win_npw;                 // window within this launch's range
    win = a.win0 + wl;
    q0 = (r - wl * a.win_npw) * (a.sk_single ? 128 : 256);
    return;
  }
  const int full = a.npairs - a.sk_tail;     // full pairs per head
  const int uf = full * a.H;
  if (u < uf) {
    h = u / full;
    q0 = (u - h * full) * 256;
  } else {
    h = u - uf;
    q0 = full * 256;
  }
}

// window attention: output token row of local query q of window w, or -1 for padding rows
// and rows beyond the chunk (window-major rows: frame t, index i < win_real in the window)
__device__ __forceinline__ int sk2_win_out_row(const AttnTC& a, int w, int q) {
  if (q >= a.win_nq) return -1;
  const int t = q / a.win_pad, i = q - t * a.win_pad;
  if (i >= a.win_real) return -1;
  const int oy = (w / a.win_cols) * a.win_h + i / a.win_w, ox = (w % a.win_cols) * a.win_w + i % a.win_w;
  const int tok = oy * a.ow + ox;
  return a.win_split_rows ? t * a.win_split_rows + tok - a.win_part * a.win_split_rows : t * a.P + tok;
}

// WIN: window attention compiled in (a separate instantiation, so the global-attention kernel
// carries none of the window code: it measurably cost the C3 softmax loop registers).
// SINGLE (window units of one 128-query tile, AttnTC::sk_single): a third instantiation, so
// the pair kernels' softmax loop carries none of its branches (they cost C3 2.5 %).
template <int HD, bool WIN, bool SINGLE>
__global__ void __launch_bounds__(576, 1)
attn_sk2_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
               const __grid_constant__ CUtensorMap tvt, const AttnTC a) {
  using L = AttnSk2Smem<HD>;
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
  const long long w_begin = sk2_begin(a, W, G, cta), w_end = sk2_begin(a, W, G, cta + 1);
  // per-CTA stamps (micro-benchmarks): 0 entry, 1 setup done, 2 first QK issued, 3 last
  // o_final committed, 4 last epilogue start, 5 owner flags seen, 6 exit, 7 segments,
  // 8..11 MMA warp: each segment's o_final commit (first 4), 12 continuation piece
  // published, 13 owner's merge done
  long long* const ct = (SK2_TRACE && a.cta_trace) ? a.cta_trace + (size_t)cta * 24 : nullptr;
  if (ct && threadIdx.x == 0) ct[0] = (long long)globaltimer();
  if (!SINGLE && threadIdx.x == 0 && a.uparts && w_end > w_begin) {
    // for sk2_combine_kernel: this CTA is the first part of the units starting in its slice
    // (flag: the slice starts exactly there) and the last part of the units ending in it
    const int NT_ = a.segs.tile0[a.segs.n];
    for (long long uu = w_begin / NT_; uu * NT_ < w_end; ++uu) {
      const long long ub_ = uu * NT_;
      if (ub_ >= w_begin) a.uparts[uu] = cta | ((ub_ == w_begin ? 1 : 0) << 16);
      if (ub_ + NT_ - 1 >= w_begin && ub_ + NT_ - 1 < w_end) a.uparts[a.units + uu] = cta;
    }
  }

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
      mbar_init(&p_full[2 * t], 4);        // one elected arrive per softmax warp of the key half
      mbar_init(&p_full[2 * t + 1], 4);
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
  // launched with programmatic dependent launch (no CTA waits on another CTA of this grid):
  // the set-up above overlaps the previous kernel's tail
  griddep_wait();
  if (threadIdx.x == 0) time_begin(a.timing);
  if (ct && threadIdx.x == 0) ct[1] = (long long)globaltimer();
  // debug timeline (VI_SK_TRACE): CTA 0, first segment's first 32 key tiles, 32 clock64 stamps per tile
  long long* const trc = (SK2_TRACE && a.trace && cta == 0) ? a.trace : nullptr;

  if (warp == 16) {
    // TMA producer: the whole warp walks the schedule, one elected lane issues
    int jg = 0, sg = 0;
    for (long long w = w_begin; w < w_end; ++sg) {
      const int u = int(w / NT), ta = int(w - (long long)u * NT);
      const int tb = (int)((long long)NT < ta + (w_end - w) ? NT : ta + (w_end - w));
      int h, q0, win;
      sk2_unit<WIN>(a, u, h, q0, win);
      const int wq = win * a.win_qstride, wk = win * a.win_kstride;   // window row offsets
      if (sg > 0) mbar_wait_warp(q_empty, (sg - 1) & 1);
      if (elect_one()) {
        mbar_arrive_expect_tx(q_full, 2 * L::QB);
#pragma unroll
        for (int t = 0; t < 2; ++t)
#pragma unroll
          for (int at = 0; at < HD / 64; ++at)
            tma_load_2d(smem + L::Q_OFF + t * L::QB + at * 16384, &tq, q_full, h * HD + at * 64, a.q_row0 + wq + q0 + t * 128);
      }
      __syncwarp();
      for (int j = ta; j < tb; ++j, ++jg) {
        int row0, nv, nskip;
        sk2_key_tile(a.segs, j, row0, nv, nskip);
        const int st = jg % ST;
        const uint32_t par = ((jg / ST) & 1) ^ 1;
        if (jg >= ST) mbar_wait_warp(&k_empty[st], par);
        if (SK2_EXPERIMENT >= 3) {   // micro only: no K / V traffic (operands stale)
          if (elect_one()) mbar_arrive(&k_full[st]);
          __syncwarp();
          if (jg >= ST) mbar_wait_warp(&v_empty[st], par);
          if (elect_one()) mbar_arrive(&v_full[st]);
          __syncwarp();
          continue;
        }
        if (elect_one()) {
          uint8_t* sk = smem + L::K_OFF + st * L::KB;
          mbar_arrive_expect_tx(&k_full[st], L::KB);
#pragma unroll
          for (int at = 0; at < HD / 64; ++at)
            tma_load_2d(sk + at * 16384, &tk, &k_full[st], h * HD + at * 64, a.krow_base + wk + row0);
        }
        __syncwarp();
        if (jg >= ST) mbar_wait_warp(&v_empty[st], par);
        if (elect_one()) {
          uint8_t* sv = smem + L::V_OFF + st * L::VB;
          mbar_arrive_expect_tx(&v_full[st], L::VB);
#pragma unroll
          for (int at = 0; at < 2; ++at)
            tma_load_2d(sv + at * (HD * 128), &tvt, &v_full[st], wk + row0 + at * 64, a.vrow_base + h * HD);
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
      int h_, q0, win_;
      sk2_unit<WIN>(a, u, h_, q0, win_);
      const int nq = WIN ? a.win_nq : a.Nq;
      const bool t1_live = q0 + 128 < nq && SK2_EXPERIMENT != 2;   // tile 1 of a tail pair: commits only
      const bool t0_live = SK2_EXPERIMENT != 2;
      // single-tile units: tile 1 does not exist (no MMAs, no commits, no waits on its warps,
      // which leave at once); the K / V stages are released with tile 0's MMAs
      const int tl = SINGLE ? 0 : 1;
      mbar_wait_warp(q_full, sg & 1);
      auto issue_pv = [&](int t, int j) {          // O_t (+)= P_t(j) V(j), j local to the segment
        const int g = jg + j, st = g % ST;
        if (t == 0) mbar_wait_warp(&v_full[st], (g / ST) & 1);
        if (j == 0 && sg > 0) mbar_wait_warp(&o_free[t], (sg - 1) & 1);   // previous segment's O read out
        const uint64_t dv = dv0 + uint64_t((st * L::VB) >> 4);
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          mbar_wait_warp(&p_full[2 * t + hh], g & 1);
          tc_fence_after();
          if (elect_one()) {
            if (trc && g < 32) trc[g * 32 + 20 + hh * 6 + t] = clock64();
            if (t == 0 ? t0_live : t1_live) {
#pragma unroll
              for (int k4 = 0; k4 < 4; ++k4)
                umma_bf16_ts(tmem + 256 + t * 128, tmem + t * 128 + hh * 64 + k4 * 8,
                             dv + uint64_t((hh * (HD * 128) + k4 * 32) >> 4), idesc_o, (j | hh | k4) != 0);
            }
            if (hh == 1 && t == tl) umma_commit(&v_empty[st]);
          }
          __syncwarp();
        }
      };
      auto issue_qk = [&](int t, int j) {          // S_t = Q_t K(j)^T
        const int g = jg + j, st = g % ST;
        if (t == 0) {
          mbar_wait_warp(&k_full[st], (g / ST) & 1);
          tc_fence_after();
        }
        const uint64_t dk = dk0 + uint64_t((st * L::KB) >> 4), dq = dq0 + uint64_t((t * L::QB) >> 4);
        if (elect_one()) {
          if (t == 0 ? t0_live : t1_live) {
#pragma unroll
            for (int kk = 0; kk < HD / 16; ++kk) {
              const uint64_t off = uint64_t(((kk >> 2) * 16384 + (kk & 3) * 32) >> 4);
              umma_bf16_ss(tmem + t * 128, dq + off, dk + off, idesc_s, kk > 0);
            }
          }
          umma_commit(&s_full[t]);
          if (trc && g < 32) trc[g * 32 + 24 + t] = clock64();
          if (ct && g == 0 && t == 0) ct[2] = (long long)globaltimer();
          if (t == tl) umma_commit(&k_empty[st]);
        }
        __syncwarp();
      };
      if (SINGLE) {
        // one Q tile, S double-buffered in the two S regions (S(j) in buffer j & 1, P(j) over
        // it), O in tile 0's O: QK(j + 1) runs while the softmax works on S(j).  QK(j + 2)
        // reuses buffer j & 1 after PV(j) in issue order (the tensor pipe completes in order).
        // o_final[1] completes once per PV: the softmax's lazy O rescale at tile j waits for
        // PV(j - 1) there.  One segment per CTA (the launch checks grid == units).
        auto qk1 = [&](int j) {
          const int g = jg + j, st = g % ST, b = j & 1;
          mbar_wait_warp(&k_full[st], (g / ST) & 1);
          tc_fence_after();
          const uint64_t dk = dk0 + uint64_t((st * L::KB) >> 4);
          if (elect_one()) {
            if (t0_live) {
#pragma unroll
              for (int kk = 0; kk < HD / 16; ++kk) {
                const uint64_t off = uint64_t(((kk >> 2) * 16384 + (kk & 3) * 32) >> 4);
                umma_bf16_ss(tmem + b * 128, dq0 + off, dk + off, idesc_s, kk > 0);
              }
            }
            umma_commit(&s_full[b]);
            if (trc && g < 32) trc[g * 32 + 24 + b] = clock64();
            if (ct && g == 0) ct[2] = (long long)globaltimer();
            umma_commit(&k_empty[st]);
          }
          __syncwarp();
        };
        auto pv1 = [&](int j) {
          const int g = jg + j, st = g % ST, b = j & 1;
          mbar_wait_warp(&v_full[st], (g / ST) & 1);
          const uint64_t dv = dv0 + uint64_t((st * L::VB) >> 4);
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            mbar_wait_warp(&p_full[2 * b + hh], (j >> 1) & 1);
            tc_fence_after();
            if (elect_one()) {
              if (t0_live) {
#pragma unroll
                for (int k4 = 0; k4 < 4; ++k4)
                  umma_bf16_ts(tmem + 256, tmem + b * 128 + hh * 64 + k4 * 8,
                               dv + uint64_t((hh * (HD * 128) + k4 * 32) >> 4), idesc_o, (j | hh | k4) != 0);
              }
              if (hh == 1) {
                umma_commit(&v_empty[st]);
                umma_commit(&o_final[1]);
              }
            }
            __syncwarp();
          }
        };
        qk1(0);
        for (int j = 1; j < n; ++j) {
          qk1(j);
          pv1(j - 1);
        }
        if (elect_one()) umma_commit(q_empty);
        __syncwarp();
        pv1(n - 1);
        if (elect_one()) umma_commit(&o_final[0]);
        __syncwarp();
      } else {
        for (int j = 0; j < n; ++j)
          for (int t = 0; t <= tl; ++t) {
            if (j > 0) issue_pv(t, j - 1);
            issue_qk(t, j);
          }
        if (elect_one()) umma_commit(q_empty);       // all QK of the segment issued: Q smem free when done
        __syncwarp();
        for (int t = 0; t <= tl; ++t) {
          issue_pv(t, n - 1);
          if (elect_one()) umma_commit(&o_final[t]);
          __syncwarp();
        }
      }
      if (ct && lane == 0) {
        const long long now = (long long)globaltimer();
        ct[3] = now;
        if (sg < 4) ct[8 + sg] = now;
        ct[7] = sg + 1;
      }
      jg += n;
      w += n;
    }
  } else if (warp < 16 && !(SINGLE && warp >= 8)) {   // (single-tile units: tile 1's warps idle)
    const int t = warp >> 3;                        // Q tile
    const int hf = (warp >> 2) & 1;                 // key half / O column half
    const int qd = warp & 3;                        // TMEM lane quadrant
    const int row = qd * 32 + lane;                 // row within the Q tile
    const int pair_bar = 1 + t * 4 + qd;            // named barrier of warps (w, w ^ 4)
    const uint32_t lane_off = uint32_t(qd * 32) << 16;
    const uint32_t TO = tmem + 256 + t * 128 + lane_off;       // (S / P: TS per key tile below)
    constexpr int OH = HD / 2;                      // O columns of this half
    float* xch = reinterpret_cast<float*>(smem + L::XCH_OFF);
    const float2 cc = make_float2(a.scale_log2, a.scale_log2);
    int jg = 0, sg = 0, ph = 0;
    // partner exchange of one float per row (double-buffered by phase parity)
    auto exchange = [&](float v) {
      float* xb = xch + ((ph & 1) * 4 + t * 2) * 128;
      xb[hf * 128 + row] = v;
      sk2_named_bar_sync(pair_bar, 64);
      const float o = xb[(hf ^ 1) * 128 + row];
      ++ph;
      return o;
    };
    for (long long w = w_begin; w < w_end; ++sg) {
      const int u = int(w / NT), ta = int(w - (long long)u * NT);
      const int tb = (int)((long long)NT < ta + (w_end - w) ? NT : ta + (w_end - w));
      const int n = tb - ta;
      int h, q0, win;
      sk2_unit<WIN>(a, u, h, q0, win);
      const int nq = WIN ? a.win_nq : a.Nq;       // query rows of the unit's row space
      // all 32 rows of this warp past Nq (a tail pair): keep the barrier phases, skip the math
      // (their P / O lanes hold garbage that only reaches rows never stored)
      const bool dead = q0 + t * 128 + qd * 32 >= nq || SK2_EXPERIMENT == 1 || SK2_EXPERIMENT == 4;
      float m_use = -INFINITY, l = 0.f;
      for (int j = 0; j < n; ++j) {
        const int g = jg + j;
        // single-tile units: S(j) / P(j) in buffer j & 1 (see the MMA warp)
        const int sb = SINGLE ? (g & 1) : t;
        mbar_wait_warp(&s_full[sb], SINGLE ? (g >> 1) & 1 : g & 1);
        if (dead) {
          if (lane == 0) mbar_arrive(&p_full[2 * sb + hf]);
          continue;
        }
        const uint32_t TS = tmem + sb * 128 + lane_off;
        int row0, nv, nskip;
        sk2_key_tile(a.segs, ta + j, row0, nv, nskip);
        tc_fence_after();
        const bool tr = trc && lane == 0 && g < 32;
        if (tr && hf == 0 && qd == 0) trc[g * 32 + 0 + t] = clock64();
        float s[64];
        tmem_ld32(TS + hf * 64, reinterpret_cast<uint32_t*>(s));
        tmem_ld32(TS + hf * 64 + 32, reinterpret_cast<uint32_t*>(s + 32));
        tmem_wait_ld();
        const int lo = nskip - hf * 64, hi = nv - hf * 64;   // valid local keys [lo, hi)
        if (lo > 0 || hi < 64) {
#pragma unroll
          for (int i = 0; i < 64; ++i)
            if (i < lo || i >= hi) s[i] = -INFINITY;
        }
        if (WIN && a.win_pad > a.win_real) {         // window padding keys (row % pad >= real)
          uint32_t pm0 = 0u, pm1 = 0u;
          const int base = row0 + hf * 64;
          for (int k = a.win_real - base % a.win_pad; k < 64; k += a.win_pad)
            for (int e = k < 0 ? 0 : k; e < k + a.win_pad - a.win_real && e < 64; ++e) {
              if (e < 32) pm0 |= 1u << e;
              else pm1 |= 1u << (e - 32);
            }
#pragma unroll
          for (int i = 0; i < 64; ++i)
            if ((((i < 32 ? pm0 : pm1) >> (i & 31)) & 1u) != 0u) s[i] = -INFINITY;
        }
        float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int i = 0; i < 64; ++i) mx[i & 3] = fmaxf(mx[i & 3], s[i]);
        const float lm = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3]));
        // both halves see the same row max, hence the same lazy-rescale decision
        const float rmax = fmaxf(lm, exchange(lm)) * a.scale_log2;
        if (tr && hf == 0 && qd == 0) trc[g * 32 + 2 + t] = clock64();
        const bool grow = rmax > m_use + 8.f;
        float alpha = 1.f;
        if (grow) {
          alpha = ex2(m_use - rmax);
          m_use = rmax;
        }
        const float2 mm = make_float2(-m_use, -m_use);
        float2 sum[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) sum[i] = make_float2(0.f, 0.f);
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          uint32_t pk[16];
#pragma unroll
          for (int k = 0; k < 16; ++k) {
            const int i = c * 16 + k;
            const float2 x = ffma2(make_float2(s[2 * i], s[2 * i + 1]), cc, mm);
            float2 p;
            if (k % SK2_POLY_MOD >= SK2_POLY_GE) {   // these exp2 pairs on the FMA pipe (polynomial)
              p = exp2_poly2(x);
            } else {
              p.x = ex2(x.x);
              p.y = ex2(x.y);
            }
            __nv_bfloat162 b = __floats2bfloat162_rn(p.x, p.y);
            pk[k] = *reinterpret_cast<uint32_t*>(&b);
            sum[k & 3] = fadd2(sum[k & 3], p);
          }
          tmem_st16(TS + hf * 64 + c * 16, pk);   // P keys [hf*64, +64) -> packed cols [hf*64, +32)
        }
        // O rescale after P (S registers dead by now); PV(j-1) is complete (s_full implies it).
        // The PV MMAs of EITHER key half accumulate into all O columns, so both warps of the
        // pair (same row maxima, same decision) finish their column half before either one
        // hands its P half over.  Rare (lazy threshold 2^8).
        if (SINGLE && j > 0) mbar_wait_warp(&o_final[1], (g - 1) & 1);   // PV(j - 1) done (every tile: phase order)
        if (__any_sync(0xffffffffu, grow) && j > 0) {
#pragma unroll 1
          for (int c = 0; c < OH; c += 32) {
            uint32_t r[32];
            tmem_ld32(TO + hf * OH + c, r);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
            tmem_st32(TO + hf * OH + c, r);
          }
          tmem_wait_st();
          sk2_named_bar_sync(pair_bar, 64);
        }
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();                                  // every lane's P stores are complete ...
        if (lane == 0) mbar_arrive(&p_full[2 * sb + hf]);   // ... then one arrive per warp
        if (tr) trc[g * 32 + 4 + t * 8 + hf * 4 + qd] = clock64();
        const float2 s01 = fadd2(fadd2(sum[0], sum[1]), fadd2(sum[2], sum[3]));
        l = l * alpha + (s01.x + s01.y);
      }
      // ---- segment epilogue: each warp owns O columns [hf*64, +64) of its 32 rows
      mbar_wait_warp(&o_final[t], sg & 1);
      tc_fence_after();
      if (ct && warp == 0 && lane == 0) ct[4] = (long long)globaltimer();
      l += exchange(l);                             // row sum over both key halves
      const int r256 = t * 128 + row;               // row in the CTA's 256-row slot
      const float lse_own = m_use + __log2f(l);
      uint8_t* stg = smem + L::STG_OFF + warp * (32 * 48);
      const int rbase = q0 + t * 128 + qd * 32;
      const uint32_t TOh = TO + hf * OH;
      // output row of this lane's accumulator row (-1: none); write_out16 fetches the rows it
      // stores by shuffle (the window mapping costs a few integer divisions: once per segment)
      const int my_orow = WIN ? sk2_win_out_row(a, win, rbase + lane) : (rbase + lane < a.Nq ? rbase + lane : -1);
      // 16 O columns -> bf16 output rows via the per-warp stage (16 rows x 32 B per store)
      auto write_out16 = [&](int c, const float* f, float scale) {   // c: column within the half
        uint4* my = reinterpret_cast<uint4*>(stg + lane * 48);
#pragma unroll
        for (int k = 0; k < 2; ++k)
          my[k] = make_uint4(pack_bf16(f[8 * k] * scale, f[8 * k + 1] * scale),
                             pack_bf16(f[8 * k + 2] * scale, f[8 * k + 3] * scale),
                             pack_bf16(f[8 * k + 4] * scale, f[8 * k + 5] * scale),
                             pack_bf16(f[8 * k + 6] * scale, f[8 * k + 7] * scale));
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int rr = i * 16 + (lane >> 1), part = lane & 1;
          const uint4 v = *reinterpret_cast<const uint4*>(stg + rr * 48 + part * 16);
          const int orow = __shfl_sync(0xffffffffu, my_orow, rr);
          if (orow >= 0)
            *reinterpret_cast<uint4*>(a.o + (size_t)orow * a.o_ld + (size_t)h * a.o_hs + hf * OH + c + part * 8) = v;
        }
        __syncwarp();
      };
      if (ta > 0 || tb < NT) {
        // part of a split unit: its normalised partial (bf16) + lse -> the CTA's piece slot
        // (2c: its first segment, 2c + 1: its last); sk2_combine_kernel merges a unit's pieces
        // after the launch (every CTA finishes its own work: no CTA waits on another)
        const float inv = 1.f / l;
        const int slot = 2 * cta + (sg == 0 ? 0 : 1);
        uint4* dst = reinterpret_cast<uint4*>(a.spart) + (size_t)slot * (HD / 8) * 256 + r256;
#pragma unroll 1
        for (int c = 0; c < OH; c += 32) {
          float f[32];
          tmem_ld32(TOh + c, reinterpret_cast<uint32_t*>(f));
          tmem_wait_ld();
#pragma unroll
          for (int k = 0; k < 32; k += 8)
            dst[((hf * OH + c + k) / 8) * 256] =
                make_uint4(pack_bf16(f[k] * inv, f[k + 1] * inv), pack_bf16(f[k + 2] * inv, f[k + 3] * inv),
                           pack_bf16(f[k + 4] * inv, f[k + 5] * inv), pack_bf16(f[k + 6] * inv, f[k + 7] * inv));
        }
        tc_fence_before();
        mbar_arrive(&o_free[t]);
        if (hf == 0) a.slse[(size_t)slot * 256 + r256] = lse_own;
        if (ct && threadIdx.x == 0) ct[12] = (long long)globaltimer();
      } else {
        const float inv = 1.f / l;
#pragma unroll 1
        for (int c = 0; c < OH; c += 16) {
          float f[16];
          tmem_ld16(TOh + c, reinterpret_cast<uint32_t*>(f));
          tmem_wait_ld();
          write_out16(c, f, inv);
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
  if (ct && threadIdx.x == 0) ct[6] = (long long)globaltimer();
  if (warp == 17) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// Merge of the split units (units whose key tiles several CTAs shared): every part wrote its
// normalised partial (bf16) + lse to its CTA's piece slot; out = sum_k 2^(lse_k - M) O_k /
// sum_k 2^(lse_k - M), online-rescaled over the parts in CTA order (deterministic); units
// covered by one CTA were written by the attention.  The parts of a unit come from the first
// and last CTAs the attention's CTAs recorded (a.uparts).  Block = (unit, 32 rows, 8 column groups),
// thread = (row, 8 columns): lane = row, so a warp reads 512 contiguous bytes of a piece
// ([HD/8][256 rows] x 16 B).
template <int HD, bool WIN>
__global__ void __launch_bounds__(256) sk2_combine_kernel(const AttnTC a) {
  griddep_wait();
  if (threadIdx.x == 0) time_begin(a.combine_timing);
  griddep_launch();
  constexpr int C8 = HD / 8;                    // 8-column groups per row
  const int u = blockIdx.x;
  const int p0 = __ldcg(a.uparts + u), c1 = __ldcg(a.uparts + a.units + u);
  const int c0 = p0 & 0xffff, b0 = p0 >> 16;     // first / last CTA of the unit
  const int np = c1 - c0 + 1;                     // parts: c0 (its first segment iff b0), c0+1 .. c1
  if (np > 1) {
    const int r = blockIdx.y * 32 + (threadIdx.x & 31), c8 = blockIdx.z * 8 + (threadIdx.x >> 5);
    int h, q0, win;
    sk2_unit<WIN>(a, u, h, q0, win);
    const int orow = WIN ? sk2_win_out_row(a, win, q0 + r) : (q0 + r < a.Nq ? q0 + r : -1);
    if (orow >= 0) {
      // online rescale over the parts in CTA order; each group of up to 4 parts has all its
      // loads issued before the sums
      const uint4* sp = reinterpret_cast<const uint4*>(a.spart);
      float m = -INFINITY, wsum = 0.f, acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      for (int k0 = 0; k0 < np; k0 += 4) {
        float lk[4];
        uint4 v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          lk[k] = -INFINITY;
          v[k] = make_uint4(0u, 0u, 0u, 0u);
          if (k0 + k < np) {
            const int slot = k0 + k == 0 ? 2 * c0 + (b0 ? 0 : 1) : 2 * (c0 + k0 + k);
            lk[k] = __ldcg(a.slse + (size_t)slot * 256 + r);
            v[k] = __ldcg(sp + ((size_t)slot * C8 + c8) * 256 + r);
          }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (k0 + k >= np) break;
          const float mn = fmaxf(m, lk[k]);
          const float sc = ex2(m - mn), w = ex2(lk[k] - mn);   // (sc = 0 for the first part)
          wsum = wsum * sc + w;
          const uint32_t wv[4] = {v[k].x, v[k].y, v[k].z, v[k].w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 p2 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wv[e]));
            acc[2 * e] = acc[2 * e] * sc + w * p2.x;
            acc[2 * e + 1] = acc[2 * e + 1] * sc + w * p2.y;
          }
          m = mn;
        }
      }
      const float inv = 1.f / wsum;
      *reinterpret_cast<uint4*>(a.o + (size_t)orow * a.o_ld + (size_t)h * a.o_hs + c8 * 8) =
          make_uint4(pack_bf16(acc[0] * inv, acc[1] * inv), pack_bf16(acc[2] * inv, acc[3] * inv),
                     pack_bf16(acc[4] * inv, acc[5] * inv), pack_bf16(acc[6] * inv, acc[7] * inv));
    }
  }
  if (a.combine_timing) {
    __syncthreads();
    if (threadIdx.x == 0) time_end(a.combine_timing, gridDim.x * gridDim.y * gridDim.z);
  }
}

template <int HD, bool WIN, bool SINGLE>
static cudaError_t launch_sk2_hd(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tvt,
                                const AttnTC& a, int grid, cudaStream_t st) {
  using L = AttnSk2Smem<HD>;
  auto kfn = attn_sk2_kernel<HD, WIN, SINGLE>;
  cudaError_t e = ensure_kernel_setup(reinterpret_cast<const void*>(kfn), L::TOTAL);
  if (e != cudaSuccess) return e;
  // single-tile units run one CTA per unit (their tile-1 warps leave at once, so no unit may be
  // split): no CTA waits on another -> plain PDL launch
  if (SINGLE) {
    if (grid != a.units) return cudaErrorInvalidValue;
    return pdl_launch(kfn, dim3(grid), dim3(576), L::TOTAL, st, tq, tk, tvt, a);
  }
  // stream-K: every CTA finishes its own slice and publishes split-unit pieces for the combine
  // kernel -- no CTA waits on another, so no cooperative launch is needed, and a programmatic
  // dependent launch lets each CTA's set-up (barriers, TMEM, descriptor prefetch) overlap the
  // QKV GEMM's tail (A/B against the former cooperative launch: C3 step 1.324 vs 1.332 ms;
  // the attention's own self-timed launch 78.2 vs 77.7 us)
  e = pdl_launch(kfn, dim3(grid), dim3(576), L::TOTAL, st, tq, tk, tvt, a);
  if (e != cudaSuccess) return e;
  // the split units' pieces -> output rows
  if (!a.uparts || grid > 65535) return cudaErrorInvalidValue;   // (CTA index in 16 bits)
  return pdl_launch(sk2_combine_kernel<HD, WIN>, dim3(a.units, 8, HD / 64), dim3(256), 0, st, a);
}

cudaError_t launch_attn_sk2(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tvt, const AttnTC& a,
                           int grid, cudaStream_t st) {
  if (a.win_n && a.sk_single) {
    if (a.hd == 128) return launch_sk2_hd<128, true, true>(tq, tk, tvt, a, grid, st);
    if (a.hd == 64) return launch_sk2_hd<64, true, true>(tq, tk, tvt, a, grid, st);
    return cudaErrorInvalidValue;
  }
  if (a.sk_single) return cudaErrorInvalidValue;   // (single-tile units exist for windows only)
  if (a.win_n) {
    if (a.hd == 128) return launch_sk2_hd<128, true, false>(tq, tk, tvt, a, grid, st);
    if (a.hd == 64) return launch_sk2_hd<64, true, false>(tq, tk, tvt, a, grid, st);
    return cudaErrorInvalidValue;
  }
  if (a.hd == 128) return launch_sk2_hd<128, false, false>(tq, tk, tvt, a, grid, st);
  if (a.hd == 64) return launch_sk2_hd<64, false, false>(tq, tk, tvt, a, grid, st);
  return cudaErrorInvalidValue;
}

}  // namespace vi
