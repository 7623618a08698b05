// Host-side launchers of the sm_100a kernels (internal to libvi.so).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "epilogue.cuh"

namespace vi {

// Programmatic dependent launch for the stream-ordered kernels of a step (see griddep_wait
// in common.cuh); g_pdl = 0 (VI_PDL=0) launches them with plain stream serialization.
extern int g_pdl;
template <typename... KArgs, typename... Args>
cudaError_t pdl_launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = g_pdl;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// Per-device, thread-safe one-time setup of a kernel (setup.cu): the dynamic shared memory
// opt-in on the CURRENT device, and (cluster > 1) the number of clusters of `cluster` CTAs
// of `block` threads that fit at once (else the SM count); returned in *max_clusters.
cudaError_t ensure_kernel_setup(const void* fn, int smem_bytes, int cluster = 1, int block = 0,
                                int* max_clusters = nullptr);

struct Geom {
  int H, W, C, kh, kw, sh, sw, ph, pw, oh, ow;
};

// ---- patch gather kernels (HBM-bound) -------------------
// soft split: in [n][H][W][C] -> out [n][P][kh*kw*C]; dtype 0 = bf16, 1 = fp32.
// timing (optional): KernelTiming the launch folds its first-CTA-start / last-CTA-end into (profile mode 3)
cudaError_t launch_unfold(const void* in, void* out, int n, const Geom& g, int dtype, cudaStream_t st,
                          unsigned long long* timing = nullptr);
// fold with cover-count division: in [n][P][kh*kw*C] (in_dtype) -> out [n][H][W][C] (out_dtype),
// optionally GELU of the folded value (Fusion-FFN).  Requires ceil(k/s) <= 3 per dimension.
cudaError_t launch_fold(const void* in, int in_dtype, void* out, int out_dtype, int n, const Geom& g, bool gelu,
                        cudaStream_t st, unsigned long long* timing = nullptr);

// ---- row kernels -------------------------------------------------------------------
// LayerNorm over D (eps 1e-5), fp32 in, out dtype 0 bf16 / 1 fp32.
cudaError_t launch_layernorm(const float* x, const float* g, const float* b, void* out, int out_dtype, int rows,
                             int D, cudaStream_t st);
// x fp32 [rows][D] -> [rows][2D] bf16 (hi | lo) for the extended-precision back projection
// split-K reduction: out = x_in (NULL: none) + bias + sum of the partials (+ pos[m % P] when
// pos != NULL), and LayerNorm(out) into h when g != NULL; ws partial s of row m at
// ws + s * split_ld + m * D (fp32)
cudaError_t launch_splitk_resid(const float* ws, int ksplit, size_t split_ld, const float* bias, const float* x_in,
                                float* x_out, const float* pos, int P, const float* g, const float* b, void* h,
                                int h_dtype, int rows, int D, cudaStream_t st, unsigned long long* timing = nullptr);
cudaError_t launch_split_bf16(const float* x, void* out, int rows, int D, cudaStream_t st);
// v [P][D] (row pitch src_ld elements) -> vt_slab[d][col0 + p] (row pitch ld)
cudaError_t launch_transpose_to_slab(const void* v, void* vt_slab, int P, int D, size_t ld, size_t col0, int dtype,
                                     cudaStream_t st, int src_ld = 0);

// ---- GEMMs ---------------------------------------------------------------------------
// tensor cores (bf16): A [M][K] and W [N][K] described by 2-D TMA maps with 64 x 128 /
// 64 x BN boxes and 128-byte swizzle.
// brow0: row offset of this layer's weight block inside the stacked W map.
// pair: 0 = single-CTA 128 x BN tiles (W box 64 x BN); 1 = CTA-pair 256 x BN tiles with the
// 2-SM MMA (W box 64 x BN/2).
// tmo (optional): output tensor map (bf16 or fp32 [M][N], box 128 bytes x 32 rows, 128-byte
// swizzle) -> the TMA-store epilogue for EPI_STORE / EPI_GELU / EPI_RESID (tmx: x_in map of
// the same shape for EPI_RESID; x_out = the tmo tensor).  EPI_QKV: tmo = Q (box 64 x 32,
// swizzled), tmx = the K slabs (box 64 x 8, swizzled), tmv = the Vt slabs (box 8 x 64, no
// swizzle); global attention with P % 8 == 0 only.
cudaError_t launch_gemm_tc(const CUtensorMap& a, const CUtensorMap& w, int brow0, int M, int N, int K, int bn,
                           const Epi& e, cudaStream_t st, int pair = 0, const CUtensorMap* tmo = nullptr,
                           const CUtensorMap* tmx = nullptr, const CUtensorMap* tmv = nullptr);
// SIMT (fp32 path): A [M][K], W [N][K] row-major fp32, FFMA accumulate.
cudaError_t launch_gemm_simt_f32(const float* A, const float* W, int M, int N, int K, const Epi& e, cudaStream_t st);

// ---- attention -----------------------------------------------------------------------
struct KeySegs {            // contiguous runs of valid ring slots, as slab row ranges
  int n;
  int row0[32];             // first row, aligned DOWN to a multiple of 8 (TMA: 16-byte start)
  int lead[32];             // rows row0 .. row0+lead-1 precede the segment: masked
  int len[32];              // lead + valid rows
  int tile0[33];            // prefix count of 128-key tiles per segment
};

// Device-side self-timing of a sequence of stream-ordered launches (graph-safe): CTA (0,0,0)
// stores its start globaltimer in tmin, every CTA counts itself done, and the last CTA to
// finish adds (its end - tmin) to total_ns, counts the launch and resets the count (tmax unused).
struct KernelTiming {
  unsigned long long tmin, tmax, done, total_ns, launches, pad[3];
};

struct AttnArgs {
  int Nq, D, H, hd, P, S, vt_ld;
  uint64_t valid;           // slot validity mask
  float scale_log2;         // log2(e) / sqrt(hd)
  const void* q;            // [Nq][D]
  const void* kslab;        // [S*P][D]        (this layer)
  const void* vtslab;       // [D][vt_ld]      (this layer)
  void* o;                  // [Nq][D]
};
cudaError_t launch_attn_simt_f32(const AttnArgs& a, cudaStream_t st);

struct AttnTC {
  int Nq, hd, D, krow_base, vrow_base;   // row offsets of this layer inside the 2-D slab maps
  int nsplit, tiles_per_split;
  float scale_log2;
  KeySegs segs;
  bf16* o;                  // [Nq][D] final (nsplit == 1)
  bf16* opart;              // [nsplit][Nq][D] normalised partial outputs, bf16 (nsplit > 1)
  float* lse;               // [nsplit][H][Nq] log2-sum-exp of the partials
  // stream-K (attn_sk_kernel): units = (query-tile pair, head), work = units x key tiles,
  // split evenly over the persistent grid; partial results of split units go through
  // spart/slse/sflag (one slot per CTA) and are merged by the unit's first CTA.
  int npairs, units;
  // attn_sk2 only: when the last query pair of every head has an empty second tile
  // (Nq mod 256 in (0, 128]), those H "tail" units are ordered last (sk_tail = 1) and the
  // work split weights their key tiles sk_tail_w / 16 of a full pair's (tile 1 and the
  // softmax quadrants past Nq are skipped); sk_wfull = work items of the full units.
  int sk_tail, sk_tail_w;
  int sk_ucost;              // attn_sk2 split cost of a unit's start (16 = one key tile of a pair)
  int sk_single;             // attn_sk2 window units of ONE 128-query tile (tile 1 idle): with one
                             // CTA per unit no unit is split, so no piece is merged
  long long sk_wfull;
  float* spart;             // [grid][256][hd]
  float* slse;              // [grid][256]
  int* sflag;               // [grid], 0 between launches
  int* uparts;              // attn_sk2 -> combine: [units] first CTA of each unit (| 1 << 16: its slice starts
                            // at the unit) and [units] last CTA, written by the attention
  long long* trace;         // debug timeline of CTA (0,0,0) (NULL = off)
  long long* cta_trace;     // attn_sk2: [grid][16] globaltimer stamps per CTA (micro-benchmarks; NULL = off)
  unsigned long long* timing;   // KernelTiming (device) or NULL: the kernels time themselves
  unsigned long long* combine_timing;   // the same for the split-merge kernels (sk2_combine,
                                        // attn_combine); NULL = untimed (vi_profile mode 4)
  int H;
  // stream-K kernels (attn_sk, attn_sk2): query rows start at row q_row0 of the Q map;
  // output row i of local head h goes to o + i * o_ld + h * o_hs (unsharded: o_ld = D,
  // o_hs = hd; head-sharded: the rank's chunk of the head-major gathered buffer, tp.h)
  int q_row0, o_ld, o_hs;
  // window attention (win_n > 0; attn_tc2 + combine only): win_npw CTAs (256 query rows
  // each) per window; window w's queries are rows w * win_qstride + [0, win_nq) of the Q map
  // (frame t's token i of the window at t * win_pad + i), its keys rows w * win_kstride + the
  // key segments (slot s at s * win_pad); rows with index % win_pad >= win_real are padding
  // (keys masked, queries not written); output row of (t, i) = t * P + token(w, i)
  int win_n, win_npw, win_qstride, win_kstride, win_pad, win_real, win_h, win_w, win_cols, ow, P, win_nq;
  // windows [win0, win0 + win_n) of the win_cols-wide window grid (head sharding with more
  // ranks than heads splits a head's windows between q ranks by window rows); with
  // win_split_rows > 0 (= P / q) an output row goes to the rank's part-local row
  // t * win_split_rows + (token - win_part * win_split_rows) instead of the token row
  int win0, win_split_rows, win_part;
};
// Window-split head sharding: the gathered head outputs og [H][q][part_rows][d] (part p of
// head h = that head's tokens [p*P/q, (p+1)*P/q) of every frame, frame-major) -> O [M][D]
// token-major for the output projection
cudaError_t launch_window_part_gather(const void* og, void* o, int M, int P, int H, int hd, int q, int part_rows,
                                      cudaStream_t st);
// two 128-query tiles per CTA, P kept in TMEM, fixed KV split (small chunks; attn.cu)
cudaError_t launch_attn_tc2(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tvt, const AttnTC& a,
                            cudaStream_t st);
cudaError_t launch_attn_combine(const AttnTC& a, cudaStream_t st);
// persistent stream-K, column-split softmax, 16 softmax warps (attn_sk2.cu; the default)
cudaError_t launch_attn_sk2(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tvt, const AttnTC& a,
                            int grid, cudaStream_t st);

}  // namespace vi
