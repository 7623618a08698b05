#include <climits>
// libvi.so engine: the vi_* C-ABI (include/vi.h) over the sm_100a kernels.
//
// Per context (one live stream on one GPU) the engine owns, in HBM:
//   weights  (bf16 matrices / fp32 biases + LN params; nn.Linear [out][in] layout,
//             the per-block matrices of all L blocks stacked so one TMA map covers them)
//   memory   K slab [L][S*P][D] and V slab stored TRANSPOSED [L][D][S*P] (ctx dtype);
//            slot s of block l holds rows s*P .. s*P+P-1 (reading Q11, slot = id mod S)
//   workspaces for one chunk of up to T_max frames (tokens, h, Q, O, u, g, F3N fold map,
//            KV-split partials) plus host-buffer staging for vi_run_step.
// Every step of the path runs in the kernels of kernels/*.cu; the host only validates,
// keeps the integer ring bookkeeping (ring.cpp) and enqueues launches.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include <unistd.h>

#include "kernels/kernels.h"
#include "ring.h"
#include "tp.h"
#include "vi.h"

using namespace vi;

namespace {

typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                      const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                      CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

PFN_encodeTiled_t encode_fn() {
  static PFN_encodeTiled_t fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled_t>(p);
  }
  return fn;
}

// 2-D bf16 tensor [outer][inner] (row pitch = inner elements), box {box_inner, box_outer},
// 128-byte swizzle, zero fill out of bounds.
bool make_tmap(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, uint32_t box_inner,
               uint32_t box_outer) {
  PFN_encodeTiled_t fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {inner * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Output tensor [rows][cols] (fp32 or bf16) for the GEMMs' TMA-store epilogue: box = one
// 128-byte row segment x 32 rows, 128-byte swizzle (gemm_tc.cu's staging layout).
bool make_tmap_out(CUtensorMap* m, const void* base, bool f32, uint64_t cols, uint64_t rows) {
  PFN_encodeTiled_t fn = encode_fn();
  if (!fn) return false;
  const uint64_t es = f32 ? 4 : 2;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * es};
  cuuint32_t box[2] = {uint32_t(128 / es), 32};
  cuuint32_t e[2] = {1, 1};
  return fn(m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
            strides, box, e, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// General 2-D bf16 map [rows][cols] with an arbitrary box, 128-byte swizzle or none
bool make_tmap_box(CUtensorMap* m, const void* base, uint64_t cols, uint64_t rows, uint32_t box_cols, uint32_t box_rows,
                   bool swizzle128) {
  PFN_encodeTiled_t fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t e[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, e,
            CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

uint16_t f2bf(float f) {  // round to nearest even
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return 0x7fc0;
  u += 0x7fffu + ((u >> 16) & 1u);
  return uint16_t(u >> 16);
}

bool is_host_ptr(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return at.type == cudaMemoryTypeHost || at.type == cudaMemoryTypeUnregistered;
}

constexpr int kMaxSplit = 16;

}  // namespace

struct vi_ctx {
  vi_config cfg{};
  Geom g{}, gf{};          // split geometry (C = feat_c) and F3N geometry (C = F / (kh*kw))
  int L = 0, H = 0, D = 0, hd = 0, P = 0, M = 0, Tmax = 0, S = 0, F = 0, Pd = 0, es = 2;
  int ST = 0;              // all memory slots: S span slots + R reference slots (ring.h)
  // window attention (vi_config.win_h / win_w): win_n windows of win_real tokens (win_pad =
  // win_real rows per frame); the memory and Q are window-major (epilogue.cuh qkv_rows), a
  // window's key region win_kstride = ST*win_pad rounded up to 8 rows
  int win_n = 0, win_real = 0, win_pad = 0, win_cols = 0, win_kstride = 0;
  int KR = 0;              // key rows per block in the slabs: ST*P, or win_n*win_kstride
  int QR = 0;              // rows of the Q buffer: T_max*P, or win_n*T_max*win_pad
  int vt_ld = 0;           // row pitch of the transposed V slab: S*P rounded up to 64 (TMA: 16-B pitch)
  bool bf16 = true;
  cudaStream_t stream = nullptr, copy_stream = nullptr;
  bool own_stream = false;
  std::string err = "ok";
  bool poisoned = false;
  int64_t launches = 0;
  // head sharding (tp.h): Hl local heads, Q/K/V width Dl = Hl * hd; the attention writes
  // the rank's chunk of the gathered head-major buffer og [H][head_rows][hd]
  bool sharded = false;
  bool win_split = false;         // windows + more ranks than heads: the head's windows split by window rows
  TpLayout tp;
  int Hl = 0, Dl = 0;
  void* comm = nullptr;           // ncclComm_t (NULL: unsharded, or exchange driven by the caller)
  void* og = nullptr;
  int attn_layer = -1;            // layer whose _attn half ran last (its _ffn half pending)
  // inside step_body (vi_run_step's own sequence of launches) a split-K reduction that
  // produces a block input also writes that block's LN1 into h (fuse_ln1); h_ready = the
  // layer whose LN1 is already in h (-1: none).  Never across public per-layer calls.
  bool fuse_ln1 = false;
  int h_ready = -1;
  cudaEvent_t ev_attn = nullptr, ev_gather = nullptr;   // vi_tp_local_allgather ordering
  Ring ring{0, 1};
  std::mutex mu;
  bool have_weights = false;
  int next_layer = -1;     // expected layer of the next vi_memory_step (-1: no push yet)

  // weights
  void *w_embed = nullptr, *w_qkv = nullptr, *w_o = nullptr, *w_1 = nullptr, *w_2 = nullptr, *w_back = nullptr;
  float *b_embed = nullptr, *pos = nullptr, *ln1_g = nullptr, *ln1_b = nullptr, *b_qkv = nullptr, *b_o = nullptr;
  float *ln2_g = nullptr, *ln2_b = nullptr, *b_1 = nullptr, *b_2 = nullptr, *b_back = nullptr;
  // memory
  void *kslab = nullptr, *vtslab = nullptr;
  // workspaces
  void *tokens = nullptr, *yp32 = nullptr, *w_back2 = nullptr, *h = nullptr, *q = nullptr, *o = nullptr, *u = nullptr, *gbuf = nullptr, *xb = nullptr;
  float *x_ws = nullptr, *fold_ws = nullptr, *lse = nullptr;
  vi::bf16* opart = nullptr;
  void *feat_in = nullptr, *feat_out = nullptr;
  // vi_run_step_async: copy streams (frames in / results out: one stream for both would order
  // step k+1's input copy behind step k's output copy, i.e. behind step k) and two staging slots
  cudaStream_t io_stream = nullptr, io_out = nullptr;
  void *async_in[2] = {nullptr, nullptr}, *async_out[2] = {nullptr, nullptr};
  cudaEvent_t ev_h2d[2] = {nullptr, nullptr}, ev_done[2] = {nullptr, nullptr}, ev_d2h[2] = {nullptr, nullptr};
  bool async_used[2] = {false, false};
  int async_slot = 0;
  std::vector<void*> allocs;
  size_t device_bytes = 0;   // everything dalloc'd (weights, memory slabs, workspaces)
  // queued refine commits: device copies of the K/V payloads, applied at the next push.  A
  // consumed buffer returns to free_kv with `released` recorded on the ctx stream after the
  // copies that read it, so a commit from another thread never touches the ctx stream (which
  // may be capturing a step graph) and still never overwrites a payload being applied.
  struct KvBuf {
    void* k = nullptr;
    void* v = nullptr;
    cudaEvent_t released = nullptr;
  };
  std::map<int64_t, KvBuf> pending_kv;
  std::vector<KvBuf> free_kv;

  // tensor maps (bf16 path)
  CUtensorMap tm_tokens, tm_wembed, tm_h, tm_wqkv, tm_o, tm_wo, tm_w1, tm_g, tm_w2, tm_xb, tm_wback;
  CUtensorMap tm_w1_128;   // W1 with 128-row boxes: FFN1 on 128-column tiles for small M
  CUtensorMap tm_w2_pair;    // W2 with a 64-row box: the CTA-pair FFN2 (256 x 128 tiles)
  CUtensorMap tm_q, tm_k, tm_vt, tm_og;
  CUtensorMap tm_u_out, tm_g_out, tm_yp_out;   // GEMM outputs through the TMA-store epilogue
  CUtensorMap tm_q_out, tm_k_out, tm_vt_out;   // QKV epilogue: Q rows, K slab rows (8-row boxes), Vt columns
  bool qkv_te = false;
  // N-tile per GEMM (persistent kernel: ~1-3 tiles per SM at M = 3600; N=64 MMAs run at 2/3 rate)
  int bn_embed = 128, bn_qkv = 128, bn_o = 128, bn_1 = 256, bn_2 = 128, bn_back = 256;

  // profiling (vi_profile)
  int prof_mode = 0;
  unsigned long long* attn_timing = nullptr;   // KernelTiming (device), used in profile mode 1
  int num_sms = 148;
  float* skws = nullptr;   // split-K GEMM partials (splitk_plan)
  size_t skws_floats = 0;
  float *sk_part = nullptr, *sk_lse = nullptr;  // stream-K partial slots [num_sms][256][hd], [num_sms][256]
  int* sk_flag = nullptr;                       // attn_sk2 unit parts [2][sk_units_cap]
  int sk_units_cap = 0;
  // CUDA graphs of whole steps (vi_run_step), keyed by everything baked into the launches
  struct GraphEntry {
    std::vector<uint64_t> key;
    cudaGraphExec_t exec;
    int64_t launches;
    int64_t last_use;
  };
  std::vector<GraphEntry> graphs;
  int64_t graph_clock = 0, weights_gen = 0;
  bool use_graphs = true;
  struct Rec { int cat; cudaEvent_t a, b; };
  std::vector<Rec> prof_recs;
  std::vector<cudaEvent_t> ev_pool;
  cudaEvent_t prof_ev() {
    if (ev_pool.empty()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      return e;
    }
    cudaEvent_t e = ev_pool.back();
    ev_pool.pop_back();
    return e;
  }

  ~vi_ctx();
  vi_status fail(vi_status st, const std::string& m) {
    err = m;
    return st;
  }
  vi_status cuda_fail(cudaError_t e, const char* where) {
    poisoned = true;
    err = std::string("CUDA error in ") + where + ": " + cudaGetErrorString(e);
    return VI_E_CUDA;
  }
  void* dalloc(size_t bytes, bool zero = true) {
    void* p = nullptr;
    if (cudaMalloc(&p, bytes ? bytes : 16) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    if (zero) cudaMemset(p, 0, bytes ? bytes : 16);
    allocs.push_back(p);
    device_bytes += bytes;
    return p;
  }
};

vi_ctx::~vi_ctx() {
  if (stream) cudaStreamSynchronize(stream);
  if (io_stream) cudaStreamSynchronize(io_stream);
  if (io_out) cudaStreamSynchronize(io_out);
  for (auto& g : graphs) cudaGraphExecDestroy(g.exec);
  for (auto& r : prof_recs) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  for (auto e : ev_pool) cudaEventDestroy(e);
  for (auto& kv : pending_kv) free_kv.push_back(kv.second);
  for (auto& kv : free_kv) {
    cudaFree(kv.k);
    cudaFree(kv.v);
    if (kv.released) cudaEventDestroy(kv.released);
  }
  for (void* p : allocs) cudaFree(p);
  if (comm) nccl().comm_destroy(comm);
  if (ev_attn) cudaEventDestroy(ev_attn);
  if (ev_gather) cudaEventDestroy(ev_gather);
  if (copy_stream) cudaStreamDestroy(copy_stream);
  if (io_stream) cudaStreamDestroy(io_stream);
  if (io_out) cudaStreamDestroy(io_out);
  for (int k = 0; k < 2; ++k)
    for (cudaEvent_t e : {ev_h2d[k], ev_done[k], ev_d2h[k]})
      if (e) cudaEventDestroy(e);
  if (own_stream && stream) cudaStreamDestroy(stream);
}

// VI_DEBUG_SYNC=1: wait for every launch (poll, 20 s limit) and name a kernel that hangs.
static const bool g_debug_sync = [] {
  const char* e = getenv("VI_DEBUG_SYNC");
  return e && e[0] == '1';
}();
// VI_SK_TAIL_W: cost of a tail pair's key tile in 16ths of a full pair's (sk2 work split);
// read when a step is recorded, so a sweep can change it between contexts
static int sk_tail_weight() {
  const char* e = getenv("VI_SK_TAIL_W");
  const int w = e ? atoi(e) : 16;
  return w < 1 ? 1 : (w > 64 ? 64 : w);
}
// VI_SK_UNIT_COST: split cost of a unit's start in 16ths of a pair key tile (the CTA that
// begins a unit switches segments and merges the unit's pieces at the end)
static int sk_unit_cost() {
  const char* e = getenv("VI_SK_UNIT_COST");
  // measured (C3 micro, same box): 0 -> 85.5 us, 16 -> 83.7, 32 -> 83.9, 48 -> 82.2,
  // 56 -> 81.7, 58-60 -> 81.5, 62 -> 83.0, 64 -> 83.0 (partition-dependent steps)
  const int b = e ? atoi(e) : 56;
  return b < 0 ? 0 : (b > 4096 ? 4096 : b);
}
// VI_SPLITK=0: no split-K for the small-M residual GEMMs (A/B measurements; read per launch
// so a test can compare both paths in one process)
static bool splitk_enabled() {
  const char* e = getenv("VI_SPLITK");
  return !(e && e[0] == '0');
}
static void debug_wait(vi_ctx* c, const char* where) {
  for (int i = 0; i < 20000; ++i) {
    cudaError_t e = cudaStreamQuery(c->stream);
    if (e == cudaSuccess) return;
    if (e != cudaErrorNotReady) {
      fprintf(stderr, "[vi debug] kernel '%s' failed: %s\n", where, cudaGetErrorString(e));
      fflush(stderr);
      _exit(3);
    }
    usleep(1000);
  }
  fprintf(stderr, "[vi debug] kernel '%s' did not finish within 20 s\n", where);
  fflush(stderr);
  _exit(4);
}

#define CK(call, where)                                 \
  do {                                                  \
    cudaError_t e_ = (call);                            \
    if (e_ != cudaSuccess) return c->cuda_fail(e_, where); \
  } while (0)
#define LAUNCH(call, where)        \
  do {                             \
    ++c->launches;                 \
    CK((call), where);             \
    if (g_debug_sync) debug_wait(c, where); \
  } while (0)
// VI_ABLATE_BUILD (a separate timing-experiment build, never the product library: its
// results are garbage): VI_ABLATE=<mask> skips the launches of the profile categories whose
// bit is set (1 attention, 2 GEMMs, 4 patch, 8 row kernels), to measure each class's
// marginal cost inside the step graph
#ifdef VI_ABLATE_BUILD
static const int g_ablate = [] {
  const char* e = getenv("VI_ABLATE");
  return e ? atoi(e) : 0;
}();
#define PLAUNCH(cat, call, where)                  \
  do {                                             \
    if (!((g_ablate >> (cat)) & 1)) {              \
      Prof p_(c, cat);                             \
      LAUNCH(call, where);                         \
    }                                              \
  } while (0)
#else
#define PLAUNCH(cat, call, where)                  \
  do {                                             \
    Prof p_(c, cat);                               \
    LAUNCH(call, where);                           \
  } while (0)
#endif
#define CK_C(ctx, call, where)                              \
  do {                                                      \
    cudaError_t e_ = (call);                                \
    if (e_ != cudaSuccess) return (ctx)->cuda_fail(e_, where); \
  } while (0)
#define LIVE(c)                                                      \
  do {                                                               \
    if (!(c)) return VI_E_ARG;                                       \
    if ((c)->poisoned) return VI_E_CUDA;                             \
  } while (0)

// Every entry point runs on its context's device (contexts of one process may live on
// different GPUs and be driven from different threads, e.g. the Refined model's two).
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess || prev == dev) {
      prev = -1;
      return;
    }
    cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// Scoped event pair around the launches of one category (vi_profile).
struct Prof {
  vi_ctx* c;
  int cat;
  cudaEvent_t b = nullptr;
  Prof(vi_ctx* c_, int cat_) : c(c_), cat(cat_) {
    if (c->prof_mode == 2) {
      cudaEvent_t a = c->prof_ev();
      b = c->prof_ev();
      cudaEventRecord(a, c->stream);
      c->prof_recs.push_back({cat, a, b});
    }
  }
  ~Prof() {
    if (b) cudaEventRecord(b, c->stream);
  }
};

// ------------------------------------------------------------------------------ setup

static vi_status validate(const vi_config* k, std::string* why) {
  auto bad = [&](const char* m) {
    *why = m;
    return VI_E_CONFIG;
  };
  if (k->layers < 1 || k->heads < 1 || k->d_model < 1 || k->mem_frames < 0 || k->max_new_frames < 1)
    return bad("layers, heads, d_model, max_new_frames must be >= 1 and mem_frames >= 0");
  if (k->ref_rate < 0 || k->max_ref_frames < 0) return bad("ref_rate and max_ref_frames must be >= 0");
  if (k->refined_mem && (k->refined_span < 0 || k->refined_rate < 0 || k->max_refined_refs < 0))
    return bad("refined_span, refined_rate and max_refined_refs must be >= 0");
  if (k->mem_frames + k->max_new_frames + (k->ref_rate > 0 ? k->max_ref_frames : 0) +
          (k->refined_mem ? k->refined_span + 1 + (k->refined_rate > 0 ? k->max_refined_refs : 0) : 0) > 64)
    return bad("mem_frames + max_new_frames + max_ref_frames + refined slots must be <= 64");
  if (k->refined_mem && k->win_h > 0) return bad("refined memory: not built for window attention (no refine commits)");
  if (k->d_model % k->heads) return bad("d_model must be divisible by heads");
  const int hd = k->d_model / k->heads;
  if (k->dtype != VI_DTYPE_BF16 && k->dtype != VI_DTYPE_FP32) return bad("dtype must be 0 (bf16) or 1 (fp32)");
  if (k->kh < 1 || k->kw < 1 || k->sh < 1 || k->sw < 1 || k->ph < 0 || k->pw < 0) return bad("bad split geometry");
  const int oh = (k->feat_h + 2 * k->ph - k->kh) / k->sh + 1, ow = (k->feat_w + 2 * k->pw - k->kw) / k->sw + 1;
  if (oh < 1 || ow < 1 || oh * ow != k->tokens_per_frame) return bad("tokens_per_frame != oh*ow of the split geometry");
  // every cell must be covered by a window (the composite divides by the count)
  if (k->kh < k->sh || k->kw < k->sw || (oh - 1) * k->sh - k->ph + k->kh < k->feat_h ||
      (ow - 1) * k->sw - k->pw + k->kw < k->feat_w || k->ph >= k->kh || k->pw >= k->kw)
    return bad("split geometry leaves feature cells uncovered");
  if ((k->kh + k->sh - 1) / k->sh > 3 || (k->kw + k->sw - 1) / k->sw > 3)
    return bad("soft split/composite kernels support at most 3 overlapping windows per dimension");
  const int vec = k->dtype == VI_DTYPE_BF16 ? 8 : 4;
  if (k->feat_c % vec) return bad("feat_c must be a multiple of 8 (bf16) / 4 (fp32)");
  if (k->ffn_hidden < 1 || (k->ffn_kind != VI_FFN_MLP && k->ffn_kind != VI_FFN_F3N)) return bad("bad ffn");
  if (k->ffn_kind == VI_FFN_F3N) {
    if (k->ffn_hidden % (k->kh * k->kw)) return bad("F3N needs ffn_hidden % (kh*kw) == 0");
    if ((k->ffn_hidden / (k->kh * k->kw)) % vec) return bad("F3N hidden channels must be a multiple of 8/4");
  }
  if (k->dtype == VI_DTYPE_BF16) {
    if (hd != 64 && hd != 128) return bad("bf16 path: head dim must be 64 or 128");
    if (k->d_model % 64 || k->ffn_hidden % 8) return bad("bf16 path: d_model % 64 and ffn_hidden % 8 required");
    if ((k->kh * k->kw * k->feat_c) % 64) return bad("bf16 path: patch dim must be a multiple of 64");
  } else {
    if (hd % 32 || hd > 128) return bad("fp32 path: head dim must be a multiple of 32, <= 128");
    if (k->d_model > 1024) return bad("d_model <= 1024");
  }
  if (k->d_model > 1024) return bad("d_model <= 1024 (LayerNorm kernel)");
  if (k->win_h < 0 || k->win_w < 0 || (k->win_h > 0) != (k->win_w > 0)) return bad("win_h / win_w: both 0 or both > 0");
  if (k->win_h > 0) {
    if (k->dtype != VI_DTYPE_BF16) return bad("window attention: bf16 path only");
    if (oh % k->win_h || ow % k->win_w) return bad("window attention: windows must tile the token grid");
    if (k->tp_size > k->heads) {   // q = tp_size / heads ranks per head split its windows by window rows
      const int q = k->tp_size / k->heads;
      if (k->tp_size % k->heads || (oh / k->win_h) % q || k->tokens_per_frame % q)
        return bad("window attention with tp_size > heads: tp_size / heads must divide the window rows");
    }
  }
  const int G = k->tp_size < 1 ? 1 : k->tp_size;
  if (G > 1 || k->nccl_id) {
    TpLayout t;
    if (k->dtype != VI_DTYPE_BF16) return bad("head sharding: bf16 path only");
    if (k->tp_rank < 0 || k->tp_rank >= G) return bad("tp_rank out of [0, tp_size)");
    if (!tp_layout(k->heads, hd, k->max_new_frames * k->tokens_per_frame, G, k->tp_rank, &t))
      return bad("tp_size must divide heads or be a multiple of heads");
  }
  return VI_OK;
}

extern "C" vi_status vi_config_default(vi_config* k) {
  if (!k) return VI_E_ARG;
  std::memset(k, 0, sizeof(*k));
  k->layers = 8; k->heads = 4; k->d_model = 512; k->tokens_per_frame = 720; k->mem_frames = 10;
  k->max_new_frames = 5; k->feat_h = 60; k->feat_w = 108; k->feat_c = 128; k->kh = k->kw = 7;
  k->sh = k->sw = 3; k->ph = k->pw = 3; k->ffn_hidden = 1960; k->ffn_kind = VI_FFN_F3N;
  k->dtype = VI_DTYPE_BF16; k->pos_embed = 0; k->device = 0; k->stream = nullptr;
  return VI_OK;
}

static vi_status build_maps(vi_ctx* c) {
  const int rows = c->Tmax * c->P;
  bool ok = true;
  ok &= make_tmap(&c->tm_tokens, c->tokens, c->Pd, rows, 64, 128);
  ok &= make_tmap(&c->tm_wembed, c->w_embed, c->Pd, c->D, 64, c->bn_embed);
  ok &= make_tmap(&c->tm_h, c->h, c->D, rows, 64, 128);
  ok &= make_tmap(&c->tm_wqkv, c->w_qkv, c->D, (uint64_t)c->L * 3 * c->Dl, 64, c->bn_qkv);
  ok &= make_tmap(&c->tm_o, c->o, c->D, rows, 64, 128);
  ok &= make_tmap(&c->tm_wo, c->w_o, c->D, (uint64_t)c->L * c->D, 64, c->bn_o);
  ok &= make_tmap(&c->tm_w1, c->w_1, c->D, (uint64_t)c->L * c->F, 64, c->bn_1);
  ok &= make_tmap(&c->tm_w1_128, c->w_1, c->D, (uint64_t)c->L * c->F, 64, 128);
  ok &= make_tmap(&c->tm_g, c->gbuf, c->F, rows, 64, 128);
  ok &= make_tmap(&c->tm_w2, c->w_2, c->F, (uint64_t)c->L * c->D, 64, c->bn_2);
  ok &= make_tmap(&c->tm_w2_pair, c->w_2, c->F, (uint64_t)c->L * c->D, 64, 64);
  ok &= make_tmap(&c->tm_xb, c->xb, 2 * c->D, rows, 64, 128);
  ok &= make_tmap(&c->tm_wback, c->w_back2, 2 * c->D, c->Pd, 64, c->bn_back);
  ok &= make_tmap(&c->tm_q, c->q, c->Dl, (uint64_t)c->QR, 64, 128);
  ok &= make_tmap(&c->tm_k, c->kslab, c->Dl, (uint64_t)c->L * c->KR, 64, 128);
  ok &= make_tmap(&c->tm_vt, c->vtslab, (uint64_t)c->vt_ld, (uint64_t)c->L * c->Dl, 64, c->hd);
  if (c->sharded) ok &= make_tmap(&c->tm_og, c->og, c->hd, (uint64_t)c->H * c->tp.head_rows, 64, 128);
  ok &= make_tmap_out(&c->tm_u_out, c->u, true, c->F, rows);
  ok &= make_tmap_out(&c->tm_g_out, c->gbuf, false, c->F, rows);
  ok &= make_tmap_out(&c->tm_yp_out, c->yp32, true, c->Pd, rows);
  c->qkv_te = !c->win_n && c->P % 8 == 0 && c->Dl % 64 == 0;
  if (c->qkv_te) {
    ok &= make_tmap_out(&c->tm_q_out, c->q, false, c->Dl, (uint64_t)c->QR);
    ok &= make_tmap_box(&c->tm_k_out, c->kslab, c->Dl, (uint64_t)c->L * c->KR, 64, 8, true);
    ok &= make_tmap_box(&c->tm_vt_out, c->vtslab, (uint64_t)c->vt_ld, (uint64_t)c->L * c->Dl, 8, 64, false);
  }
  return ok ? VI_OK : c->fail(VI_E_CUDA, "cuTensorMapEncodeTiled failed");
}

extern "C" vi_status vi_create_ex(vi_ctx** out, const vi_config* cfg) {
  if (!out || !cfg) return VI_E_ARG;
  *out = nullptr;
  std::string why;
  vi_status st = validate(cfg, &why);
  if (st != VI_OK) return st;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || cfg->device < 0 || cfg->device >= ndev) {
    cudaGetLastError();
    return VI_E_CUDA;
  }
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, cfg->device) != cudaSuccess || prop.major != 10) return VI_E_CUDA;
  if (cudaSetDevice(cfg->device) != cudaSuccess) return VI_E_CUDA;

  vi_ctx* c = new (std::nothrow) vi_ctx();
  if (!c) return VI_E_OOM;
  c->cfg = *cfg;
  c->L = cfg->layers; c->H = cfg->heads; c->D = cfg->d_model; c->hd = c->D / c->H;
  c->P = cfg->tokens_per_frame; c->M = cfg->mem_frames; c->Tmax = cfg->max_new_frames; c->S = c->M + c->Tmax;
  c->ring = Ring(c->M, c->Tmax, cfg->ref_rate, cfg->max_ref_frames, cfg->refined_mem, cfg->refined_span,
                 cfg->refined_rate, cfg->max_refined_refs);
  c->ST = c->ring.slots();
  c->F = cfg->ffn_hidden; c->Pd = cfg->kh * cfg->kw * cfg->feat_c;
  if (cfg->win_h > 0) {
    const int oh = (cfg->feat_h + 2 * cfg->ph - cfg->kh) / cfg->sh + 1, ow = (cfg->feat_w + 2 * cfg->pw - cfg->kw) / cfg->sw + 1;
    c->win_cols = ow / cfg->win_w;
    c->win_n = (oh / cfg->win_h) * c->win_cols;
    c->win_real = cfg->win_h * cfg->win_w;
    // rows per (window, frame): no padding (pad rows cost a per-key mask in the softmax); a
    // window's key region is padded to 8 rows so every V^T box starts 16-byte aligned
    c->win_pad = c->win_real;
    c->win_kstride = (c->ST * c->win_pad + 7) / 8 * 8;
    c->KR = c->win_n * c->win_kstride;
    c->QR = c->win_n * c->Tmax * c->win_pad;
  } else {
    c->KR = c->ST * c->P;
    c->QR = c->Tmax * c->P;
  }
  c->vt_ld = (c->KR + 63) / 64 * 64;
  c->bf16 = cfg->dtype == VI_DTYPE_BF16; c->es = c->bf16 ? 2 : 4;

  {
    const int G = cfg->tp_size < 1 ? 1 : cfg->tp_size;
    c->sharded = G > 1 || cfg->nccl_id != nullptr;
    tp_layout(c->H, c->hd, c->Tmax * c->P, G, c->sharded ? cfg->tp_rank : 0, &c->tp);
    c->Hl = c->tp.nheads;
    c->Dl = c->Hl * c->hd;
    c->win_split = c->sharded && cfg->win_h > 0 && c->tp.qparts > 1;
    c->cfg.nccl_id = nullptr;   // caller memory: only read here
  }
  const int oh = (cfg->feat_h + 2 * cfg->ph - cfg->kh) / cfg->sh + 1;
  const int ow = (cfg->feat_w + 2 * cfg->pw - cfg->kw) / cfg->sw + 1;
  c->g = Geom{cfg->feat_h, cfg->feat_w, cfg->feat_c, cfg->kh, cfg->kw, cfg->sh, cfg->sw, cfg->ph, cfg->pw, oh, ow};
  c->gf = c->g;
  c->gf.C = cfg->ffn_kind == VI_FFN_F3N ? c->F / (cfg->kh * cfg->kw) : 0;
  if (cfg->stream) {
    c->stream = static_cast<cudaStream_t>(cfg->stream);
  } else {
    if (cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, cfg->stream_priority) != cudaSuccess) {
      delete c;
      return VI_E_CUDA;
    }
    c->own_stream = true;
  }
  if (cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete c;
    return VI_E_CUDA;
  }
  const size_t es = c->es, L = c->L, D = c->D, F = c->F, Pd = c->Pd, S = c->ST, P = c->P;
  const size_t rows = (size_t)c->Tmax * P;
  const size_t fmap = (size_t)c->Tmax * cfg->feat_h * cfg->feat_w * cfg->feat_c;
  bool ok = true;
  auto A = [&](size_t bytes) {
    void* p = c->dalloc(bytes);
    ok &= p != nullptr;
    return p;
  };
  c->w_embed = A(D * Pd * es); c->b_embed = (float*)A(D * 4); c->pos = (float*)A(P * D * 4);
  c->ln1_g = (float*)A(L * D * 4); c->ln1_b = (float*)A(L * D * 4);
  const size_t Dl = c->Dl;
  c->w_qkv = A(L * 3 * Dl * D * es); c->b_qkv = (float*)A(L * 3 * Dl * 4);   // this rank's heads only
  c->w_o = A(L * D * D * es); c->b_o = (float*)A(L * D * 4);
  c->ln2_g = (float*)A(L * D * 4); c->ln2_b = (float*)A(L * D * 4);
  c->w_1 = A(L * F * D * es); c->b_1 = (float*)A(L * F * 4);
  c->w_2 = A(L * D * F * es); c->b_2 = (float*)A(L * D * 4);
  c->w_back = A(Pd * D * es); c->b_back = (float*)A(Pd * 4);
  c->kslab = A(L * (size_t)c->KR * Dl * es); c->vtslab = A(L * Dl * (size_t)c->vt_ld * es);
  c->tokens = A(rows * Pd * es); c->h = A(rows * D * es); c->q = A((size_t)c->QR * Dl * es); c->o = A(rows * D * es);
  if (c->sharded) c->og = A((size_t)c->H * c->tp.head_rows * c->hd * es);
  c->u = A(rows * F * 4);   // FFN1 output kept fp32 for the F3N fold (one rounding less)
  c->gbuf = A(rows * F * es); c->xb = A(rows * 2 * D * es);
  if (c->bf16) {
    c->yp32 = A(rows * Pd * 4);          // back-projection output kept fp32 for the fold
    c->w_back2 = A(Pd * 2 * D * es);     // [Wb | Wb] for the hi/lo split of x
  }
  c->x_ws = (float*)A(rows * D * 4);
  c->fold_ws = (float*)A((size_t)c->Tmax * cfg->feat_h * cfg->feat_w * std::max(c->gf.C, 1) * 4);
  if (c->bf16) {
    c->opart = (vi::bf16*)A((size_t)kMaxSplit * std::max(rows, (size_t)c->QR) * D * 2);
    c->lse = (float*)A((size_t)kMaxSplit * c->H * std::max(rows, (size_t)c->QR) * 4);
  }
  c->feat_in = A(fmap * es); c->feat_out = A(fmap * es);
  c->attn_timing = (unsigned long long*)A(3 * sizeof(KernelTiming));   // [0] attention, [1] GEMMs, [2] patch
  c->num_sms = prop.multiProcessorCount;
  if (c->bf16) {
    c->sk_part = (float*)A((size_t)c->num_sms * 256 * c->hd * 4);
    c->sk_lse = (float*)A((size_t)2 * c->num_sms * 256 * 4);   // two piece slots per CTA
    c->sk_units_cap = ((c->QR + 255) / 256 + c->win_n + 1) * c->H;
    c->sk_flag = (int*)A((size_t)2 * c->sk_units_cap * 4);   // stream-K unit parts [2][units]
    // split-K partials: num_sms 128 x 128 tiles, or two k-halves of a CTA-pair-tiled chunk
    c->skws_floats = std::max((size_t)c->num_sms * 128 * 128, (size_t)2 * ((rows + 255) / 256 * 256) * D);
    c->skws = (float*)A(c->skws_floats * 4);
  }
  if (!ok) {
    delete c;
    return VI_E_OOM;
  }
  if (cudaEventCreateWithFlags(&c->ev_attn, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_gather, cudaEventDisableTiming) != cudaSuccess) {
    delete c;
    return VI_E_CUDA;
  }
  if (cfg->nccl_id) {   // collective: every rank of the group is inside this call
    const Nccl& nc = nccl();
    NcclId id;
    std::memcpy(&id, cfg->nccl_id, sizeof(id));
    if (!nc.ok || nc.comm_init_rank(&c->comm, c->tp.G, id, c->tp.rank) != 0) {
      c->comm = nullptr;
      delete c;
      return VI_E_NCCL;
    }
  }
  if (cudaDeviceSynchronize() != cudaSuccess) {
    delete c;
    return VI_E_CUDA;
  }
  {
    KernelTiming kt[3];
    std::memset(kt, 0, sizeof(kt));
    kt[0].tmin = kt[1].tmin = kt[2].tmin = ~0ull;
    if (cudaMemcpy(c->attn_timing, kt, sizeof(kt), cudaMemcpyHostToDevice) != cudaSuccess) {
      delete c;
      return VI_E_CUDA;
    }
    const char* ng = getenv("VI_NO_GRAPH");
    c->use_graphs = !(ng && ng[0] == '1') && c->own_stream;
  }
  if (c->bf16) {
    if (c->D % 128) c->bn_o = c->bn_2 = 64;
    if (build_maps(c) != VI_OK) {
      delete c;
      return VI_E_CUDA;
    }
  }
  *out = c;
  return VI_OK;
}

extern "C" vi_status vi_create(vi_ctx** out, int layers, int heads, int d_model, int tokens_per_frame,
                               int mem_frames) {
  vi_config k;
  vi_config_default(&k);
  k.layers = layers; k.heads = heads; k.d_model = d_model; k.tokens_per_frame = tokens_per_frame;
  k.mem_frames = mem_frames;
  return vi_create_ex(out, &k);
}

extern "C" vi_status vi_destroy(vi_ctx* c) {
  delete c;
  return VI_OK;
}

static vi_status upload_mat(vi_ctx* c, void* dst, const float* src, size_t n) {
  if (c->bf16) {
    std::vector<uint16_t> tmp(n);
    for (size_t i = 0; i < n; ++i) tmp[i] = f2bf(src[i]);
    CK(cudaMemcpy(dst, tmp.data(), n * 2, cudaMemcpyHostToDevice), "upload");
  } else {
    CK(cudaMemcpy(dst, src, n * 4, cudaMemcpyHostToDevice), "upload");
  }
  return VI_OK;
}
static vi_status upload_f32(vi_ctx* c, float* dst, const float* src, size_t n) {
  CK(cudaMemcpy(dst, src, n * 4, cudaMemcpyHostToDevice), "upload");
  return VI_OK;
}

extern "C" vi_status vi_set_weights(vi_ctx* c, const vi_weights* w) {
  LIVE(c);
  DeviceGuard dg_(c->cfg.device);
  if (!w || !w->embed_w || !w->embed_b || !w->ln1_g || !w->ln1_b || !w->wqkv || !w->bqkv || !w->wo || !w->bo ||
      !w->ln2_g || !w->ln2_b || !w->w1 || !w->b1 || !w->w2 || !w->b2 || !w->back_w || !w->back_b)
    return c->fail(VI_E_ARG, "vi_set_weights: NULL weight pointer");
  if (c->cfg.pos_embed && !w->pos) return c->fail(VI_E_ARG, "vi_set_weights: pos_embed=1 needs pos");
  CK(cudaStreamSynchronize(c->stream), "set_weights sync");
  const size_t L = c->L, D = c->D, F = c->F, Pd = c->Pd;
  vi_status st = VI_OK;
  auto U = [&](vi_status s) {
    if (s != VI_OK) st = s;
  };
  U(upload_mat(c, c->w_embed, w->embed_w, D * Pd));
  U(upload_f32(c, c->b_embed, w->embed_b, D));
  if (c->cfg.pos_embed) U(upload_f32(c, c->pos, w->pos, (size_t)c->P * D));
  U(upload_f32(c, c->ln1_g, w->ln1_g, L * D));
  U(upload_f32(c, c->ln1_b, w->ln1_b, L * D));
  if (c->sharded) {   // this rank's heads: rows [part*D + head0*hd, +Dl) of Wq, Wk, Wv
    const size_t Dl = c->Dl, h0 = (size_t)c->tp.head0 * c->hd;
    std::vector<float> wl(L * 3 * Dl * D), bl(L * 3 * Dl);
    for (size_t l = 0; l < L; ++l)
      for (size_t part = 0; part < 3; ++part) {
        std::memcpy(&wl[(l * 3 + part) * Dl * D], w->wqkv + (l * 3 * D + part * D + h0) * D, Dl * D * 4);
        std::memcpy(&bl[(l * 3 + part) * Dl], w->bqkv + l * 3 * D + part * D + h0, Dl * 4);
      }
    U(upload_mat(c, c->w_qkv, wl.data(), L * 3 * Dl * D));
    U(upload_f32(c, c->b_qkv, bl.data(), L * 3 * Dl));
  } else {
    U(upload_mat(c, c->w_qkv, w->wqkv, L * 3 * D * D));
    U(upload_f32(c, c->b_qkv, w->bqkv, L * 3 * D));
  }
  U(upload_mat(c, c->w_o, w->wo, L * D * D));
  U(upload_f32(c, c->b_o, w->bo, L * D));
  U(upload_f32(c, c->ln2_g, w->ln2_g, L * D));
  U(upload_f32(c, c->ln2_b, w->ln2_b, L * D));
  U(upload_mat(c, c->w_1, w->w1, L * F * D));
  U(upload_f32(c, c->b_1, w->b1, L * F));
  U(upload_mat(c, c->w_2, w->w2, L * D * F));
  U(upload_f32(c, c->b_2, w->b2, L * D));
  U(upload_mat(c, c->w_back, w->back_w, Pd * D));
  if (c->bf16) {   // [Wb | Wb]: row r = (Wb[r], Wb[r])
    std::vector<float> w2(Pd * 2 * D);
    for (size_t r = 0; r < Pd; ++r) {
      std::memcpy(&w2[r * 2 * D], w->back_w + r * D, D * 4);
      std::memcpy(&w2[r * 2 * D + D], w->back_w + r * D, D * 4);
    }
    U(upload_mat(c, c->w_back2, w2.data(), Pd * 2 * D));
  }
  U(upload_f32(c, c->b_back, w->back_b, Pd));
  if (st == VI_OK) c->have_weights = true;
  ++c->weights_gen;
  return st;
}

// ------------------------------------------------------------------------------ ring

static vi_status apply_commits(vi_ctx* c, const std::vector<int64_t>& ids) {
  const size_t es = c->es, P = c->P, D = c->D, Dl = c->Dl, SP = (size_t)c->ST * c->P;
  const size_t h0 = (size_t)c->tp.head0 * c->hd;   // this rank's columns of the full [P][D] payload
  for (int64_t id : ids) {
    auto it = c->pending_kv.find(id);
    if (it == c->pending_kv.end()) continue;
    const int slot = c->ring.slot_of(id);
    if (slot < 0) continue;
    for (int l = 0; l < c->L; ++l) {
      const uint8_t* ksrc = static_cast<const uint8_t*>(it->second.k) + ((size_t)l * P * D + h0) * es;
      const uint8_t* vsrc = static_cast<const uint8_t*>(it->second.v) + ((size_t)l * P * D + h0) * es;
      uint8_t* kdst = static_cast<uint8_t*>(c->kslab) + ((size_t)l * SP + (size_t)slot * P) * Dl * es;
      CK(cudaMemcpy2DAsync(kdst, Dl * es, ksrc, D * es, Dl * es, P, cudaMemcpyDeviceToDevice, c->stream), "commit K");
      uint8_t* vt = static_cast<uint8_t*>(c->vtslab) + (size_t)l * Dl * c->vt_ld * es;
      PLAUNCH(VI_PROF_ROW,
              launch_transpose_to_slab(vsrc, vt, c->P, c->Dl, c->vt_ld, (size_t)slot * P, c->bf16 ? 0 : 1, c->stream, c->D),
              "commit V");
    }
  }
  return VI_OK;
}

// Frames becoming references (ring.h): their K rows and Vt columns move from the span slot
// to the reference slot, on the ctx stream before the new chunk's step overwrites the span slot.
static vi_status apply_moves(vi_ctx* c, const std::vector<Ring::Move>& moves) {
  const size_t es = c->es, P = c->P, Dl = c->Dl, SP = (size_t)c->KR, ld = c->vt_ld;
  if (c->win_n) {   // window-major memory: a slot is win_pad rows inside every window's region
    const size_t wp = c->win_pad, ks = c->win_kstride;
    for (const auto& mv : moves) {
      for (int l = 0; l < c->L; ++l) {
        uint8_t* kb = static_cast<uint8_t*>(c->kslab) + (size_t)l * SP * Dl * es;
        CK(cudaMemcpy2DAsync(kb + (size_t)mv.dst * wp * Dl * es, ks * Dl * es, kb + (size_t)mv.src * wp * Dl * es,
                             ks * Dl * es, wp * Dl * es, c->win_n, cudaMemcpyDeviceToDevice, c->stream),
           "reference move K");
        uint8_t* vb = static_cast<uint8_t*>(c->vtslab) + (size_t)l * Dl * ld * es;
        for (int w = 0; w < c->win_n; ++w)
          CK(cudaMemcpy2DAsync(vb + ((size_t)w * ks + (size_t)mv.dst * wp) * es, ld * es,
                               vb + ((size_t)w * ks + (size_t)mv.src * wp) * es, ld * es, wp * es, Dl,
                               cudaMemcpyDeviceToDevice, c->stream),
             "reference move V");
      }
    }
    return VI_OK;
  }
  for (const auto& mv : moves) {
    for (int l = 0; l < c->L; ++l) {
      uint8_t* kb = static_cast<uint8_t*>(c->kslab) + (size_t)l * SP * Dl * es;
      CK(cudaMemcpyAsync(kb + (size_t)mv.dst * P * Dl * es, kb + (size_t)mv.src * P * Dl * es, P * Dl * es,
                         cudaMemcpyDeviceToDevice, c->stream),
         "reference move K");
      uint8_t* vb = static_cast<uint8_t*>(c->vtslab) + (size_t)l * Dl * ld * es;
      CK(cudaMemcpy2DAsync(vb + (size_t)mv.dst * P * es, ld * es, vb + (size_t)mv.src * P * es, ld * es, P * es, Dl,
                           cudaMemcpyDeviceToDevice, c->stream),
         "reference move V");
    }
  }
  return VI_OK;
}

extern "C" vi_status vi_memory_push(vi_ctx* c, int n, int64_t* first_id, int64_t* evicted, int* n_evicted) {
  LIVE(c);
  DeviceGuard dg_(c->cfg.device);
  if (n < 1 || n > c->Tmax) return c->fail(VI_E_ARG, "vi_memory_push: n out of [1, max_new_frames]");
  std::lock_guard<std::mutex> lk(c->mu);
  std::vector<int64_t> ev, apply;
  std::vector<Ring::Move> moves;
  const int64_t f = c->ring.push(n, &ev, &apply, &moves);
  vi_status st = apply_moves(c, moves);
  if (st == VI_OK) st = apply_commits(c, apply);
  // all queued payloads are consumed (applied, or dropped because the frame left)
  for (auto& kv : c->pending_kv) {
    if (st == VI_OK) {
      cudaError_t e = cudaEventRecord(kv.second.released, c->stream);
      if (e != cudaSuccess) st = c->cuda_fail(e, "commit release");
    }
    c->free_kv.push_back(kv.second);
  }
  c->pending_kv.clear();
  if (st != VI_OK) return st;
  c->next_layer = 0;
  c->attn_layer = -1;
  if (first_id) *first_id = f;
  if (evicted)
    for (size_t i = 0; i < ev.size(); ++i) evicted[i] = ev[i];
  if (n_evicted) *n_evicted = int(ev.size());
  return VI_OK;
}

extern "C" vi_status vi_memory_evict(vi_ctx* c, int64_t frame_id) {
  LIVE(c);
  DeviceGuard dg_(c->cfg.device);
  std::lock_guard<std::mutex> lk(c->mu);
  const vi_status st = c->ring.evict(frame_id);
  if (st == VI_OK) {
    auto it = c->pending_kv.find(frame_id);
    if (it != c->pending_kv.end()) {
      c->free_kv.push_back(it->second);
      c->pending_kv.erase(it);
    }
  }
  return st;
}

extern "C" vi_status vi_refine_commit(vi_ctx* c, int64_t frame_id, const void* k, const void* v) {
  LIVE(c);
  DeviceGuard dg_(c->cfg.device);
  if (!k || !v) return VI_E_ARG;
  if (c->win_n) return c->fail(VI_E_CONFIG, "vi_refine_commit: not built for window attention (window-major memory)");
  std::lock_guard<std::mutex> lk(c->mu);
  const vi_status st = c->ring.commit(frame_id);
  if (st != VI_OK) return st;
  const size_t bytes = (size_t)c->L * c->P * c->D * c->es;
  auto it = c->pending_kv.find(frame_id);
  vi_ctx::KvBuf buf;
  if (it != c->pending_kv.end()) {
    buf = it->second;                       // queued, not applied yet: overwrite in place
  } else if (!c->free_kv.empty()) {
    buf = c->free_kv.back();
    c->free_kv.pop_back();
    // the apply copies that read this buffer at an earlier push must be done
    CK(cudaStreamWaitEvent(c->copy_stream, buf.released, 0), "commit wait");
  } else {
    if (cudaMalloc(&buf.k, bytes) != cudaSuccess || cudaMalloc(&buf.v, bytes) != cudaSuccess ||
        cudaEventCreateWithFlags(&buf.released, cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      if (buf.k) cudaFree(buf.k);
      if (buf.v) cudaFree(buf.v);
      return c->fail(VI_E_OOM, "vi_refine_commit: staging allocation failed");
    }
  }
  const cudaMemcpyKind kk = is_host_ptr(k) ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
  const cudaMemcpyKind kv = is_host_ptr(v) ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
  CK(cudaMemcpyAsync(buf.k, k, bytes, kk, c->copy_stream), "commit copy K");
  CK(cudaMemcpyAsync(buf.v, v, bytes, kv, c->copy_stream), "commit copy V");
  CK(cudaStreamSynchronize(c->copy_stream), "commit sync");
  c->pending_kv[frame_id] = buf;
  return VI_OK;
}

extern "C" vi_status vi_memory_read(vi_ctx* c, int64_t frame_id, void* k, void* v) {
  LIVE(c);
  DeviceGuard dg_(c->cfg.device);
  if (!k || !v) return c->fail(VI_E_ARG, "vi_memory_read: NULL buffer");
  if (c->win_n) return c->fail(VI_E_CONFIG, "vi_memory_read: not built for window attention (window-major memory)");
  {
    std::lock_guard<std::mutex> lk(c->mu);
    const int32_t st = c->ring.check_past(frame_id);
    if (st != VI_OK) return st;
  }
  const size_t es = c->es, P = c->P, Dl = c->Dl, SP = (size_t)c->ST * c->P, per = P * Dl * es;
  size_t slot;
  {
    std::lock_guard<std::mutex> lk(c->mu);
    slot = size_t(c->ring.slot_of(frame_id));
  }
  const bool hk = is_host_ptr(k), hv = is_host_ptr(v);
  // V leaves the slab through a transpose kernel: a host destination is staged on the device
  void* vd = v;
  if (hv && cudaMalloc(&vd, (size_t)c->L * per) != cudaSuccess) {
    cudaGetLastError();
    return c->fail(VI_E_OOM, "vi_memory_read: staging allocation failed");
  }
  vi_status st = VI_OK;
  for (int l = 0; l < c->L && st == VI_OK; ++l) {
    const uint8_t* ks = static_cast<const uint8_t*>(c->kslab) + ((size_t)l * SP + slot * P) * Dl * es;
    cudaError_t e = cudaMemcpyAsync(static_cast<uint8_t*>(k) + l * per, ks, per,
                                    hk ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, c->stream);
    if (e != cudaSuccess) st = c->cuda_fail(e, "memory_read K");
    // Vt [Dl][vt_ld] columns slot*P.. (a [Dl][P] matrix of pitch vt_ld) -> [P][Dl]
    const uint8_t* vs = static_cast<const uint8_t*>(c->vtslab) + ((size_t)l * Dl * c->vt_ld + slot * P) * es;
    if (st == VI_OK) {
      e = launch_transpose_to_slab(vs, static_cast<uint8_t*>(vd) + l * per, c->Dl, c->P, c->Dl, 0, c->bf16 ? 0 : 1,
                                   c->stream, c->vt_ld);
      ++c->launches;
      if (e != cudaSuccess) st = c->cuda_fail(e, "memory_read V");
    }
  }
  if (st == VI_OK && hv) {
    cudaError_t e = cudaMemcpyAsync(v, vd, (size_t)c->L * per, cudaMemcpyDeviceToHost, c->stream);
    if (e != cudaSuccess) st = c->cuda_fail(e, "memory_read V d2h");
  }
  cudaError_t e = cudaStreamSynchronize(c->stream);
  if (st == VI_OK && e != cudaSuccess) st = c->cuda_fail(e, "memory_read sync");
  if (hv) cudaFree(vd);
  return st;
}

extern "C" vi_status vi_memory_state(vi_ctx* c, int64_t* slot_id, uint8_t* refined, uint64_t* valid_mask) {
  if (!c) return VI_E_ARG;
  std::lock_guard<std::mutex> lk(c->mu);
  for (int s = 0; s < c->ST; ++s) {
    if (slot_id) slot_id[s] = c->ring.slot_id[s];
    if (refined) refined[s] = c->ring.refined[s];
  }
  if (valid_mask) *valid_mask = c->ring.valid_mask();
  return VI_OK;
}

// ------------------------------------------------------------------------------ compute

// the patch kernels' self-timing slot (vi_profile mode 3) or NULL; VI_PATCH_TIME_ONLY=<kind>
// (s split, f F3N fold, u F3N unfold, c composite) times that kernel alone (breakdowns)
static unsigned long long* patch_timing(const vi_ctx* c, char kind) {
  static const char only = [] {
    const char* e = getenv("VI_PATCH_TIME_ONLY");
    return e && e[0] ? e[0] : '\0';
  }();
  if (c->prof_mode != 3 || (only && only != kind)) return nullptr;
  return c->attn_timing + 2 * (sizeof(KernelTiming) / sizeof(unsigned long long));
}
static Epi epi_base(const vi_ctx* c, int kind, int M, int N, const float* bias) {
  Epi e;
  std::memset(&e, 0, sizeof(e));
  e.kind = kind; e.M = M; e.N = N; e.bias = bias; e.P = 1; e.S = 1;
  if (c->prof_mode == 3)   // the GEMMs' self-timing slot (vi_profile mode 3)
    e.timing = c->attn_timing + sizeof(KernelTiming) / sizeof(unsigned long long);
  return e;
}

// Split-K plan for a residual GEMM [M x N] += A[M x K] W^T.
//  * single-CTA 128 x 128 tiles: when the output has at most num_sms / 2 tiles (one frame per
//    chunk, the paper's T = 1 mode) most SMs would idle, so every tile's k-blocks are cut into
//    ks consecutive ranges, one work item each (<= num_sms items).
//  * CTA-pair 256 x 256 tiles, ks = 2 (returned with kSplitPair set): the patch embedding at
//    full chunks (K = 6272; C3: 15 x 2 pair tiles -> 60 work items on 74 SM pairs).  A 256 x 256
//    pair tile runs the MMA at the full per-SM rate where 128 x 128 tiles are operand-bound at
//    about half of it (tools/micro/gemm_splitk: embedding + LN 41.0 -> 33.3 us); block 0's LN1
//    rides on the reduction.  (FFN2, K = 1960, measured no faster in the step.)
// Returns 0 (do not split), ks, or ks | kSplitPair.
static constexpr int kSplitPair = 1 << 8;
static int splitk_plan(const vi_ctx* c, int M, int N, int K) {
  if (!splitk_enabled() || !c->bf16 || !c->skws || N % 128) return 0;
  const int out = (M + 127) / 128 * (N / 128), nk = (K + 63) / 64;
  if (out * 2 > c->num_sms) {
    const int pair_tiles = (M + 255) / 256 * (N / 256);
    if (N % 256 || K < 4096 || 2 * pair_tiles > c->num_sms / 2 ||
        (size_t)2 * ((M + 255) / 256 * 256) * N > c->skws_floats)
      return 0;
    return 2 | kSplitPair;
  }
  int ks = std::min(std::min(c->num_sms / out, 8), nk);
  if (ks < 2) return 0;
  const int kper = (nk + ks - 1) / ks;
  ks = (nk + kper - 1) / kper;   // every split non-empty
  return ks < 2 ? 0 : ks;
}

// x_out = x_in + bias + A W^T through ks split-K partials and the deterministic reduction
// (which also writes LayerNorm(x_out) to h when ln_g != NULL).  plan = splitk_plan's value;
// with kSplitPair the partials come from CTA-pair 256 x 256 tiles (wmap's box: 64 x 128).
static vi_status splitk_resid(vi_ctx* c, int plan, const CUtensorMap& amap, const CUtensorMap& wmap, int brow0, int M,
                              int N, int K, int a_hs, int a_kpb, const float* bias, const float* x_in, float* x_out,
                              const float* pos, const float* ln_g, const float* ln_b, void* h, const char* where) {
  const bool pair = plan & kSplitPair;
  const int ks = plan & (kSplitPair - 1);
  const int kpad = pair ? (M + 255) / 256 * 256 : (M + 127) / 128 * 128;
  Epi e = epi_base(c, EPI_STORE, M, N, nullptr);
  e.out = c->skws; e.ldo = N; e.out_f32 = 1;
  e.ksplit = ks; e.kpad_rows = kpad;
  e.a_hs = a_hs; e.a_kpb = a_kpb;
  CUtensorMap tws;
  if (!make_tmap_out(&tws, c->skws, true, N, (uint64_t)ks * kpad))
    return c->fail(VI_E_CUDA, std::string(where) + ": split-K workspace map");
  PLAUNCH(VI_PROF_GEMM, launch_gemm_tc(amap, wmap, brow0, M, N, K, pair ? 256 : 128, e, c->stream, pair ? 1 : 0, &tws, nullptr),
          where);
  PLAUNCH(VI_PROF_GEMM,
          launch_splitk_resid(c->skws, ks, (size_t)kpad * N, bias, x_in, x_out, pos, c->P, ln_g, ln_b, h, c->bf16 ? 0 : 1, M, N,
                              c->stream, e.timing),
          where);
  return VI_OK;
}

extern "C" vi_status vi_soft_split(vi_ctx* c, const void* feat, int n, void* out, int project) {
  LIVE(c);
  DeviceGuard dg_(c->cfg.device);
  if (!feat || !out || n < 1 || n > c->Tmax || (project != 0 && project != 1))
    return c->fail(VI_E_ARG, "vi_soft_split: bad argument");
  if (project && !c->have_weights) return c->fail(VI_E_PROTOCOL, "vi_soft_split: weights not set");
  const int dt = c->bf16 ? 0 : 1;
  void* tok = project ? c->tokens : out;
  PLAUNCH(VI_PROF_PATCH, launch_unfold(feat, tok, n, c->g, dt, c->stream, patch_timing(c, 's')), "unfold");
  if (project) {
    const int M = n * c->P;
    Epi e = epi_base(c, EPI_STORE, M, c->D, c->b_embed);
    e.out = out; e.ldo = c->D; e.out_f32 = 1; e.pos = c->cfg.pos_embed ? c->pos : nullptr; e.P = c->P;
    CUtensorMap tmo;
    const bool te = c->bf16 && make_tmap_out(&tmo, out, true, c->D, M);
    // small M (one frame: 24 output tiles, K = 6272): split-K partials + one reduction kernel
    const int ks = te && c->bn_embed == 128 ? splitk_plan(c, M, c->D, c->Pd) : 0;
    if (ks) {
      const bool ln0 = c->fuse_ln1;   // block 0's LN1 in the same pass (inside vi_run_step only)
      const vi_status r = splitk_resid(c, ks, c->tm_tokens, c->tm_wembed, 0, M, c->D, c->Pd, 0, 0, c->b_embed, nullptr,
                                       static_cast<float*>(out), e.pos, ln0 ? c->ln1_g : nullptr,
                                       ln0 ? c->ln1_b : nullptr, ln0 ? c->h : nullptr, "embed gemm (split-K)");
      if (r != VI_OK) return r;
      if (ln0) c->h_ready = 0;
    } else if (c->bf16)
      PLAUNCH(VI_PROF_GEMM, launch_gemm_tc(c->tm_tokens, c->tm_wembed, 0, M, c->D, c->Pd, c->bn_embed, e, c->stream, 0,
                                           te ? &tmo : nullptr),
              "embed gemm");
    else
      PLAUNCH(VI_PROF_GEMM, launch_gemm_simt_f32((const float*)c->tokens, (const float*)c->w_embed, M, c->D, c->Pd, e, c->stream),
             "embed gemm");
  }
  return VI_OK;
}

static void choose_split(int units, int ntiles, int* nsplit, int* tps) {
  double best = 1e30;
  *nsplit = 1;
  *tps = ntiles;
  for (int s = 1; s <= kMaxSplit && s <= ntiles; ++s) {
    const int t = (ntiles + s - 1) / s;
    const int waves = (units * s + 147) / 148;
    // per-CTA fixed cost (TMEM alloc, Q load, pipeline fill, partial epilogue) ~ 4 tiles
    const double cost = double(waves) * (t + 4.0) + (s > 1 ? 1.0 + 0.3 * s : 0.0);
    if (cost < best - 1e-9) {
      best = cost;
      *nsplit = s;
      *tps = t;
    }
  }
}

static KeySegs make_segs(const vi_ctx* c, uint64_t valid) {
  KeySegs k;
  std::memset(&k, 0, sizeof(k));
  int s = 0;
  while (s < c->ST) {
    if (!((valid >> s) & 1)) {
      ++s;
      continue;
    }
    int e = s;
    while (e + 1 < c->ST && ((valid >> (e + 1)) & 1)) ++e;
    const int rows_per_slot = c->win_n ? c->win_pad : c->P;   // windows: rows within the window's region
    const int r0 = s * rows_per_slot;
    k.row0[k.n] = r0 & ~7;
    k.lead[k.n] = r0 & 7;
    k.len[k.n] = (e - s + 1) * rows_per_slot + k.lead[k.n];
    k.tile0[k.n + 1] = k.tile0[k.n] + (k.len[k.n] + 127) / 128;
    ++k.n;
    s = e + 1;
  }
  return k;
}

// The attention half of block l: LN1, Q/K/V projection (this rank's heads) + memory write,
// attention over every valid slot.  Output: c->o [M][D] (unsharded) or this rank's chunk
// of the head-major gathered buffer c->og (head-sharded, tp.h).
static vi_status step_attn(vi_ctx* c, int l, const float* x_in) {
  const int n = c->ring.cur_n, M = n * c->P, D = c->D, Dl = c->Dl;
  const int dt = c->bf16 ? 0 : 1;
  const size_t es = c->es, SP = (size_t)c->KR;
  void* kl = static_cast<uint8_t*>(c->kslab) + (size_t)l * SP * Dl * es;
  void* vl = static_cast<uint8_t*>(c->vtslab) + (size_t)l * c->vt_ld * Dl * es;
  const uint64_t valid = c->ring.valid_mask();

  // a3: LN1 (unless the reduction that produced x_in wrote it)
  if (!(c->fuse_ln1 && c->h_ready == l))
    PLAUNCH(VI_PROF_ROW, launch_layernorm(x_in, c->ln1_g + (size_t)l * D, c->ln1_b + (size_t)l * D, c->h, dt, M, D, c->stream), "ln1");
  c->h_ready = -1;
  // a4: QKV projection + memory write
  Epi eq = epi_base(c, EPI_QKV, M, 3 * Dl, c->b_qkv + (size_t)l * 3 * Dl);
  eq.D = Dl; eq.q = c->q; eq.kslab = kl; eq.vtslab = vl; eq.first_slot = int(c->ring.cur_first % c->S);
  eq.S = c->S; eq.P = c->P; eq.vt_ld = c->vt_ld;
  if (c->win_n) {
    eq.win_pad = c->win_pad; eq.win_h = c->cfg.win_h; eq.win_w = c->cfg.win_w; eq.win_cols = c->win_cols;
    eq.ow = c->g.ow; eq.win_qstride = c->Tmax * c->win_pad; eq.win_kstride = c->win_kstride;
  }
  eq.qkv_krow0 = int(l * SP);
  eq.qkv_vrow0 = l * Dl;
  const bool qte = c->bf16 && c->qkv_te;
  if (c->bf16)
    PLAUNCH(VI_PROF_GEMM, launch_gemm_tc(c->tm_h, c->tm_wqkv, l * 3 * Dl, M, 3 * Dl, D, c->bn_qkv, eq, c->stream, 0,
                                         qte ? &c->tm_q_out : nullptr, qte ? &c->tm_k_out : nullptr,
                                         qte ? &c->tm_vt_out : nullptr),
            "qkv gemm");
  else
    PLAUNCH(VI_PROF_GEMM, launch_gemm_simt_f32((const float*)c->h, (const float*)c->w_qkv + (size_t)l * 3 * Dl * D, M, 3 * Dl, D,
                                               eq, c->stream),
            "qkv gemm");
  // a5: memory attention over every valid slot
  const float scale_log2 = float(1.4426950408889634 / std::sqrt(double(c->hd)));
  if (!c->bf16) {
    AttnArgs a;
    a.Nq = M; a.D = D; a.H = c->H; a.hd = c->hd; a.P = c->P; a.S = c->ST; a.vt_ld = c->vt_ld; a.valid = valid;
    a.scale_log2 = scale_log2; a.q = c->q; a.kslab = kl; a.vtslab = vl; a.o = c->o;
    PLAUNCH(VI_PROF_ATTN, launch_attn_simt_f32(a, c->stream), "attention");
    return VI_OK;
  }
  AttnTC a;
  std::memset(&a, 0, sizeof(a));
  a.Nq = M; a.hd = c->hd; a.D = Dl; a.H = c->Hl; a.krow_base = int(l * SP); a.vrow_base = l * Dl;
  a.scale_log2 = scale_log2; a.segs = make_segs(c, valid);
  a.o = static_cast<bf16*>(c->o); a.o_ld = D; a.o_hs = c->hd; a.q_row0 = 0;
  if (c->win_n) {   // window attention: the fixed KV split over (window, 256 queries) units
    a.win_n = c->win_n; a.win_qstride = c->Tmax * c->win_pad; a.win_kstride = c->win_kstride;
    a.win_pad = c->win_pad; a.win_real = c->win_real; a.win_h = c->cfg.win_h; a.win_w = c->cfg.win_w;
    a.win_cols = c->win_cols; a.ow = c->g.ow; a.P = c->P; a.win_nq = n * c->win_pad;
    a.win_npw = (a.win_nq + 255) / 256;
    a.Nq = c->win_n * a.win_qstride;   // rows of the KV-split partials (window-major)
  }
  if (c->sharded) {   // this rank's query rows, written head-major into its chunk of og
    if (!c->win_n) {
      a.q_row0 = c->tp.row0();
      a.Nq = c->tp.rows(M);
      if (a.Nq == 0) return VI_OK;   // a query part beyond a short chunk: nothing to attend
    } else if (c->win_split) {
      // q ranks per head: rank part p takes window rows [p*wr/q, (p+1)*wr/q) -- tokens
      // [p*P/q, (p+1)*P/q) of every frame -- and writes them part-locally (frame-major)
      const int q = c->tp.qparts, nw = c->win_n / q;
      a.win_n = nw;
      a.win0 = c->tp.qpart * nw;
      a.win_split_rows = c->P / q;
      a.win_part = c->tp.qpart;
      a.Nq = nw * a.win_qstride;
    }
    a.o = static_cast<bf16*>(c->og) + (size_t)c->tp.rank * c->tp.chunk_elems;
    a.o_ld = c->hd;
    a.o_hs = c->tp.head_rows * c->hd;
  }
  const int ntiles = a.segs.tile0[a.segs.n];
  a.opart = c->opart; a.lse = c->lse;
  a.timing = (c->prof_mode == 1 || c->prof_mode == 3 || c->prof_mode == 4) ? c->attn_timing : nullptr;
  a.combine_timing = c->prof_mode == 4 ? nullptr : a.timing;   // mode 4: the attention kernel alone
  // Stream-K needs enough (query-pair, head) units: with few units (a chunk of one frame:
  // 720 queries -> 12 units for 148 SMs) every unit splits ~12 ways, so small chunks take the
  // fixed KV split + parallel combine kernel (round 1, owner merge: C3T1 28 vs 60 us per block;
  // round 2, PDL-launched stream-K + combine kernel: C3T1 step 0.603 vs 0.598 ms, C2 0.436 vs
  // 0.441 -- mixed, the KV split stays).
  const int sk_units = ((a.Nq + 255) / 256) * a.H;
  const bool small = sk_units * 4 < c->num_sms;
  // window attention: sk2 over (head, window, query pair) units, stream-K split over up to
  // VI_WIN_SPLIT CTAs per unit (C4: 64 units of 6 key tiles; attn_tc2's KV split + combine
  // kernel measured 28 us/block)
  // With one CTA per (head, window, 128-query tile) unit fitting in one wave (C4: 16 windows x
  // 2 tiles x 4 heads = 128), units are single Q tiles and never split: no merge tail
  // (each CTA's tile-1 warps idle).
  // (VI_WIN_SPLIT > 1 or VI_WIN_PAIRS: the pair units with a stream-K split, A/B and tests)
  const char* ws = getenv("VI_WIN_SPLIT");
  const int single_units = c->win_n ? a.win_n * ((a.win_nq + 127) / 128) * a.H : 0;
  const bool single = c->win_n && single_units <= c->num_sms && !getenv("VI_WIN_PAIRS") && !(ws && atoi(ws) > 1);
  if (single) a.win_npw = (a.win_nq + 127) / 128;
  const int win_units = c->win_n ? a.win_n * a.win_npw * a.H : 0;
  if (c->win_n && win_units <= c->num_sms) {
    a.npairs = a.win_npw;
    a.units = win_units;
    a.sk_single = single ? 1 : 0;
    a.spart = c->sk_part; a.slse = c->sk_lse; a.uparts = c->sk_flag;
    a.sk_tail = 0; a.sk_tail_w = 16; a.sk_ucost = 0;
    a.sk_wfull = (long long)a.units * ntiles;
    const int split = single ? 1 : std::max(1, ws ? atoi(ws) : 2);
    const long long work = (long long)a.units * ntiles;
    const int grid = int(std::min<long long>(std::min<long long>((long long)a.units * split, work), c->num_sms));
    if (a.units > c->sk_units_cap) return c->fail(VI_E_ARG, "attention: more stream-K units than the context holds");
    PLAUNCH(VI_PROF_ATTN, launch_attn_sk2(c->tm_q, c->tm_k, c->tm_vt, a, grid, c->stream), "attention");
    return VI_OK;
  }
  if (!small && !c->win_n) {
    // persistent stream-K: one CTA per SM over (query-tile pair, head) x key tiles
    a.npairs = (a.Nq + 255) / 256;
    a.units = a.npairs * a.H;
    a.spart = c->sk_part; a.slse = c->sk_lse; a.uparts = c->sk_flag;
    const long long work = (long long)a.units * ntiles;
    // a last pair with an empty second tile (C3: 3600 = 14 x 256 + 16) skips tile 1's MMAs
    // and the dead softmax quadrants, but its key tiles still cost about a full pair's (the
    // per-tile chain QK -> softmax -> PV is the bound, not the work): VI_SK_TAIL_W = 16
    // (measured: 8 -> +46 % attention time, 10 -> +22 %)
    const int rem = a.Nq % 256;
    a.sk_tail = (rem > 0 && rem <= 128) ? 1 : 0;
    a.sk_tail_w = 16;
    if (a.sk_tail) a.sk_tail_w = sk_tail_weight();
    a.sk_ucost = sk_unit_cost();
    a.sk_wfull = (long long)(a.npairs - a.sk_tail) * a.H * ntiles;
    const int grid = int(work < c->num_sms ? work : c->num_sms);
    if (a.units > c->sk_units_cap) return c->fail(VI_E_ARG, "attention: more stream-K units than the context holds");
    PLAUNCH(VI_PROF_ATTN, launch_attn_sk2(c->tm_q, c->tm_k, c->tm_vt, a, grid, c->stream), "attention");
  } else {   // small chunks (and windows beyond one wave): fixed KV split + combine kernel
    const int units = c->win_n ? a.win_n * a.win_npw * a.H : ((a.Nq + 255) / 256) * a.H;
    choose_split(units, ntiles, &a.nsplit, &a.tiles_per_split);
    a.nsplit = (ntiles + a.tiles_per_split - 1) / a.tiles_per_split;
    PLAUNCH(VI_PROF_ATTN, launch_attn_tc2(c->tm_q, c->tm_k, c->tm_vt, a, c->stream), "attention");
    if (a.nsplit > 1) PLAUNCH(VI_PROF_ATTN, launch_attn_combine(a, c->stream), "attention combine");
  }
  return VI_OK;
}

// The rest of block l: (all-gather of the head outputs), output projection + residual,
// LN2, FFN (+ F3N fold/unfold) + residual.
static vi_status step_ffn(vi_ctx* c, int l, const float* x_in, float* x_out) {
  const int n = c->ring.cur_n, M = n * c->P, D = c->D, F = c->F;
  const int dt = c->bf16 ? 0 : 1;
  // a6: head all-gather (NCCL, in place: rank r's chunk is already at offset r * chunk)
  if (c->comm) {
    const size_t bytes = (size_t)c->tp.chunk_elems * c->es;
    uint8_t* base = static_cast<uint8_t*>(c->og);
    const int r = nccl().all_gather(base + (size_t)c->tp.rank * bytes, base, bytes, kNcclUint8, c->comm, c->stream);
    if (r != 0) {
      c->poisoned = true;
      return c->fail(VI_E_NCCL, std::string("ncclAllGather: ") + nccl().error_string(r));
    }
  }
  // window-split head sharding: the gathered parts back to token-major rows (O-proj's A)
  if (c->win_split)
    PLAUNCH(VI_PROF_ROW, launch_window_part_gather(c->og, c->o, M, c->P, c->H, c->hd, c->tp.qparts, c->tp.part_rows,
                                                   c->stream),
            "window part gather");
  // a7: output projection + residual
  Epi eo = epi_base(c, EPI_RESID, M, D, c->b_o + (size_t)l * D);
  eo.x_in = x_in; eo.x_out = x_out;
  if (c->sharded && !c->win_split) {   // A = concat_h(O_h) read head-major from the gathered buffer
    eo.a_hs = c->tp.head_rows;
    eo.a_kpb = c->hd / 64;
  }
  CUtensorMap tx_in, tx_out;
  const bool te = c->bf16 && make_tmap_out(&tx_in, x_in, true, D, M) && make_tmap_out(&tx_out, x_out, true, D, M);
  // small M: split-K partials, then one kernel for reduction + residual + LN2 (a7 + a8)
  const int ks_o = te ? splitk_plan(c, M, D, D) : 0;
  if (ks_o) {
    const vi_status r = splitk_resid(c, ks_o, (c->sharded && !c->win_split) ? c->tm_og : c->tm_o, c->tm_wo, l * D, M, D,
                                     D, eo.a_hs, eo.a_kpb, eo.bias, x_in, x_out, nullptr, c->ln2_g + (size_t)l * D,
                                     c->ln2_b + (size_t)l * D, c->h, "o gemm (split-K)");
    if (r != VI_OK) return r;
  } else if (c->bf16)
    PLAUNCH(VI_PROF_GEMM, launch_gemm_tc((c->sharded && !c->win_split) ? c->tm_og : c->tm_o, c->tm_wo, l * D, M, D, D,
                                         c->bn_o, eo, c->stream, 0,
                                         te ? &tx_out : nullptr, te ? &tx_in : nullptr),
            "o gemm");
  else
    PLAUNCH(VI_PROF_GEMM, launch_gemm_simt_f32((const float*)c->o, (const float*)c->w_o + (size_t)l * D * D, M, D, D, eo, c->stream),
            "o gemm");
  // a8: LN2
  if (!ks_o)
    PLAUNCH(VI_PROF_ROW, launch_layernorm(x_out, c->ln2_g + (size_t)l * D, c->ln2_b + (size_t)l * D, c->h, dt, M, D, c->stream), "ln2");
  // a9 / a10: FFN1 (+ F3N fold/unfold) + GELU
  const bool f3n = c->cfg.ffn_kind == VI_FFN_F3N;
  Epi e1 = epi_base(c, f3n ? EPI_STORE : EPI_GELU, M, F, c->b_1 + (size_t)l * F);
  const bool ffn1_small = c->bn_1 == 256 && ((M + 127) / 128) * ((F + 255) / 256) * 2 <= c->num_sms;
  e1.out = f3n ? c->u : c->gbuf; e1.ldo = F; e1.out_f32 = f3n ? 1 : 0;
  if (c->bf16)
    // small M (one frame): 128-column tiles, twice the CTAs of the 256-column ones
    PLAUNCH(VI_PROF_GEMM, launch_gemm_tc(c->tm_h, ffn1_small ? c->tm_w1_128 : c->tm_w1, l * F, M, F, D,
                                         ffn1_small ? 128 : c->bn_1, e1, c->stream, 0,
                                         f3n ? &c->tm_u_out : &c->tm_g_out),
            "ffn1 gemm");
  else
    PLAUNCH(VI_PROF_GEMM, launch_gemm_simt_f32((const float*)c->h, (const float*)c->w_1 + (size_t)l * F * D, M, F, D, e1, c->stream),
            "ffn1 gemm");
  if (f3n) {
    // g = GELU(unfold(fold(u))) = unfold(GELU(fold(u))): GELU once per folded cell
    PLAUNCH(VI_PROF_PATCH, launch_fold(c->u, 1, c->fold_ws, dt, n, c->gf, true, c->stream, patch_timing(c, 'f')), "f3n fold");
    PLAUNCH(VI_PROF_PATCH, launch_unfold(c->fold_ws, c->gbuf, n, c->gf, dt, c->stream, patch_timing(c, 'u')), "f3n unfold");
  }
  // a11: FFN2 + residual
  Epi e2 = epi_base(c, EPI_RESID, M, D, c->b_2 + (size_t)l * D);
  e2.x_in = x_out; e2.x_out = x_out;
  // FFN2 (K = F = 1960) on CTA-pair tiles 256 x 128 (tools/micro/gemm_micro: 16.9 vs 18.3 us)
  const bool pair2 = te;
  const int ks_2 = te ? splitk_plan(c, M, D, F) : 0;
  if (ks_2) {
    const bool ln_next = c->fuse_ln1 && l + 1 < c->L;   // the next block's LN1 in the same pass
    const vi_status r = splitk_resid(c, ks_2, c->tm_g, c->tm_w2, l * D, M, D, F, 0, 0, e2.bias, x_out, x_out, nullptr,
                                     ln_next ? c->ln1_g + (size_t)(l + 1) * D : nullptr,
                                     ln_next ? c->ln1_b + (size_t)(l + 1) * D : nullptr, ln_next ? c->h : nullptr,
                                     "ffn2 gemm (split-K)");
    if (r != VI_OK) return r;
    if (ln_next) c->h_ready = l + 1;
  } else if (c->bf16)
    PLAUNCH(VI_PROF_GEMM, launch_gemm_tc(c->tm_g, pair2 ? c->tm_w2_pair : c->tm_w2, l * D, M, D, F, pair2 ? 128 : c->bn_2, e2,
                                         c->stream, pair2 ? 1 : 0, te ? &tx_out : nullptr, te ? &tx_out : nullptr),
            "ffn2 gemm");
  else
    PLAUNCH(VI_PROF_GEMM, launch_gemm_simt_f32((const float*)c->gbuf, (const float*)c->w_2 + (size_t)l * D * F, M, D, F, e2,
                                               c->stream),
            "ffn2 gemm");
  return VI_OK;
}

static vi_status check_step(vi_ctx* c, int layer, const void* x_in, const void* x_out, const char* who) {
  if (!x_in || !x_out) return c->fail(VI_E_ARG, std::string(who) + ": NULL x");
  if (!c->have_weights) return c->fail(VI_E_PROTOCOL, std::string(who) + ": weights not set");
  if (c->next_layer < 0 || layer != c->next_layer || layer >= c->L)
    return c->fail(VI_E_PROTOCOL, std::string(who) + ": needs a push, then layers 0..L-1 in order");
  return VI_OK;
}

static void layer_done(vi_ctx* c, int layer) {
  c->attn_layer = -1;
  c->next_layer = layer + 1;
  if (c->next_layer == c->L) {
    std::lock_guard<std::mutex> lk(c->mu);
    c->ring.mark_stepped();
  }
}

extern "C" vi_status vi_memory_step_attn(vi_ctx* c, int layer, const float* x_in) {
  LIVE(c);
  DeviceGuard dg_(c->cfg.device);
  vi_status st = check_step(c, layer, x_in, x_in, "vi_memory_step_attn");
  if (st != VI_OK) return st;
  if (c->attn_layer == layer) return c->fail(VI_E_PROTOCOL, "vi_memory_step_attn: this layer's _ffn is pending");
  if ((st = step_attn(c, layer, x_in)) != VI_OK) return st;
  c->attn_layer = layer;
  return VI_OK;
}

extern "C" vi_status vi_memory_step_ffn(vi_ctx* c, int layer, const float* x_in, float* x_out) {
  LIVE(c);
  DeviceGuard dg_(c->cfg.device);
  vi_status st = check_step(c, layer, x_in, x_out, "vi_memory_step_ffn");
  if (st != VI_OK) return st;
  if (c->attn_layer != layer) return c->fail(VI_E_PROTOCOL, "vi_memory_step_ffn: needs vi_memory_step_attn of this layer");
  if ((st = step_ffn(c, layer, x_in, x_out)) != VI_OK) return st;
  layer_done(c, layer);
  return VI_OK;
}

extern "C" vi_status vi_memory_step(vi_ctx* c, int layer, const float* x_in, float* x_out) {
  LIVE(c);
  DeviceGuard dg_(c->cfg.device);
  vi_status st = check_step(c, layer, x_in, x_out, "vi_memory_step");
  if (st != VI_OK) return st;
  if (c->sharded && !c->comm)
    return c->fail(VI_E_PROTOCOL, "vi_memory_step: head-sharded context without a communicator: use "
                                  "vi_memory_step_attn / vi_tp_local_allgather / vi_memory_step_ffn");
  if (c->attn_layer >= 0) return c->fail(VI_E_PROTOCOL, "vi_memory_step: a vi_memory_step_attn is pending");
  if ((st = step_attn(c, layer, x_in)) != VI_OK) return st;
  if ((st = step_ffn(c, layer, x_in, x_out)) != VI_OK) return st;
  layer_done(c, layer);
  return VI_OK;
}

extern "C" vi_status vi_tp_local_allgather(vi_ctx* const* ctxs, int n) {
  if (!ctxs || n < 1) return VI_E_ARG;
  for (int i = 0; i < n; ++i) {
    vi_ctx* c = ctxs[i];
    LIVE(c);
  DeviceGuard dg_(c->cfg.device);
    if (!c->sharded || c->comm || c->tp.G != n || c->tp.rank != i)
      return c->fail(VI_E_CONFIG, "vi_tp_local_allgather: ctxs[r] must be rank r of a communicator-less group of n");
    if (c->tp.chunk_elems != ctxs[0]->tp.chunk_elems || c->H != ctxs[0]->H || c->hd != ctxs[0]->hd)
      return c->fail(VI_E_SHAPE, "vi_tp_local_allgather: contexts of different shapes");
    if (c->attn_layer < 0 || c->attn_layer != ctxs[0]->attn_layer)
      return c->fail(VI_E_PROTOCOL, "vi_tp_local_allgather: every rank must have run _attn of the same layer");
  }
  for (int i = 0; i < n; ++i) CK_C(ctxs[i], cudaEventRecord(ctxs[i]->ev_attn, ctxs[i]->stream), "allgather record");
  const size_t bytes = (size_t)ctxs[0]->tp.chunk_elems * ctxs[0]->es;
  for (int j = 0; j < n; ++j) {
    vi_ctx* d = ctxs[j];
    for (int i = 0; i < n; ++i) CK_C(d, cudaStreamWaitEvent(d->stream, ctxs[i]->ev_attn, 0), "allgather wait");
    for (int i = 0; i < n; ++i) {
      if (i == j) continue;
      uint8_t* dst = static_cast<uint8_t*>(d->og) + i * bytes;
      const uint8_t* src = static_cast<const uint8_t*>(ctxs[i]->og) + i * bytes;
      CK_C(d, cudaMemcpyPeerAsync(dst, d->cfg.device, src, ctxs[i]->cfg.device, bytes, d->stream), "allgather copy");
    }
    CK_C(d, cudaEventRecord(d->ev_gather, d->stream), "allgather record");
  }
  // no rank overwrites its chunk (next layer's attention) before every peer has copied it
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) CK_C(ctxs[i], cudaStreamWaitEvent(ctxs[i]->stream, ctxs[j]->ev_gather, 0), "allgather wait");
  return VI_OK;
}

extern "C" vi_status vi_soft_composite(vi_ctx* c, const void* in, int n, void* feat, int project) {
  LIVE(c);
  DeviceGuard dg_(c->cfg.device);
  if (!in || !feat || n < 1 || n > c->Tmax || (project != 0 && project != 1))
    return c->fail(VI_E_ARG, "vi_soft_composite: bad argument");
  if (project && !c->have_weights) return c->fail(VI_E_PROTOCOL, "vi_soft_composite: weights not set");
  const int dt = c->bf16 ? 0 : 1;
  const void* tok = in;
  if (project) {
    const int M = n * c->P;
    Epi e = epi_base(c, EPI_STORE, M, c->Pd, c->b_back);
    e.out = c->tokens; e.ldo = c->Pd;
    if (c->bf16) {
      // x enters the GEMM as bf16 hi + lo (K = 2D against [Wb | Wb]) and Yp leaves it in
      // fp32: the back projection adds no bf16 rounding of its own
      e.out = c->yp32; e.out_f32 = 1;
      PLAUNCH(VI_PROF_ROW, launch_split_bf16((const float*)in, c->xb, M, c->D, c->stream), "cast");
      PLAUNCH(VI_PROF_GEMM, launch_gemm_tc(c->tm_xb, c->tm_wback, 0, M, c->Pd, 2 * c->D, c->bn_back, e, c->stream, 0,
                                           &c->tm_yp_out),
              "back gemm");
    } else {
      PLAUNCH(VI_PROF_GEMM, launch_gemm_simt_f32((const float*)in, (const float*)c->w_back, M, c->Pd, c->D, e, c->stream),
             "back gemm");
    }
    tok = c->bf16 ? c->yp32 : c->tokens;
  }
  PLAUNCH(VI_PROF_PATCH, launch_fold(tok, (project && c->bf16) ? 1 : dt, feat, dt, n, c->g, false, c->stream,
                                     patch_timing(c, 'c')),
          "fold");
  return VI_OK;
}

// The device part of one step (split+embed, L blocks, back-projection+composite).
static vi_status step_body_seq(vi_ctx* c, const void* fin, int n, void* fout) {
  vi_status st;
  if ((st = vi_soft_split(c, fin, n, c->x_ws, 1)) != VI_OK) return st;
  for (int l = 0; l < c->L; ++l)
    if ((st = vi_memory_step(c, l, c->x_ws, c->x_ws)) != VI_OK) return st;
  return vi_soft_composite(c, c->x_ws, n, fout, 1);
}
static vi_status step_body(vi_ctx* c, const void* fin, int n, void* fout) {
  c->fuse_ln1 = true;     // x_ws flows from block to block untouched: LN1 may ride on a reduction
  c->h_ready = -1;
  const vi_status st = step_body_seq(c, fin, n, fout);
  c->fuse_ln1 = false;
  c->h_ready = -1;
  return st;
}

// Enqueue the device part of a step (after the push) on the ctx stream: replay of the step's
// CUDA graph, captured on first use for this (shape, ring state, buffers, weights, profiling).
static vi_status step_graph(vi_ctx* c, const void* fin, int n, void* fout) {
  vi_status st;
  const bool graphs = c->use_graphs && !g_debug_sync && c->prof_mode != 2;
  if (!graphs) return step_body(c, fin, n, fout);
  // everything a replay bakes in: shapes, ring state, buffers, weights, profiling mode
  std::vector<uint64_t> key = {uint64_t(n), uint64_t(c->ring.cur_first % c->S), c->ring.valid_mask(),
                               uint64_t(reinterpret_cast<uintptr_t>(fin)), uint64_t(reinterpret_cast<uintptr_t>(fout)),
                               uint64_t(c->prof_mode), uint64_t(c->weights_gen)};
  vi_ctx::GraphEntry* hit = nullptr;
  for (auto& g : c->graphs)
    if (g.key == key) hit = &g;
  if (!hit) {
    const int64_t l0 = c->launches;
    cudaGraph_t graph = nullptr;
    CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal), "graph capture");
    st = step_body(c, fin, n, fout);
    cudaError_t ce = cudaStreamEndCapture(c->stream, &graph);
    if (st != VI_OK) {
      if (graph) cudaGraphDestroy(graph);
      return st;
    }
    if (ce != cudaSuccess) return c->cuda_fail(ce, "graph capture end");
    cudaGraphExec_t exec = nullptr;
    ce = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ce != cudaSuccess) return c->cuda_fail(ce, "graph instantiate");
    if (c->graphs.size() >= 64) {   // evict the least recently used (64: every (ring state, buffer)
                                    // pair of a one-frame step cycling over 4 buffers stays cached)
      auto lru = std::min_element(c->graphs.begin(), c->graphs.end(),
                                  [](const vi_ctx::GraphEntry& a, const vi_ctx::GraphEntry& b) {
                                    return a.last_use < b.last_use;
                                  });
      cudaGraphExecDestroy(lru->exec);
      c->graphs.erase(lru);
    }
    c->graphs.push_back({key, exec, c->launches - l0, 0});
    c->launches = l0;
    hit = &c->graphs.back();
  } else {
    c->next_layer = c->L;               // the host-side protocol state a replay skips
    std::lock_guard<std::mutex> lk(c->mu);
    c->ring.mark_stepped();
  }
  hit->last_use = ++c->graph_clock;
  c->launches += hit->launches;
  CK(cudaGraphLaunch(hit->exec, c->stream), "graph launch");
  return VI_OK;
}

static vi_status check_run_step(vi_ctx* c, const void* feat, int n, const void* out, const char* who) {
  if (!feat || !out || n < 1 || n > c->Tmax) return c->fail(VI_E_ARG, std::string(who) + ": bad argument");
  if (!c->have_weights) return c->fail(VI_E_PROTOCOL, std::string(who) + ": weights not set");
  if (c->sharded && !c->comm)
    return c->fail(VI_E_PROTOCOL, std::string(who) + ": head-sharded context without a communicator");
  return VI_OK;
}

extern "C" vi_status vi_run_step(vi_ctx* c, const void* feat, int n, void* out, int64_t* first_id) {
  LIVE(c);
  DeviceGuard dg_(c->cfg.device);
  vi_status st = check_run_step(c, feat, n, out, "vi_run_step");
  if (st != VI_OK) return st;
  st = vi_memory_push(c, n, first_id, nullptr, nullptr);   // host bookkeeping + queued commits
  if (st != VI_OK) return st;
  const size_t fbytes = (size_t)n * c->g.H * c->g.W * c->g.C * c->es;
  const bool hin = is_host_ptr(feat), hout = is_host_ptr(out);
  const void* fin = feat;
  if (hin) {
    CK(cudaMemcpyAsync(c->feat_in, feat, fbytes, cudaMemcpyHostToDevice, c->stream), "run_step h2d");
    fin = c->feat_in;
  }
  void* fout = hout ? c->feat_out : out;
  if ((st = step_graph(c, fin, n, fout)) != VI_OK) return st;
  if (hout) {
    CK(cudaMemcpyAsync(out, c->feat_out, fbytes, cudaMemcpyDeviceToHost, c->stream), "run_step d2h");
    CK(cudaStreamSynchronize(c->stream), "run_step sync");
  }
  return VI_OK;
}

// First use of vi_run_step_async: the copy streams, staging slots and events, created into
// locals and published only when all of them exist (a failure leaves the context unchanged).
static vi_status async_init(vi_ctx* c) {
  cudaStream_t in_s = nullptr, out_s = nullptr;
  void* bufs[4] = {nullptr, nullptr, nullptr, nullptr};
  cudaEvent_t evs[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  const size_t fmap = (size_t)c->Tmax * c->g.H * c->g.W * c->g.C * c->es;
  bool ok = cudaStreamCreateWithFlags(&in_s, cudaStreamNonBlocking) == cudaSuccess &&
            cudaStreamCreateWithFlags(&out_s, cudaStreamNonBlocking) == cudaSuccess;
  for (int i = 0; i < 4 && ok; ++i) ok = cudaMalloc(&bufs[i], fmap) == cudaSuccess;
  for (int i = 0; i < 6 && ok; ++i) ok = cudaEventCreateWithFlags(&evs[i], cudaEventDisableTiming) == cudaSuccess;
  if (!ok) {
    cudaGetLastError();
    for (void* b : bufs)
      if (b) cudaFree(b);
    for (cudaEvent_t e : evs)
      if (e) cudaEventDestroy(e);
    if (in_s) cudaStreamDestroy(in_s);
    if (out_s) cudaStreamDestroy(out_s);
    return c->fail(VI_E_OOM, "vi_run_step_async: staging streams / buffers / events could not be created");
  }
  for (int k = 0; k < 2; ++k) {
    c->async_in[k] = bufs[2 * k];
    c->async_out[k] = bufs[2 * k + 1];
    c->allocs.push_back(bufs[2 * k]);
    c->allocs.push_back(bufs[2 * k + 1]);
    c->device_bytes += 2 * fmap;
    c->ev_h2d[k] = evs[3 * k];
    c->ev_done[k] = evs[3 * k + 1];
    c->ev_d2h[k] = evs[3 * k + 2];
  }
  c->io_out = out_s;
  c->io_stream = in_s;       // published last: io_stream != NULL <=> everything above exists
  return VI_OK;
}

extern "C" vi_status vi_run_step_async(vi_ctx* c, const void* feat, int n, void* out, int64_t* first_id) {
  LIVE(c);
  DeviceGuard dg_(c->cfg.device);
  vi_status st = check_run_step(c, feat, n, out, "vi_run_step_async");
  if (st != VI_OK) return st;
  if (!c->io_stream && (st = async_init(c)) != VI_OK) return st;
  // the push first: the only call here that can fail without poisoning the context, and its
  // device work (queued commits, reference moves) is on the ctx stream ahead of the step
  st = vi_memory_push(c, n, first_id, nullptr, nullptr);
  if (st != VI_OK) return st;
  const size_t fbytes = (size_t)n * c->g.H * c->g.W * c->g.C * c->es;
  const int k = c->async_slot;
  c->async_slot ^= 1;
  const bool hin = is_host_ptr(feat), hout = is_host_ptr(out);
  // io stream: this slot's input staging is free once the step that read it (two calls ago)
  // is done; copy the frames in
  const void* fin = feat;
  if (hin) {
    if (c->async_used[k]) CK(cudaStreamWaitEvent(c->io_stream, c->ev_done[k], 0), "async wait");
    CK(cudaMemcpyAsync(c->async_in[k], feat, fbytes, cudaMemcpyHostToDevice, c->io_stream), "async h2d");
    CK(cudaEventRecord(c->ev_h2d[k], c->io_stream), "async record");
    CK(cudaStreamWaitEvent(c->stream, c->ev_h2d[k], 0), "async wait");
    fin = c->async_in[k];
  }
  // compute stream: the output staging is free once its previous copy-out is done
  if (hout && c->async_used[k]) CK(cudaStreamWaitEvent(c->stream, c->ev_d2h[k], 0), "async wait");
  void* fout = hout ? c->async_out[k] : out;
  if ((st = step_graph(c, fin, n, fout)) != VI_OK) return st;
  CK(cudaEventRecord(c->ev_done[k], c->stream), "async record");
  // io stream: copy the result out while the next step computes
  if (hout) {
    CK(cudaStreamWaitEvent(c->io_out, c->ev_done[k], 0), "async wait");
    CK(cudaMemcpyAsync(out, c->async_out[k], fbytes, cudaMemcpyDeviceToHost, c->io_out), "async d2h");
    CK(cudaEventRecord(c->ev_d2h[k], c->io_out), "async record");
  }
  c->async_used[k] = true;
  return VI_OK;
}

extern "C" vi_status vi_sync(vi_ctx* c) {
  LIVE(c);
  DeviceGuard dg_(c->cfg.device);
  CK(cudaStreamSynchronize(c->stream), "vi_sync");
  if (c->io_stream) CK(cudaStreamSynchronize(c->io_stream), "vi_sync");
  if (c->io_out) CK(cudaStreamSynchronize(c->io_out), "vi_sync");
  return VI_OK;
}

extern "C" vi_status vi_profile(vi_ctx* c, int mode) {
  LIVE(c);
  DeviceGuard dg_(c->cfg.device);
  if (mode < 0 || mode > 4) return VI_E_ARG;
  c->prof_mode = mode;
  return VI_OK;
}

extern "C" vi_status vi_profile_read(vi_ctx* c, double* ms, int64_t* launches) {
  LIVE(c);
  DeviceGuard dg_(c->cfg.device);
  CK(cudaStreamSynchronize(c->stream), "profile sync");
  double acc[VI_PROF_N] = {0, 0, 0, 0};
  int64_t cnt[VI_PROF_N] = {0, 0, 0, 0};
  {  // kernels' self-timing (modes 1, 3; graph-safe): [0] attention, [1] GEMMs, [2] patch kernels
    KernelTiming kt[3];
    CK(cudaMemcpy(kt, c->attn_timing, sizeof(kt), cudaMemcpyDeviceToHost), "profile read");
    acc[VI_PROF_ATTN] += double(kt[0].total_ns) * 1e-6;
    cnt[VI_PROF_ATTN] += int64_t(kt[0].launches);
    acc[VI_PROF_GEMM] += double(kt[1].total_ns) * 1e-6;
    cnt[VI_PROF_GEMM] += int64_t(kt[1].launches);
    acc[VI_PROF_PATCH] += double(kt[2].total_ns) * 1e-6;
    cnt[VI_PROF_PATCH] += int64_t(kt[2].launches);
    std::memset(kt, 0, sizeof(kt));
    kt[0].tmin = kt[1].tmin = kt[2].tmin = ~0ull;
    CK(cudaMemcpy(c->attn_timing, kt, sizeof(kt), cudaMemcpyHostToDevice), "profile reset");
  }
  for (auto& r : c->prof_recs) {
    float t = 0.f;
    if (cudaEventElapsedTime(&t, r.a, r.b) == cudaSuccess) {
      acc[r.cat] += t;
      cnt[r.cat] += 1;
    } else {
      cudaGetLastError();
    }
    c->ev_pool.push_back(r.a);
    c->ev_pool.push_back(r.b);
  }
  c->prof_recs.clear();
  for (int i = 0; i < VI_PROF_N; ++i) {
    if (ms) ms[i] = acc[i];
    if (launches) launches[i] = cnt[i];
  }
  return VI_OK;
}

extern "C" const char* vi_last_error(const vi_ctx* c) { return c ? c->err.c_str() : "null context"; }
extern "C" int64_t vi_kernel_launches(const vi_ctx* c) { return c ? c->launches : 0; }
extern "C" vi_status vi_memory_footprint(const vi_ctx* c, int64_t* slab_bytes, int64_t* total_bytes) {
  if (!c) return VI_E_ARG;
  if (slab_bytes) *slab_bytes = int64_t(c->L) * c->ST * c->P * c->Dl * c->es + int64_t(c->L) * c->Dl * c->vt_ld * c->es;
  if (total_bytes) *total_bytes = int64_t(c->device_bytes);
  return VI_OK;
}
extern "C" int vi_num_slots(const vi_ctx* c) { return c ? c->ST : 0; }
extern "C" int64_t vi_refined_watermark(vi_ctx* c) {
  if (!c) return -1;
  std::lock_guard<std::mutex> lk(c->mu);
  return c->ring.t;
}
extern "C" void* vi_stream(const vi_ctx* c) { return c ? (void*)c->stream : nullptr; }
extern "C" const char* vi_version(void) { return "vi-memstep 0.1 (sm_100a)"; }

extern "C" vi_status vi_debug_read(vi_ctx* c, int what, int layer, int slot, void* dst, size_t bytes) {
  LIVE(c);
  DeviceGuard dg_(c->cfg.device);
  if (!dst) return VI_E_ARG;
  const int n = std::max(c->ring.cur_n, 1);
  const size_t es = c->es, rows = (size_t)n * c->P, D = c->D, Dl = c->Dl, SP = (size_t)c->ST * c->P;
  const void* src = nullptr;
  size_t need = 0;
  if (c->win_n && (what == VI_DBG_Q || what == VI_DBG_K || what == VI_DBG_V))
    return c->fail(VI_E_CONFIG, "vi_debug_read: Q / K / V are window-major under window attention");
  switch (what) {
    case VI_DBG_TOKENS: src = c->tokens; need = rows * c->Pd * es; break;
    case VI_DBG_H: src = c->h; need = rows * D * es; break;
    case VI_DBG_Q: src = c->q; need = rows * Dl * es; break;
    case VI_DBG_O: src = c->o; need = rows * D * es; break;
    case VI_DBG_U:
      if (c->cfg.ffn_kind != VI_FFN_F3N) return c->fail(VI_E_CONFIG, "vi_debug_read: u exists for F3N only");
      src = c->u; need = rows * c->F * 4; break;
    case VI_DBG_G: src = c->gbuf; need = rows * c->F * es; break;
    case VI_DBG_K:
    case VI_DBG_V: need = (size_t)c->P * Dl * es; break;
    default: return VI_E_ARG;
  }
  if (bytes != need) return c->fail(VI_E_SHAPE, "vi_debug_read: byte count mismatch");
  if ((what == VI_DBG_K || what == VI_DBG_V) && (layer < 0 || layer >= c->L || slot < 0 || slot >= c->ST))
    return VI_E_ARG;
  CK(cudaStreamSynchronize(c->stream), "debug sync");
  if (what == VI_DBG_K) {
    src = static_cast<const uint8_t*>(c->kslab) + ((size_t)layer * SP + (size_t)slot * c->P) * Dl * es;
    CK(cudaMemcpy(dst, src, need, cudaMemcpyDefault), "debug copy");
  } else if (what == VI_DBG_V) {
    // Vt [Dl][S*P] columns slot*P.. -> [P][Dl]
    std::vector<uint8_t> tmp(need);
    const uint8_t* base =
        static_cast<const uint8_t*>(c->vtslab) + ((size_t)layer * Dl * c->vt_ld + (size_t)slot * c->P) * es;
    CK(cudaMemcpy2D(tmp.data(), c->P * es, base, (size_t)c->vt_ld * es, c->P * es, Dl, cudaMemcpyDeviceToHost),
       "debug copy V");
    std::vector<uint8_t> tr(need);
    for (size_t d = 0; d < Dl; ++d)
      for (int p = 0; p < c->P; ++p) std::memcpy(&tr[((size_t)p * Dl + d) * es], &tmp[(d * c->P + p) * es], es);
    CK(cudaMemcpy(dst, tr.data(), need, cudaMemcpyDefault), "debug copy V");
  } else if (what == VI_DBG_O && c->sharded && !c->win_split) {
    // gathered head-major [H][head_rows][hd] -> [rows][D]
    const size_t hr = c->tp.head_rows, hd = c->hd;
    std::vector<uint8_t> tmp((size_t)c->H * hr * hd * es), out(need);
    CK(cudaMemcpy(tmp.data(), c->og, tmp.size(), cudaMemcpyDeviceToHost), "debug copy O");
    for (int h = 0; h < c->H; ++h)
      for (size_t r = 0; r < rows; ++r)
        std::memcpy(&out[(r * D + h * hd) * es], &tmp[((size_t)h * hr + r) * hd * es], hd * es);
    CK(cudaMemcpy(dst, out.data(), need, cudaMemcpyDefault), "debug copy O");
  } else {
    CK(cudaMemcpy(dst, src, need, cudaMemcpyDefault), "debug copy");
  }
  return VI_OK;
}
