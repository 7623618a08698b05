/*
 * vi.h -- C-ABI of the B200 memory-step engine (libvi.so).
 *
 * What it computes: the per-frame memory step of an online video-inpainting
 * transformer, the "Memory" model of arXiv 2403.16161 (§3.4, Eq. 3,
 * P:119-132) and the refined-memory hand-off of the "Refined" model (§3.5, Eq. 4,
 * P:142-154).  Citations: P:n = /root/reference/PAPER.md line n.  Readings Qn are
 * listed in DESIGN.md ("Readings of the paper").
 *
 * One step of n new frames (1 <= n <= max_new_frames) is, in this order:
 *   1. vi_memory_push(n)               frame ids f..f+n-1 enter the ring memory,
 *                                      frames older than f-M leave it (Eq. 3 span s=M);
 *   2. vi_soft_split(project=1)        overlapping unfold + patch embedding;
 *   3. vi_memory_step(l), l = 0..L-1   block l: queries = the new frames only,
 *                                      keys/values = the new frames + the memory,
 *                                      the new frames' K/V written into the memory of
 *                                      block l ("after each transformer, the new result is
 *                                      saved for later", Fig. 2);
 *   4. vi_soft_composite(project=1)    back-projection + overlapping fold with
 *                                      overlap-count normalisation ("blended").
 * vi_run_step() does 1-4 in one call.
 *
 * Conventions
 *   - Status: 0 = VI_OK, 1 = VI_NOT_RESIDENT (informational, nothing done), < 0 error.
 *   - Arguments, shapes and protocol are validated synchronously BEFORE any side
 *     effect: a call that returns an error changed nothing.
 *   - Device work is enqueued on the context's CUDA stream; calls return after
 *     enqueue (vi_sync waits).  CUDA errors are sticky: the context is poisoned and
 *     every later call returns VI_E_CUDA (vi_last_error tells why).
 *   - Buffers ("device" below) are caller-owned, contiguous, 16-byte aligned device
 *     pointers unless a function says host pointers are accepted.  The context owns
 *     its weights, K/V memory slabs and workspaces; nothing returned must be freed
 *     except the context itself (vi_destroy).
 *   - Element type "ctx dtype" = bf16 (dtype 0, tensor-core path) or fp32 (dtype 1,
 *     SIMT path).  The residual stream x is always fp32.
 *   - Layouts: feature maps [n][H][W][C] channels-last; tokens [n][P][k*k*C] with the
 *     patch vector ordered (ky, kx, c) and tokens row-major (oy, ox) (reading Q6);
 *     x [n][P][D]; weights in nn.Linear layout [out][in].
 *   - Not thread-safe per context, except vi_refine_commit, which may be called from
 *     another (refiner) thread.
 */
#ifndef VI_H_
#define VI_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t vi_status;
#define VI_OK            0
#define VI_NOT_RESIDENT  1   /* evict/commit of a frame no longer in memory: no-op */
#define VI_E_ARG        -1   /* bad argument value (NULL, negative id, n out of range) */
#define VI_E_SHAPE      -2   /* inconsistent shapes */
#define VI_E_CONFIG     -3   /* unsupported configuration */
#define VI_E_PROTOCOL   -4   /* call out of protocol order (see each function) */
#define VI_E_CUDA       -5   /* CUDA failure (sticky) or no usable sm_100 device */
#define VI_E_OOM        -6   /* device allocation failed */
#define VI_E_NCCL       -7   /* collective failure */

#define VI_DTYPE_BF16 0
#define VI_DTYPE_FP32 1
#define VI_FFN_MLP    0     /* FFN1 -> GELU -> FFN2 */
#define VI_FFN_F3N    1     /* FuseFormer Fusion-FFN: FFN1 -> fold/count -> unfold -> GELU -> FFN2 */

typedef struct vi_ctx vi_ctx;

typedef struct vi_config {
  int layers;            /* L transformer blocks ("8 consecutive transformer blocks") */
  int heads;             /* H attention heads */
  int d_model;           /* D hidden width; head dim d = D/H (16..128, multiple of 16 on bf16) */
  int tokens_per_frame;  /* P; must equal oh*ow of the split geometry below */
  int mem_frames;        /* M = memory span s of Eq. 3 (frames f-M..f-1 are attended) */
  int max_new_frames;    /* T_max frames per step; ring slots S = M + T_max <= 64 */
  int feat_h, feat_w, feat_c;   /* feature map H x W x C */
  int kh, kw, sh, sw, ph, pw;   /* soft split kernel / stride / symmetric zero padding */
  int ffn_hidden;        /* F; F3N requires F % (kh*kw) == 0 */
  int ffn_kind;          /* VI_FFN_MLP or VI_FFN_F3N */
  int dtype;             /* VI_DTYPE_BF16 or VI_DTYPE_FP32 */
  int pos_embed;         /* 0 none, 1 additive [P][D] table given in vi_weights.pos */
  int device;            /* CUDA device ordinal */
  void* stream;          /* cudaStream_t to enqueue on (NULL = the context creates one) */
  /* Head sharding (BASELINE north_star "attention heads are split across
   * GPUs and the head outputs are all-gathered with NCCL over NVLink before the output
   * projection").  tp_size G = 1 (or 0): unsharded.  G > 1: this context is rank
   * tp_rank of G; see vi_tp_layout for which heads / query rows it owns.  Sharded per
   * rank: the Q/K/V projection of its heads, its K/V memory (memory per GPU / G when
   * G <= H) and its attention; replicated: everything else (bitwise identical on every
   * rank).  bf16 path only.
   *   nccl_id != NULL: 128-byte ncclUniqueId (vi_tp_unique_id on one rank, broadcast by
   *     the caller); vi_create_ex joins an NCCL communicator of G ranks (collective: all
   *     ranks must call it) and vi_memory_step all-gathers the head outputs itself.
   *     G = 1 with an id runs the sharded code path over a 1-rank communicator.
   *   nccl_id == NULL and G > 1: no communicator; the caller drives the exchange with
   *     vi_memory_step_attn / vi_tp_local_allgather / vi_memory_step_ffn (several
   *     contexts of one process, on one or several GPUs). */
  int tp_size, tp_rank;
  const void* nccl_id;
  /* Priority of the stream the context creates (stream == NULL): CUDA convention, lower
   * = higher priority (cudaDeviceGetStreamPriorityRange); 0 = default.  The Refined
   * dual-model run gives the online context the high priority and the refiner 0. */
  int stream_priority;
  /* Reference frames, Eq. 3's M_{1,r}^{f-1}: with ref_rate r > 0, a frame whose
   * id is a multiple of r stays in the memory after it leaves the span, in one of
   * max_ref_frames reference slots (its K/V move there at the push; the oldest reference
   * leaves when the slots are full; reading Q12).  0 = span only.  Slots in total:
   * mem_frames + max_new_frames + max_ref_frames <= 64 (vi_num_slots). */
  int ref_rate, max_ref_frames;
  /* Window attention (E2FGVI-shaped, BASELINE configs[3]): a query sees only the keys of
   * its own win_h x win_w token window (non-overlapping, tiling the token grid), in every
   * frame of the memory and the chunk (reference frames included).  0 = global attention.
   * bf16 path; head sharding (tp_size > heads: the tp_size/heads ranks of a head split its
   * windows by window rows; they must divide the window rows); no refine commits or memory reads (the
   * memory is window-major). */
  int win_h, win_w;
  /* Refined memory M-bar of Eq. 4 (SPEC select_refined S:467-475; reading Q22):
   * with refined_mem = 1 the memory also keeps the refining inpainter's results for frames
   * that have left the online span: the frames t-s'..t (refined_span s' >= 0; t = the newest
   * frame a refine commit has been applied for, the watermark) in s'+1 refined-span slots,
   * and, with refined_rate r' > 0, the max_refined_refs newest refined frames whose id is a
   * multiple of r' (refined references; the oldest leaves first).  The online span M keeps
   * its own frames (an online frame with a refined entry holds it in its online slot:
   * refined wins).  Slots in total: mem_frames + max_new_frames + max_ref_frames
   * + (s'+1) + max_refined_refs <= 64.  0 = off: commits only overwrite online frames. */
  int refined_mem, refined_span, refined_rate, max_refined_refs;
} vi_config;

/* Weights, host fp32 pointers in nn.Linear layout (y = x W^T + b); converted to the
 * ctx dtype (round-to-nearest-even) and copied into ctx-owned device buffers.
 * Biases and LayerNorm parameters stay fp32 on the device. */
typedef struct vi_weights {
  const float* embed_w;  /* [D][kh*kw*C] */
  const float* embed_b;  /* [D] */
  const float* pos;      /* [P][D] or NULL (only read when pos_embed = 1) */
  const float* ln1_g;    /* [L][D] */
  const float* ln1_b;    /* [L][D] */
  const float* wqkv;     /* [L][3D][D]  rows 0..D-1 = Wq, D..2D-1 = Wk, 2D..3D-1 = Wv */
  const float* bqkv;     /* [L][3D] */
  const float* wo;       /* [L][D][D] */
  const float* bo;       /* [L][D] */
  const float* ln2_g;    /* [L][D] */
  const float* ln2_b;    /* [L][D] */
  const float* w1;       /* [L][F][D] */
  const float* b1;       /* [L][F] */
  const float* w2;       /* [L][D][F] */
  const float* b2;       /* [L][D] */
  const float* back_w;   /* [kh*kw*C][D] */
  const float* back_b;   /* [kh*kw*C] */
} vi_weights;

/* Fill *cfg with the FuseFormer-shaped defaults (BASELINE.json configs[2]): L=8, H=4,
 * D=512, P=720, M=10, T_max=5, 60x108x128 map, 7x7 s3 p3, F3N 1960, bf16, device 0. */
vi_status vi_config_default(vi_config* cfg);

/* Create a context: the short form of BASELINE.json's north_star
 * (vi_create(layers, heads, d_model, tokens_per_frame, mem_frames)); every other field
 * takes vi_config_default's value.  tokens_per_frame must match the default geometry
 * (720).  VI_E_CUDA if no sm_100 device is present.  *out is NULL on error. */
vi_status vi_create(vi_ctx** out, int layers, int heads, int d_model, int tokens_per_frame,
                    int mem_frames);
vi_status vi_create_ex(vi_ctx** out, const vi_config* cfg);
vi_status vi_destroy(vi_ctx* ctx);

/* Upload weights (see vi_weights).  Must precede any compute call (else VI_E_PROTOCOL).
 * Synchronous: the host arrays may be freed on return. */
vi_status vi_set_weights(vi_ctx* ctx, const vi_weights* w);

/* Ring memory, push: frames f..f+n-1 (f = next id, ids are consecutive from 0) enter
 * the memory at slots id mod S; resident frames with id < f-M leave it (Eq. 3 span,
 * P:127-130; "removing information from ancient frames"), reported in
 * evicted[0..*n_evicted) (capacity S, may be NULL).  Refine commits queued since the
 * last push are applied now, for frames still resident (reading Q13).
 * VI_E_ARG if n < 1 or n > max_new_frames.  first_id may be NULL. */
vi_status vi_memory_push(vi_ctx* ctx, int n, int64_t* first_id, int64_t* evicted, int* n_evicted);

/* Explicit eviction of a past frame.  VI_E_PROTOCOL for a future frame or a frame of
 * the current chunk whose step has not finished; VI_NOT_RESIDENT if already gone. */
vi_status vi_memory_evict(vi_ctx* ctx, int64_t frame_id);

/* Soft split of n feature maps feat [n][H][W][C] (device, ctx dtype).
 * project = 0: out = raw tokens [n][P][kh*kw*C] (ctx dtype), any 1 <= n <= T_max;
 * project = 1: out = x0 [n][P][D] fp32 = tokens We^T + be (+pos).  Bit-exact copies
 * for project = 0 (padding positions are 0). */
vi_status vi_soft_split(vi_ctx* ctx, const void* feat, int n, void* out, int project);

/* Block `layer` of the memory step for the chunk pushed last (n frames):
 *   h = LN1(x); Q,K,V = h Wqkv^T + bqkv; K,V rows -> memory slab of block `layer`;
 *   O = softmax(Q K^T / sqrt(d)) V over the keys of every valid slot (the chunk +
 *   resident frames f-M..f-1), per head; x += O Wo^T + bo; x += FFN(LN2(x)).
 * x_in / x_out: device fp32 [n][P][D]; x_in == x_out allowed.
 * VI_E_PROTOCOL unless called after a push with layer = 0, 1, ..., L-1 in order. */
vi_status vi_memory_step(vi_ctx* ctx, int layer, const float* x_in, float* x_out);

/* The two halves of vi_memory_step for head-sharded contexts driven without a
 * communicator (tp_size > 1, nccl_id == NULL); any context may use them.
 *   _attn: LN1, Q/K/V projection of the rank's heads, memory write, attention of the
 *          rank's (heads, query rows) into its chunk of the gathered head-output buffer;
 *   _ffn : (NCCL all-gather of that buffer if the ctx has a communicator), output
 *          projection + residual, LN2, FFN + residual.
 * vi_memory_step(l) == _attn(l) then _ffn(l).  VI_E_PROTOCOL out of that order. */
vi_status vi_memory_step_attn(vi_ctx* ctx, int layer, const float* x_in);
vi_status vi_memory_step_ffn(vi_ctx* ctx, int layer, const float* x_in, float* x_out);

/* Partition of the attention over G ranks (CUDA-free, the same function every context
 * uses).  G <= H: G must divide H; rank r owns heads [r*H/G, (r+1)*H/G), every query
 * row.  G > H: G must be a multiple of H; q = G/H query parts; rank r owns head r/q and
 * query rows [(r%q)*Nh, min((r%q+1)*Nh, Nq)), Nh = ceil(T_max*P/q), of the chunk of
 * Nq = n*P queries.  The gathered head outputs are head-major [H][q*Nh][d] (bf16);
 * rank r contributes elements [r*chunk, (r+1)*chunk), chunk = (H*q*Nh*d)/G.
 * Outputs may be NULL.  VI_E_CONFIG for an unsupported (H, G). */
vi_status vi_tp_layout(int heads, int head_dim, int rows_max, int tp_size, int tp_rank,
                       int* head0, int* nheads, int* qparts, int* row0, int* rows_per_part,
                       int64_t* chunk_elems);
/* ncclGetUniqueId (NCCL loaded at run time): out = 128 bytes.  VI_E_NCCL if NCCL is
 * unavailable. */
vi_status vi_tp_unique_id(void* out128);
/* All-gather of the head outputs among the G contexts of one process (tp_size = G,
 * ctxs[r] = rank r, no communicator; same or different devices): each rank's chunk is
 * copied into every other rank's buffer (device-to-device / peer copies), ordered after
 * every rank's _attn and before any rank's next launch.  Call between _attn and _ffn. */
vi_status vi_tp_local_allgather(vi_ctx* const* ctxs, int n);

/* Soft composite of n frames into feat [n][H][W][C] (device, ctx dtype).
 * project = 0: in = raw tokens [n][P][kh*kw*C] (ctx dtype);
 * project = 1: in = x [n][P][D] fp32, back-projected with back_w / back_b first.
 * out[y][x][c] = sum of the patch entries landing on (y,x) / cover count (IEEE div). */
vi_status vi_soft_composite(vi_ctx* ctx, const void* in, int n, void* feat, int project);

/* Refine commit (Eq. 4's refined memory M-bar): the refined memory entries of a
 * past frame for every block, k, v = [L][P][D] (host or device, ctx dtype; a head-sharded
 * context keeps only its heads' columns).  Queued and applied at the next vi_memory_push,
 * so a frame is never torn across blocks; a later commit for the same frame replaces an
 * earlier one.  A frame still resident is overwritten in place (refined wins); with
 * vi_config.refined_mem a frame that has left the online span lands in the refined memory
 * if Eq. 4 selects it at that push (within s' of the watermark, or a refined reference),
 * else it is dropped.  The payload is copied before return (buffers may be reused).
 * Thread-safe w.r.t. the context's other calls.  VI_E_PROTOCOL for a future frame or the
 * current chunk before its step finished; VI_NOT_RESIDENT if it can no longer be used. */
vi_status vi_refine_commit(vi_ctx* ctx, int64_t frame_id, const void* k, const void* v);

/* Read the memory entries of a resident past frame for every block into k, v =
 * [L][P][Dl] (host or device, ctx dtype; Dl = D unless head-sharded): the refiner side of
 * Eq. 4's hand-off -- a refining context's K/V of a frame, committed into the
 * online context with vi_refine_commit.  Synchronous: returns once the copies landed.
 * VI_E_PROTOCOL for a future frame or the current chunk before its step finished;
 * VI_NOT_RESIDENT if the frame left the memory. */
vi_status vi_memory_read(vi_ctx* ctx, int64_t frame_id, void* k, void* v);

/* Eq. 4's watermark t of a context with refined memory (-1: no refined frame yet). */
int64_t vi_refined_watermark(vi_ctx* ctx);

/* Host snapshot of the ring: slot_id[N] (-1 = empty), refined[N] (0/1), N = vi_num_slots
 * (the S = mem_frames + max_new_frames span slots, then the reference slots, then the refined
 * span and refined reference slots of Eq. 4), valid bitmask
 * (bit s = slot s holds a resident frame).  Any pointer may be NULL. */
vi_status vi_memory_state(vi_ctx* ctx, int64_t* slot_id, uint8_t* refined, uint64_t* valid_mask);

/* One whole step: push(n) + split(project=1) + L blocks + composite(project=1).
 * feat / out may be HOST or device pointers ([n][H][W][C], ctx dtype); host buffers
 * are staged through ctx-owned device buffers on the ctx stream (the call then
 * returns after the output has landed in host memory). */
vi_status vi_run_step(vi_ctx* ctx, const void* feat, int n, void* out, int64_t* first_id);

/* vi_run_step, pipelined for live streams: returns after enqueue.  Host inputs are copied in
 * and results copied out on two copy streams (in, out) through two device staging slots, so the
 * copies of one step overlap the compute of the previous / next one.  The host buffers
 * must stay valid (and out unread) until a later vi_sync; consecutive calls may reuse a
 * buffer only after vi_sync.  Device buffers work as in vi_run_step (no copies). */
vi_status vi_run_step_async(vi_ctx* ctx, const void* feat, int n, void* out, int64_t* first_id);

/* Wait for all work enqueued on the context's streams. */
vi_status vi_sync(vi_ctx* ctx);
/* Last error message of this context (static storage inside the ctx; never NULL). */
const char* vi_last_error(const vi_ctx* ctx);
/* Number of kernels this context has launched so far (test / bench evidence). */
int64_t vi_kernel_launches(const vi_ctx* ctx);
/* Device memory of the context (Table 3 analogue): slab_bytes = the K and V
 * memory of all blocks (2 L S P Dl elements, V rows padded to vt_ld); total_bytes = every
 * device buffer the context owns (weights, memory, workspaces).  Either may be NULL. */
vi_status vi_memory_footprint(const vi_ctx* ctx, int64_t* slab_bytes, int64_t* total_bytes);
/* Ring slot count (span + reference slots) and the ctx stream (cudaStream_t). */
int vi_num_slots(const vi_ctx* ctx);
void* vi_stream(const vi_ctx* ctx);

/* Device-side timing of the context's own kernels with CUDA events on its stream.
 * mode 0 = off, 1 = memory attention only (kernel self-timing, graph-safe),
 * 2 = every category (CUDA events; eager launches), 3 = attention, GEMMs and the patch
 * kernels of the fixed 7x7 / stride-3 geometry (kernel self-timing inside the step graph),
 * 4 = as 1 but the attention kernel alone (the split-merge kernel that follows it untimed).
 * Modes 1 and 3 time the attention as its kernel's window plus the split-merge kernel's.
 * vi_profile_read waits for the stream, then returns per category
 * the summed milliseconds and the number of timed launches and resets the counters.
 * Categories: VI_PROF_ATTN, VI_PROF_GEMM (all tensor-core / SIMT GEMMs),
 * VI_PROF_PATCH (soft split / composite / F3N fold-unfold), VI_PROF_ROW (LN, casts). */
#define VI_PROF_ATTN  0
#define VI_PROF_GEMM  1
#define VI_PROF_PATCH 2
#define VI_PROF_ROW   3
#define VI_PROF_N     4
vi_status vi_profile(vi_ctx* ctx, int mode);
vi_status vi_profile_read(vi_ctx* ctx, double* ms /*[VI_PROF_N]*/, int64_t* launches /*[VI_PROF_N]*/);

/* Test hook: copy an internal buffer to dst (host or device), `bytes` must match.
 *   VI_DBG_TOKENS  raw split tokens of the last split       [n][P][kh*kw*C] ctx dtype
 *   VI_DBG_H       LN output last written                    [n][P][D] ctx dtype
 *   VI_DBG_Q       queries of the last block                 [n][P][Dl] ctx dtype
 *   VI_DBG_O       attention output of the last block        [n][P][D] ctx dtype
 *                  (head-sharded: the gathered outputs, after _ffn or an all-gather)
 *   VI_DBG_U       FFN1 output of the last block (F3N only)  [n][P][F] fp32
 *   VI_DBG_G       GELU(F3N(u)) of the last block            [n][P][F] ctx dtype
 *   VI_DBG_K, VI_DBG_V   memory rows of (layer, slot)        [P][Dl] ctx dtype
 * `n` is the chunk size of the last push; Dl = D (unsharded) or the rank's heads x d. */
#define VI_DBG_TOKENS 0
#define VI_DBG_H      1
#define VI_DBG_Q      2
#define VI_DBG_O      3
#define VI_DBG_U      4
#define VI_DBG_G      5
#define VI_DBG_K      6
#define VI_DBG_V      7
vi_status vi_debug_read(vi_ctx* ctx, int what, int layer, int slot, void* dst, size_t bytes);

/* ---- Ring bookkeeping alone (CUDA-free; the same code every context uses) ---------
 * For tests of the integer bookkeeping on machines without a GPU. */
typedef struct vi_ring vi_ring;
vi_status vi_ring_create(vi_ring** out, int mem_frames, int max_new_frames);
/* With reference frames (see vi_config.ref_rate / max_ref_frames). */
vi_status vi_ring_create_ex(vi_ring** out, int mem_frames, int max_new_frames, int ref_rate,
                            int max_ref_frames);
/* With Eq. 4's refined memory (see vi_config.refined_mem; refined_mem = 1 implied). */
vi_status vi_ring_create_refined(vi_ring** out, int mem_frames, int max_new_frames, int ref_rate,
                                 int max_ref_frames, int refined_span, int refined_rate,
                                 int max_refined_refs);
/* Eq. 4's watermark t: the newest frame id a refine commit has been applied for (-1: none). */
int64_t vi_ring_watermark(const vi_ring* r);
vi_status vi_ring_destroy(vi_ring* r);
vi_status vi_ring_push(vi_ring* r, int n, int64_t* first_id, int64_t* evicted, int* n_evicted);
vi_status vi_ring_evict(vi_ring* r, int64_t frame_id);
vi_status vi_ring_commit(vi_ring* r, int64_t frame_id);     /* bookkeeping of a commit only */
vi_status vi_ring_mark_stepped(vi_ring* r);                  /* the chunk went through all blocks */
vi_status vi_ring_state(const vi_ring* r, int64_t* slot_id, uint8_t* refined, uint64_t* valid_mask);

/* Library version string. */
const char* vi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* VI_H_ */
