// GEMM epilogues of the memory step.
// C[m][n] = sum_k A[m][k] * W[n][k]  (fp32 accumulate), then one of:
//   EPI_STORE   out[m][n] = C + bias[n] (+ pos[m % P][n])        -> T_out (bf16 or fp32)
//   EPI_GELU    out[m][n] = GELU_erf(C + bias[n])                -> T_out
//   EPI_RESID   x_out[m][n] = x_in[m][n] + C + bias[n]           (fp32 residual stream)
//   EPI_QKV     n <  D : Q[m][n] = C + b
//               n < 2D : K slab row (slot(t)*P + p), col n-D     (the memory write)
//               else   : Vt slab [D][vt_ld] column (slot(t)*P + p) (V stored transposed)
//               with m = t*P + p, slot(t) = (first_slot + t) % S.
#pragma once
#include "common.cuh"

namespace vi {

enum EpiKind : int { EPI_STORE = 0, EPI_GELU = 1, EPI_RESID = 2, EPI_QKV = 3, EPI_NONE = 4 };

struct Epi {
  int kind;
  int M, N;
  const float* bias;      // [N]
  void* out;              // EPI_STORE / EPI_GELU
  int ldo;
  int out_f32;            // EPI_STORE: 1 = write fp32 (the residual stream x0), 0 = ctx dtype
  const float* pos;       // EPI_STORE optional, [P][N]
  int P;
  const float* x_in;      // EPI_RESID
  float* x_out;
  int D;                  // EPI_QKV
  void* q;                // [M][D]
  void* kslab;            // [S*P][D] (this layer)
  void* vtslab;           // [D][S*P] (this layer)
  int first_slot, S;
  int vt_ld;              // row pitch (elements) of the Vt slab, >= S*P, multiple of 64
  unsigned long long* timing;  // KernelTiming of the GEMM category (profile mode 1) or NULL
  // A operand stored head-major (head-sharded output projection, tp.h): a_hs > 0 means
  // A[m][k] = Amap row (k / (64 * a_kpb)) * a_hs + m, column k % (64 * a_kpb)
  int a_hs, a_kpb;
  // EPI_QKV with window attention (win_pad > 0): token p = (oy, ox) of frame t belongs to
  // window w = (oy / win_h) * win_cols + ox / win_w at index i = (oy % win_h) * win_w + ox % win_w;
  // Q goes to row w * win_qstride + t * win_pad + i, K / Vt to row / column
  // w * win_kstride + slot * win_pad + i (window-major memory, pad rows never written)
  int win_pad, win_h, win_w, win_cols, ow, win_qstride, win_kstride;
  // EPI_QKV through the TMA-store epilogue: rows of this layer's block in the K map (l * S * P)
  // and in the Vt map (l * D)
  int qkv_krow0, qkv_vrow0;
  // split-K (small M: too few output tiles for the SMs): ksplit > 1 runs every tile as ksplit
  // work items over consecutive k-block ranges, each storing its raw fp32 partial (EPI_STORE,
  // out_f32, no bias) at rows split * kpad_rows + m of the workspace; splitk_reduce_kernel then
  // sums the partials in split order and applies the real epilogue (deterministic)
  int ksplit, kpad_rows;
};

// QKV destinations of row m (token p of chunk frame t): Q row and memory (K row / Vt column)
__device__ __forceinline__ void qkv_rows(const Epi& e, int m, size_t& qrow, size_t& krow) {
  const int t = m / e.P, p = m - t * e.P;
  const int slot = (e.first_slot + t) % e.S;
  if (e.win_pad) {
    const int oy = p / e.ow, ox = p - oy * e.ow;
    const int w = (oy / e.win_h) * e.win_cols + ox / e.win_w;
    const int i = (oy % e.win_h) * e.win_w + ox % e.win_w;
    qrow = (size_t)w * e.win_qstride + (size_t)t * e.win_pad + i;
    krow = (size_t)w * e.win_kstride + (size_t)slot * e.win_pad + i;
  } else {
    qrow = (size_t)m;
    krow = (size_t)slot * e.P + p;
  }
}

template <typename T>
__device__ __forceinline__ void epi_one(const Epi& e, int m, int n, float acc) {
  float v = acc + (e.bias ? e.bias[n] : 0.f);
  switch (e.kind) {
    case EPI_STORE:
      if (e.pos) v += e.pos[(size_t)(m % e.P) * e.N + n];
      if (e.out_f32)
        reinterpret_cast<float*>(e.out)[(size_t)m * e.ldo + n] = v;
      else
        reinterpret_cast<T*>(e.out)[(size_t)m * e.ldo + n] = from_f<T>(v);
      break;
    case EPI_GELU:
      reinterpret_cast<T*>(e.out)[(size_t)m * e.ldo + n] = from_f<T>(gelu_erf(v));
      break;
    case EPI_RESID:
      e.x_out[(size_t)m * e.N + n] = e.x_in[(size_t)m * e.N + n] + v;
      break;
    default: {
      size_t qrow, row;
      qkv_rows(e, m, qrow, row);
      if (n < e.D) {
        reinterpret_cast<T*>(e.q)[qrow * e.D + n] = from_f<T>(v);
      } else if (n < 2 * e.D) {
        reinterpret_cast<T*>(e.kslab)[row * e.D + (n - e.D)] = from_f<T>(v);
      } else {
        reinterpret_cast<T*>(e.vtslab)[(size_t)(n - 2 * e.D) * (size_t)e.vt_ld + row] = from_f<T>(v);
      }
    }
  }
}

// 32 consecutive columns n0..n0+31 of row m (tensor-core epilogue; one thread per row).
// bias_s: the bias of these columns staged in shared memory (broadcast reads) or NULL;
// xin: x_in[m][n0..n0+31] already loaded (EPI_RESID; issued before the TMEM load wait).
__device__ __forceinline__ void epi_row32_bf16(const Epi& e, int m, int n0, float* v, const float* bias_s,
                                               const float4* xin) {
  if (m >= e.M || e.kind == EPI_NONE) return;
  if (n0 + 32 > e.N) {                        // ragged N tail: element-wise, still in registers
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (n0 + i < e.N) epi_one<bf16>(e, m, n0 + i, v[i]);
    return;
  }
  if (bias_s) {
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] += bias_s[i];
  }
  switch (e.kind) {
    case EPI_STORE:
    case EPI_GELU: {
      if (e.kind == EPI_GELU) {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = gelu_erf(v[i]);
      } else if (e.pos) {
        const float4* pr = reinterpret_cast<const float4*>(e.pos + (size_t)(m % e.P) * e.N + n0);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float4 p = __ldg(pr + i);
          v[4 * i] += p.x; v[4 * i + 1] += p.y; v[4 * i + 2] += p.z; v[4 * i + 3] += p.w;
        }
      }
      if (e.out_f32) {
        float4* d4 = reinterpret_cast<float4*>(reinterpret_cast<float*>(e.out) + (size_t)m * e.ldo + n0);
#pragma unroll
        for (int i = 0; i < 8; ++i) d4[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
        break;
      }
      uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<bf16*>(e.out) + (size_t)m * e.ldo + n0);
#pragma unroll
      for (int i = 0; i < 4; ++i)
        dst[i] = make_uint4(pack_bf16(v[8 * i], v[8 * i + 1]), pack_bf16(v[8 * i + 2], v[8 * i + 3]),
                            pack_bf16(v[8 * i + 4], v[8 * i + 5]), pack_bf16(v[8 * i + 6], v[8 * i + 7]));
      break;
    }
    case EPI_RESID: {
      float4* xo = reinterpret_cast<float4*>(e.x_out + (size_t)m * e.N + n0);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float4 a = xin[i];
        xo[i] = make_float4(a.x + v[4 * i], a.y + v[4 * i + 1], a.z + v[4 * i + 2], a.w + v[4 * i + 3]);
      }
      break;
    }
    default: {  // EPI_QKV; a 32-column group never straddles Q/K/V (D % 32 == 0)
      size_t qrow, row;
      qkv_rows(e, m, qrow, row);
      if (n0 < 2 * e.D) {
        bf16* base = (n0 < e.D) ? reinterpret_cast<bf16*>(e.q) + qrow * e.D + n0
                                : reinterpret_cast<bf16*>(e.kslab) + row * e.D + (n0 - e.D);
        uint4* dst = reinterpret_cast<uint4*>(base);
#pragma unroll
        for (int i = 0; i < 4; ++i)
          dst[i] = make_uint4(pack_bf16(v[8 * i], v[8 * i + 1]), pack_bf16(v[8 * i + 2], v[8 * i + 3]),
                              pack_bf16(v[8 * i + 4], v[8 * i + 5]), pack_bf16(v[8 * i + 6], v[8 * i + 7]));
      } else {
        bf16* vt = reinterpret_cast<bf16*>(e.vtslab);
        const size_t ld = (size_t)e.vt_ld;
#pragma unroll
        for (int i = 0; i < 32; ++i) vt[(size_t)(n0 - 2 * e.D + i) * ld + row] = __float2bfloat16_rn(v[i]);
      }
    }
  }
}

}  // namespace vi
