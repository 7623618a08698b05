// Row kernels: pre-norm LayerNorm (reading Q1, eps 1e-5), fp32 -> bf16 cast, and the
// V transpose used by refine commits (the memory stores V transposed, [D][S*P]).
#include <cstdlib>

#include "kernels.h"

namespace vi {

// VI_PDL=0 turns programmatic dependent launch off (A/B measurements)
int g_pdl = [] {
  const char* e = getenv("VI_PDL");
  return (e && e[0] == '0') ? 0 : 1;
}();

// One warp per row; D <= 1024 and D % 32 == 0.  Two-pass mean / variance in registers.
template <typename Tout, int PER>
__global__ void layernorm_kernel(const float* __restrict__ x, const float* __restrict__ g,
                                 const float* __restrict__ b, Tout* __restrict__ out, int rows, int D) {
  griddep_wait();
  griddep_launch();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= rows) return;
  const float* xr = x + (size_t)warp * D;
  float v[PER];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int c = i * 32 + lane;
    v[i] = c < D ? xr[c] : 0.f;
    s += v[i];
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const float mu = s / D;
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int c = i * 32 + lane;
    const float d = c < D ? v[i] - mu : 0.f;
    q += d * d;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
  const float rstd = rsqrtf(q / D + 1e-5f);
  Tout* orow = out + (size_t)warp * D;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int c = i * 32 + lane;
    if (c < D) orow[c] = from_f<Tout>((v[i] - mu) * rstd * g[c] + b[c]);
  }
}

// Vectorised variant for D % 128 == 0 (D <= 1024): lane l owns float4 columns l, l+32, ...
// so every load / store instruction of a warp covers one contiguous 512 B (256 B) span.
// LayerNorm of one row held as float4 v[NV] by a warp (lane l owns float4 columns l, l+32, ...)
template <typename Tout, int NV>
__device__ __forceinline__ void ln_row_v4(const float4 (&v)[NV], const float4* __restrict__ g,
                                          const float4* __restrict__ b, Tout* __restrict__ out, size_t row, int D,
                                          int lane) {
  const int D4 = D / 4;
  float sm = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) sm += (v[i].x + v[i].y) + (v[i].z + v[i].w);
#pragma unroll
  for (int o = 16; o; o >>= 1) sm += __shfl_xor_sync(0xffffffffu, sm, o);
  const float mu = sm / D;
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const float a0 = v[i].x - mu, a1 = v[i].y - mu, a2 = v[i].z - mu, a3 = v[i].w - mu;
    q += (a0 * a0 + a1 * a1) + (a2 * a2 + a3 * a3);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
  const float rstd = rsqrtf(q / D + 1e-5f);
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const float4 gg = __ldg(g + i * 32 + lane), bb = __ldg(b + i * 32 + lane);
    const float o0 = (v[i].x - mu) * rstd * gg.x + bb.x, o1 = (v[i].y - mu) * rstd * gg.y + bb.y;
    const float o2 = (v[i].z - mu) * rstd * gg.z + bb.z, o3 = (v[i].w - mu) * rstd * gg.w + bb.w;
    if constexpr (sizeof(Tout) == 2) {
      reinterpret_cast<uint2*>(out)[row * D4 + i * 32 + lane] = make_uint2(pack_bf16(o0, o1), pack_bf16(o2, o3));
    } else {
      reinterpret_cast<float4*>(out)[row * D4 + i * 32 + lane] = make_float4(o0, o1, o2, o3);
    }
  }
}

// Vectorised variant for D % 128 == 0 (D <= 1024): lane l owns float4 columns l, l+32, ...
// so every load / store instruction of a warp covers one contiguous 512 B (256 B) span.
template <typename Tout, int NV>
__global__ void __launch_bounds__(256) layernorm_v4_kernel(const float4* __restrict__ x, const float4* __restrict__ g,
                                                           const float4* __restrict__ b, Tout* __restrict__ out,
                                                           int rows, int D) {
  griddep_wait();
  griddep_launch();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= rows) return;
  const float4* xr = x + (size_t)warp * (D / 4);
  float4 v[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) v[i] = xr[i * 32 + lane];
  ln_row_v4<Tout, NV>(v, g, b, out, warp, D, lane);
}

// Split-K reduction (gemm_tc with Epi::ksplit > 1): row m of the output is
// out = x_in + (bias + sum_s ws[s][m]) (x_in == NULL: no residual) with the partials added in
// split order s = 0, 1, ... (deterministic), then + pos[m % P] when pos != NULL (the embedding's
// positional table, the unsplit epilogue's order); LN (g != NULL) also writes LayerNorm(out)
// to h, i.e. the next pre-norm (Q1) fused into the reduction.  One warp per row, D % 128 == 0,
// D <= 1024.
template <typename Tout, int NV, bool LN>
__global__ void __launch_bounds__(256) splitk_resid_kernel(const float4* __restrict__ ws, int ksplit, size_t split_ld4,
                                                           const float4* __restrict__ bias, const float4* x_in,
                                                           float4* x_out, const float4* __restrict__ pos, int P,
                                                           const float4* __restrict__ g, const float4* __restrict__ b,
                                                           Tout* __restrict__ h, int rows, int D,
                                                           unsigned long long* timing) {
  griddep_wait();
  if (threadIdx.x == 0) time_begin(timing);
  griddep_launch();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp < rows) {   // (x_in may alias x_out: each element is read before it is written, by one thread)
    const size_t r4 = (size_t)warp * (D / 4);
    float4 v[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] = ws[r4 + i * 32 + lane];
    for (int s = 1; s < ksplit; ++s) {
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        const float4 p = ws[s * split_ld4 + r4 + i * 32 + lane];
        v[i].x += p.x; v[i].y += p.y; v[i].z += p.z; v[i].w += p.w;
      }
    }
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const float4 bb = __ldg(bias + i * 32 + lane);
      v[i].x += bb.x; v[i].y += bb.y; v[i].z += bb.z; v[i].w += bb.w;
      if (x_in) {
        const float4 xi = x_in[r4 + i * 32 + lane];
        v[i].x = xi.x + v[i].x; v[i].y = xi.y + v[i].y; v[i].z = xi.z + v[i].z; v[i].w = xi.w + v[i].w;
      }
      if (pos) {
        const float4 pp = __ldg(pos + (size_t)(warp % P) * (D / 4) + i * 32 + lane);
        v[i].x += pp.x; v[i].y += pp.y; v[i].z += pp.z; v[i].w += pp.w;
      }
      x_out[r4 + i * 32 + lane] = v[i];
    }
    if constexpr (LN) ln_row_v4<Tout, NV>(v, g, b, h, warp, D, lane);
  }
  if (timing) {
    __syncthreads();
    if (threadIdx.x == 0) time_end(timing, gridDim.x);
  }
}

cudaError_t launch_splitk_resid(const float* ws, int ksplit, size_t split_ld, const float* bias, const float* x_in,
                                float* x_out, const float* pos, int P, const float* g, const float* b, void* h,
                                int h_dtype, int rows, int D, cudaStream_t st, unsigned long long* timing) {
  if (D % 128 || D > 1024 || ksplit < 1 || split_ld % 4 || (pos && P < 1)) return cudaErrorInvalidValue;
  const int blocks = (rows * 32 + 255) / 256;
  const size_t ld4 = split_ld / 4;
#define SKR(NV)                                                                                                    \
  if (D == NV * 128) {                                                                                             \
    if (!g)                                                                                                        \
      pdl_launch(splitk_resid_kernel<bf16, NV, false>, dim3(blocks), dim3(256), 0, st, (const float4*)ws, ksplit,  \
                 ld4, (const float4*)bias, (const float4*)x_in, (float4*)x_out, (const float4*)pos, P,             \
                 (const float4*)nullptr, (const float4*)nullptr, (bf16*)nullptr, rows, D, timing);                 \
    else if (h_dtype == 0)                                                                                         \
      pdl_launch(splitk_resid_kernel<bf16, NV, true>, dim3(blocks), dim3(256), 0, st, (const float4*)ws, ksplit,   \
                 ld4, (const float4*)bias, (const float4*)x_in, (float4*)x_out, (const float4*)pos, P,             \
                 (const float4*)g, (const float4*)b, (bf16*)h, rows, D, timing);                                   \
    else                                                                                                           \
      pdl_launch(splitk_resid_kernel<float, NV, true>, dim3(blocks), dim3(256), 0, st, (const float4*)ws, ksplit,  \
                 ld4, (const float4*)bias, (const float4*)x_in, (float4*)x_out, (const float4*)pos, P,             \
                 (const float4*)g, (const float4*)b, (float*)h, rows, D, timing);                                  \
    return cudaGetLastError();                                                                                     \
  }
  SKR(1) SKR(2) SKR(3) SKR(4) SKR(5) SKR(6) SKR(7) SKR(8)
#undef SKR
  return cudaErrorInvalidValue;
}

cudaError_t launch_layernorm(const float* x, const float* g, const float* b, void* out, int out_dtype, int rows,
                             int D, cudaStream_t st) {
  const int blocks = (rows * 32 + 255) / 256;
  if (D % 128 == 0 && D <= 1024) {
#define LNV(NV)                                                                                                    if (D == NV * 128) {                                                                                               if (out_dtype == 0)                                                                                                pdl_launch(layernorm_v4_kernel<bf16, NV>, dim3(blocks), dim3(256), 0, st, (const float4*)x, (const float4*)g, (const float4*)b,                                                             (bf16*)out, rows, D);                                   else                                                                                                               pdl_launch(layernorm_v4_kernel<float, NV>, dim3(blocks), dim3(256), 0, st, (const float4*)x, (const float4*)g,                                                                              (const float4*)b, (float*)out, rows, D);                return cudaGetLastError();                                                                                     }
    LNV(1) LNV(2) LNV(3) LNV(4) LNV(5) LNV(6) LNV(7) LNV(8)
#undef LNV
  }
#define LN_CASE(PER)                                                                                   \
  if (D <= PER * 32) {                                                                                 \
    if (out_dtype == 0)                                                                                \
      pdl_launch(layernorm_kernel<bf16, PER>, dim3(blocks), dim3(256), 0, st, x, g, b, (bf16*)out, rows, D);               \
    else                                                                                               \
      pdl_launch(layernorm_kernel<float, PER>, dim3(blocks), dim3(256), 0, st, x, g, b, (float*)out, rows, D);             \
    return cudaGetLastError();                                                                         \
  }
  LN_CASE(2) LN_CASE(4) LN_CASE(8) LN_CASE(16) LN_CASE(32)
#undef LN_CASE
  return cudaErrorInvalidValue;
}

// x [rows][D] fp32 -> [rows][2D] bf16 with hi = bf16(x) in columns 0..D-1 and
// lo = bf16(x - hi) in D..2D-1: a K = 2D GEMM against [W | W] then sees x to ~2^-17.
__global__ void split_bf16_kernel(const float4* __restrict__ x, uint2* __restrict__ out, int rows, int D4) {
  griddep_wait();
  griddep_launch();
  const size_t n4 = (size_t)rows * D4;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    const size_t r = i / D4, c = i - r * D4;
    const float4 v = x[i];
    const __nv_bfloat162 h01 = __floats2bfloat162_rn(v.x, v.y), h23 = __floats2bfloat162_rn(v.z, v.w);
    const float2 f01 = __bfloat1622float2(h01), f23 = __bfloat1622float2(h23);
    out[r * 2 * D4 + c] = make_uint2(*reinterpret_cast<const uint32_t*>(&h01), *reinterpret_cast<const uint32_t*>(&h23));
    out[r * 2 * D4 + D4 + c] = make_uint2(pack_bf16(v.x - f01.x, v.y - f01.y), pack_bf16(v.z - f23.x, v.w - f23.y));
  }
}

cudaError_t launch_split_bf16(const float* x, void* out, int rows, int D, cudaStream_t st) {
  const size_t n4 = (size_t)rows * D / 4;
  size_t blocks = (n4 + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (!blocks) blocks = 1;
  pdl_launch(split_bf16_kernel, dim3(unsigned(blocks)), dim3(256), 0, st, reinterpret_cast<const float4*>(x), reinterpret_cast<uint2*>(out),
                                                      rows, D / 4);
  return cudaGetLastError();
}

// v [P][D] (row pitch sld) -> vt[d][col0 + p] (row pitch ld elements), 32x32 smem tiles.
template <typename T>
__global__ void transpose_kernel(const T* __restrict__ v, T* __restrict__ vt, int P, int D, size_t ld, size_t col0,
                                 int sld) {
  griddep_wait();
  griddep_launch();
  __shared__ T tile[32][33];
  const int p0 = blockIdx.x * 32, d0 = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int p = p0 + i, d = d0 + threadIdx.x;
    if (p < P && d < D) tile[i][threadIdx.x] = v[(size_t)p * sld + d];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int d = d0 + i, p = p0 + threadIdx.x;
    if (p < P && d < D) vt[(size_t)d * ld + col0 + p] = tile[threadIdx.x][i];
  }
}

cudaError_t launch_transpose_to_slab(const void* v, void* vt_slab, int P, int D, size_t ld, size_t col0, int dtype,
                                     cudaStream_t st, int src_ld) {
  dim3 grid((P + 31) / 32, (D + 31) / 32), block(32, 8);
  const int sld = src_ld > 0 ? src_ld : D;
  if (dtype == 0)
    pdl_launch(transpose_kernel<bf16>, dim3(grid), dim3(block), 0, st, (const bf16*)v, (bf16*)vt_slab, P, D, ld, col0, sld);
  else
    pdl_launch(transpose_kernel<float>, dim3(grid), dim3(block), 0, st, (const float*)v, (float*)vt_slab, P, D, ld, col0, sld);
  return cudaGetLastError();
}

}  // namespace vi

namespace vi {

// og [H][q][part_rows][hd] -> o [M][H*hd]: token m = t*P + i of head h comes from part
// p = i / (P/q), row t*(P/q) + i - p*(P/q) (16-byte vectors; bf16)
__global__ void window_part_gather_kernel(const uint4* __restrict__ og, uint4* __restrict__ o, int M, int P, int H,
                                          int hd8, int q, int part_rows) {
  griddep_wait();
  griddep_launch();
  const int split = P / q;
  const size_t total = (size_t)M * H * hd8;
  for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total; idx += (size_t)gridDim.x * blockDim.x) {
    const int c = int(idx % hd8);
    const size_t r = idx / hd8;
    const int h = int(r % H), m = int(r / H);
    const int t = m / P, i = m - t * P, p = i / split;
    const size_t src_row = ((size_t)h * q + p) * part_rows + (size_t)t * split + (i - p * split);
    o[((size_t)m * H + h) * hd8 + c] = og[src_row * hd8 + c];
  }
}

cudaError_t launch_window_part_gather(const void* og, void* o, int M, int P, int H, int hd, int q, int part_rows,
                                      cudaStream_t st) {
  if (hd % 8 || q < 1 || P % q) return cudaErrorInvalidValue;
  const size_t total = (size_t)M * H * (hd / 8);
  int blocks = int((total + 255) / 256);
  if (blocks > 148 * 8) blocks = 148 * 8;
  pdl_launch(window_part_gather_kernel, dim3(blocks), dim3(256), 0, st, (const uint4*)og, (uint4*)o, M, P, H, hd / 8,
             q, part_rows);
  return cudaGetLastError();
}

}  // namespace vi
