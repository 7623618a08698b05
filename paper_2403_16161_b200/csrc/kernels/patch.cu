// Soft split / soft composite / Fusion-FFN fold-unfold gather kernels (HBM-bound).
//
// Geometry (reading Q6): nn.Unfold semantics with symmetric zero padding; the patch
// vector of token (oy, ox) is ordered (ky, kx, c); feature maps are channels-last.
//   unfold: Tp[t][oy*ow+ox][(ky*kw+kx)*C + c] = F[t][oy*sh-ph+ky][ox*sw-pw+kx][c] (0 if outside)
//   fold:   out[t][y][x][c] = (sum over windows covering (y,x), in token order) / count
// Both are written as GATHERS, so every output byte is written once, coalesced, without
// atomics (deterministic), and the overlapping reads (each input cell is read by up to 9
// windows) hit L1/L2: the 7x7 unfold with one warp per token (its patch vector is kh runs of
// kw*C contiguous input elements; 8 16-byte loads per lane in flight before the stores), the
// fold with one thread per 16-byte vector of an output cell.
// The fold sums in fp32 and divides with IEEE round-to-nearest (no fast-math).
#include <cstdlib>

#include "kernels.h"

namespace vi {

template <typename T, int VEC> struct Vec;
template <> struct Vec<bf16, 8> {
  static __device__ __forceinline__ void ld(const bf16* p, float* f) {
    uint4 u = *reinterpret_cast<const uint4*>(p);
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      f[2 * i] = __uint_as_float(w[i] << 16);
      f[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
    }
  }
  static __device__ __forceinline__ void st(bf16* p, const float* f) {
    *reinterpret_cast<uint4*>(p) =
        make_uint4(pack_bf16(f[0], f[1]), pack_bf16(f[2], f[3]), pack_bf16(f[4], f[5]), pack_bf16(f[6], f[7]));
  }
  static __device__ __forceinline__ void zero(bf16* p) { *reinterpret_cast<uint4*>(p) = make_uint4(0, 0, 0, 0); }
};
template <> struct Vec<float, 4> {
  static __device__ __forceinline__ void ld(const float* p, float* f) {
    float4 v = *reinterpret_cast<const float4*>(p);
    f[0] = v.x; f[1] = v.y; f[2] = v.z; f[3] = v.w;
  }
  static __device__ __forceinline__ void st(float* p, const float* f) {
    *reinterpret_cast<float4*>(p) = make_float4(f[0], f[1], f[2], f[3]);
  }
  static __device__ __forceinline__ void zero(float* p) { *reinterpret_cast<float4*>(p) = make_float4(0, 0, 0, 0); }
};
template <> struct Vec<float, 8> {
  static __device__ __forceinline__ void ld(const float* p, float* f) {
    Vec<float, 4>::ld(p, f);
    Vec<float, 4>::ld(p + 4, f + 4);
  }
  static __device__ __forceinline__ void st(float* p, const float* f) {
    Vec<float, 4>::st(p, f);
    Vec<float, 4>::st(p + 4, f + 4);
  }
  static __device__ __forceinline__ void zero(float* p) {
    Vec<float, 4>::zero(p);
    Vec<float, 4>::zero(p + 4);
  }
};

// Pure copy (bit-exact) unfold.  One CTA per token (t, oy, ox): its kh*kw*C outputs are
// contiguous, so the CTA writes one contiguous run with 16-byte vectors; 32-bit index math.
template <typename T, int VEC>
__global__ void __launch_bounds__(256) unfold_kernel(const T* __restrict__ in, T* __restrict__ out, Geom g, int ntok) {
  griddep_wait();
  griddep_launch();
  const int CV = g.C / VEC, KK = g.kh * g.kw, P = g.oh * g.ow;
  // a CTA covers tpb consecutive tokens (one contiguous output run); v = (j, cv) per token
  const int per = KK * CV;
  const int tpb = (per >= 512) ? 1 : (512 + per - 1) / per;
  const int tok0 = blockIdx.x * tpb;
  for (int vv = threadIdx.x; vv < tpb * per; vv += blockDim.x) {
    const int ti = vv / per, v = vv - ti * per;
    const int gt = tok0 + ti;
    if (gt >= ntok) break;
    const int tok = gt % P, t = gt / P;
    const int oy = tok / g.ow, ox = tok - oy * g.ow;
    const int j = v / CV, cv = v - j * CV;
    const int ky = j / g.kw, kx = j - ky * g.kw;
    const int y = oy * g.sh - g.ph + ky, x = ox * g.sw - g.pw + kx;
    T* d = out + (size_t)gt * KK * g.C + v * VEC;
    if (y < 0 || y >= g.H || x < 0 || x >= g.W) {
      Vec<T, VEC>::zero(d);
    } else {
      const T* src = in + (((size_t)t * g.H + y) * g.W + x) * g.C + cv * VEC;
      if constexpr (sizeof(T) == 2)
        *reinterpret_cast<uint4*>(d) = __ldg(reinterpret_cast<const uint4*>(src));
      else
        *reinterpret_cast<float4*>(d) = __ldg(reinterpret_cast<const float4*>(src));
    }
  }
}

// Fold with cover-count normalisation (gather form), optional GELU of the folded value.
// One CTA per output row (t, y): the covering window rows are CTA-uniform; each thread
// owns 16-byte vectors of cells (x, c).  Up to MAXC x MAXC covering windows are loaded
// first (predicated, all in flight) and then summed in token order (oy, then ox).
// GELU(unfold(z)) = unfold(GELU(z)) (unfold copies, GELU(0) = 0), so the Fusion-FFN
// applies its GELU here, once per folded cell.
template <typename Tin, typename Tout, int VEC, bool GELU>
__global__ void __launch_bounds__(256) fold_kernel(const Tin* __restrict__ in, Tout* __restrict__ out, Geom g) {
  griddep_wait();
  griddep_launch();
  constexpr int MAXC = 3;
  const int CV = g.C / VEC, KK = g.kh * g.kw, P = g.oh * g.ow;
  const int y = blockIdx.x % g.H, t = blockIdx.x / g.H;
  const int yy = y + g.ph;
  int oy0 = yy - g.kh + 1;
  oy0 = oy0 <= 0 ? 0 : (oy0 + g.sh - 1) / g.sh;
  int oy1 = yy / g.sh;
  if (oy1 > g.oh - 1) oy1 = g.oh - 1;
  const Tin* in_t = in + (size_t)t * P * KK * g.C;
  Tout* out_row = out + ((size_t)t * g.H + y) * g.W * g.C;
  for (int v = threadIdx.x; v < g.W * CV; v += blockDim.x) {
    const int x = v / CV, cv = v - x * CV;
    const int xx = x + g.pw;
    int ox0 = xx - g.kw + 1;
    ox0 = ox0 <= 0 ? 0 : (ox0 + g.sw - 1) / g.sw;
    int ox1 = xx / g.sw;
    if (ox1 > g.ow - 1) ox1 = g.ow - 1;
    float f[MAXC][MAXC][VEC];
#pragma unroll
    for (int a = 0; a < MAXC; ++a)
#pragma unroll
      for (int b = 0; b < MAXC; ++b) {
        const int oy = oy0 + a, ox = ox0 + b;
        if (oy <= oy1 && ox <= ox1) {
          const int ky = yy - oy * g.sh, kx = xx - ox * g.sw;
          Vec<Tin, VEC>::ld(in_t + ((size_t)(oy * g.ow + ox) * KK + ky * g.kw + kx) * g.C + cv * VEC, f[a][b]);
        }
      }
    float acc[VEC];
#pragma unroll
    for (int k = 0; k < VEC; ++k) acc[k] = 0.f;
#pragma unroll
    for (int a = 0; a < MAXC; ++a)
#pragma unroll
      for (int b = 0; b < MAXC; ++b)
        if (oy0 + a <= oy1 && ox0 + b <= ox1) {
#pragma unroll
          for (int k = 0; k < VEC; ++k) acc[k] += f[a][b][k];
        }
    const float c = (float)((oy1 - oy0 + 1) * (ox1 - ox0 + 1));
#pragma unroll
    for (int k = 0; k < VEC; ++k) {
      acc[k] = __fdiv_rn(acc[k], c);
      if (GELU) acc[k] = gelu_erf(acc[k]);
    }
    Vec<Tout, VEC>::st(out_row + x * g.C + cv * VEC, acc);
  }
}

// ---- compile-time-geometry variants (the hot shapes: 7x7 kernel, stride 3) ----------------
// Same results as the generic kernels above; all index divisions are by constants.
template <typename T, int VEC, int CV, int KH, int KW>
__global__ void __launch_bounds__(256) unfold_fixed_kernel(const T* __restrict__ in, T* __restrict__ out, Geom g,
                                                           int ntok, unsigned long long* timing) {
  griddep_wait();
  griddep_launch();
  if (timing && threadIdx.x == 0) time_begin(timing);
  constexpr int KK = KH * KW, PER = KK * CV, U = 4;   // U vectors per thread in flight
  const int P = g.oh * g.ow;
  const int total = ntok * PER, stride = gridDim.x * blockDim.x;
  for (int base = blockIdx.x * blockDim.x + threadIdx.x; base < total; base += U * stride) {
    uint4 val[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = base + u * stride;
      val[u] = make_uint4(0u, 0u, 0u, 0u);
      if (i < total) {
        const int gt = i / PER, v = i - gt * PER;        // token, vector within the token
        const int j = v / CV, cv = v - j * CV;
        const int ky = j / KW, kx = j - ky * KW;
        const int t = gt / P, tok = gt - t * P;
        const int oy = tok / g.ow, ox = tok - oy * g.ow;
        const int y = oy * g.sh - g.ph + ky, x = ox * g.sw - g.pw + kx;
        if (y >= 0 && y < g.H && x >= 0 && x < g.W) {
          const T* src = in + (((size_t)t * g.H + y) * g.W + x) * (CV * VEC) + cv * VEC;
          val[u] = __ldg(reinterpret_cast<const uint4*>(src));   // 16 B: 8 bf16 or 4 fp32
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = base + u * stride;
      if (i < total) *reinterpret_cast<uint4*>(out + (size_t)i * VEC) = val[u];
    }
  }
  if (timing) {
    __syncthreads();
    if (threadIdx.x == 0) time_end(timing, gridDim.x);
  }
}

// (4 CTAs of 256 threads per SM: all 9 window loads of a thread stay in flight.  Capping the
// registers for 6 or 8 CTAs per SM, no spills, made the compiler serialise the loads: the F3N
// fold 0.057 -> 0.145 / 0.217 ms per C3 step)
// HH, WW > 0: the output map is HH x WW with padding (KH - 1) / 2 (the memory step's shapes:
// 60 x 108, 7x7 / 3 / 3 -> 20 x 36 tokens) -- every index division is by a constant and the
// input offsets are 32-bit (the launcher checks the tensor fits); the same arithmetic in the
// same order as the runtime-geometry instantiation (bitwise equal results)
template <typename Tin, typename Tout, int VEC, int CV, int KH, int KW, int SH, int SW, bool GELU, int HH = 0, int WW = 0>
__global__ void __launch_bounds__(256, 4) fold_fixed_kernel(const Tin* __restrict__ in, Tout* __restrict__ out, Geom g,
                                                         int ncell, unsigned long long* timing) {
  griddep_wait();
  griddep_launch();
  if (timing && threadIdx.x == 0) time_begin(timing);
  constexpr int KK = KH * KW, C = CV * VEC;
  constexpr int MAXC = (KH + SH - 1) / SH > (KW + SW - 1) / SW ? (KH + SH - 1) / SH : (KW + SW - 1) / SW;
  constexpr bool CG = HH > 0 && WW > 0;
  constexpr int CPH = (KH - 1) / 2, CPW = (KW - 1) / 2;
  constexpr int COH = CG ? (HH + 2 * CPH - KH) / SH + 1 : 1, COW = CG ? (WW + 2 * CPW - KW) / SW + 1 : 1;
  const int H = CG ? HH : g.H, W = CG ? WW : g.W, ph = CG ? CPH : g.ph, pw = CG ? CPW : g.pw;
  const int oh = CG ? COH : g.oh, ow = CG ? COW : g.ow;
  const int P = oh * ow;
  const int total = ncell * CV;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int cell = i / CV, cv = i - cell * CV;
    const int tw = cell / W, x = cell - tw * W;
    const int t = tw / H, y = tw - t * H;
    const int yy = y + ph, xx = x + pw;
    int oy0 = yy - KH + 1;
    oy0 = oy0 <= 0 ? 0 : (oy0 + SH - 1) / SH;
    int oy1 = yy / SH;
    oy1 = oy1 < oh - 1 ? oy1 : oh - 1;
    int ox0 = xx - KW + 1;
    ox0 = ox0 <= 0 ? 0 : (ox0 + SW - 1) / SW;
    int ox1 = xx / SW;
    ox1 = ox1 < ow - 1 ? ox1 : ow - 1;
    const Tin* in_t = in + (CG ? (size_t)(unsigned)(t * P * KK * C) : (size_t)t * P * KK * C) + cv * VEC;
    float acc[VEC];
#pragma unroll
    for (int k = 0; k < VEC; ++k) acc[k] = 0.f;
    float f[MAXC][MAXC][VEC];
#pragma unroll
    for (int a = 0; a < MAXC; ++a)
#pragma unroll
      for (int b = 0; b < MAXC; ++b)
        if (oy0 + a <= oy1 && ox0 + b <= ox1) {
          const int oy = oy0 + a, ox = ox0 + b;
          const int ky = yy - oy * SH, kx = xx - ox * SW;
          if constexpr (CG)
            Vec<Tin, VEC>::ld(in_t + (unsigned)(((oy * ow + ox) * KK + ky * KW + kx) * C), f[a][b]);
          else
            Vec<Tin, VEC>::ld(in_t + ((size_t)(oy * ow + ox) * KK + ky * KW + kx) * C, f[a][b]);
        }
#pragma unroll
    for (int a = 0; a < MAXC; ++a)
#pragma unroll
      for (int b = 0; b < MAXC; ++b)
        if (oy0 + a <= oy1 && ox0 + b <= ox1) {
#pragma unroll
          for (int k = 0; k < VEC; ++k) acc[k] += f[a][b][k];
        }
    const float c = (float)((oy1 - oy0 + 1) * (ox1 - ox0 + 1));
#pragma unroll
    for (int k = 0; k < VEC; ++k) {
      acc[k] = __fdiv_rn(acc[k], c);
      if (GELU) acc[k] = gelu_erf(acc[k]);
    }
    if constexpr (CG)
      Vec<Tout, VEC>::st(out + (unsigned)(cell * C + cv * VEC), acc);
    else
      Vec<Tout, VEC>::st(out + (size_t)cell * C + cv * VEC, acc);
  }
  if (timing) {
    __syncthreads();
    if (threadIdx.x == 0) time_end(timing, gridDim.x);
  }
}

// ---- warp-per-token unfold (7x7 patches) --------------------------------------------------
// One warp per token: the token's patch vector is KH runs (one per kernel row ky) of KW
// consecutive input cells, i.e. KH contiguous spans of KW*C elements of the input row y; the
// warp issues all its 16-B loads (R per lane) before any store.  Same bytes as unfold_fixed.
template <typename T, int CV, int KH, int KW, int R>
__global__ void __launch_bounds__(256) unfold_warp_kernel(const T* __restrict__ in, T* __restrict__ out, Geom g,
                                                          int ntok, unsigned long long* timing) {
  griddep_wait();
  griddep_launch();
  if (timing && threadIdx.x == 0) time_begin(timing);
  constexpr int PER = KH * KW * CV, VEC = 16 / sizeof(T);
  const int gt = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (gt < ntok) {
    const int P = g.oh * g.ow, t = gt / P, tok = gt - t * P;
    const int oy = tok / g.ow, ox = tok - oy * g.ow;
    const int ybase = oy * g.sh - g.ph, xbase = ox * g.sw - g.pw;
    const T* in_t = in + (size_t)t * g.H * g.W * (CV * VEC);
    uint4* dst = reinterpret_cast<uint4*>(out + (size_t)gt * PER * VEC);
#pragma unroll 1
    for (int v0 = 0; v0 < PER; v0 += 32 * R) {
      uint4 val[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int v = v0 + r * 32 + lane;
        val[r] = make_uint4(0u, 0u, 0u, 0u);
        if (v < PER) {
          const int j = v / CV, cv = v - j * CV;
          const int ky = j / KW, kx = j - ky * KW;
          const int y = ybase + ky, x = xbase + kx;
          if (y >= 0 && y < g.H && x >= 0 && x < g.W)
            val[r] = __ldg(reinterpret_cast<const uint4*>(in_t + ((size_t)y * g.W + x) * (CV * VEC)) + cv);
        }
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int v = v0 + r * 32 + lane;
        if (v < PER) dst[v] = val[r];
      }
    }
  }
  if (timing) {
    __syncthreads();
    if (threadIdx.x == 0) time_end(timing, gridDim.x);
  }
}

template <> struct Vec<bf16, 4> {
  static __device__ __forceinline__ void ld(const bf16* p, float* f) {
    uint2 u = *reinterpret_cast<const uint2*>(p);
    f[0] = __uint_as_float(u.x << 16); f[1] = __uint_as_float(u.x & 0xFFFF0000u);
    f[2] = __uint_as_float(u.y << 16); f[3] = __uint_as_float(u.y & 0xFFFF0000u);
  }
  static __device__ __forceinline__ void st(bf16* p, const float* f) {
    *reinterpret_cast<uint2*>(p) = make_uint2(pack_bf16(f[0], f[1]), pack_bf16(f[2], f[3]));
  }
  static __device__ __forceinline__ void zero(bf16* p) { *reinterpret_cast<uint2*>(p) = make_uint2(0, 0); }
};

static int grid_cap(long long total, int per_block = 256) {
  long long b = (total + per_block - 1) / per_block;
  return int(b < 148 * 32 ? (b ? b : 1) : 148 * 32);
}

// VI_PATCH_V=0 (A/B only): the 7x7 unfold as per-vector gathers (unfold_fixed_kernel) instead
// of one warp per token, and the fold with runtime geometry instead of the compile-time
// 60 x 108 map (tests/test_gpu_patch_variants.py: bitwise equal)
static int patch_variant() {
  static const int v = [] {
    const char* e = getenv("VI_PATCH_V");
    return e && e[0] == '0' ? 0 : 1;
  }();
  return v;
}

cudaError_t launch_unfold(const void* in, void* out, int n, const Geom& g, int dtype, cudaStream_t st,
                          unsigned long long* timing) {
  const int ntok = n * g.oh * g.ow;
  if (g.kh == 7 && g.kw == 7 && patch_variant() == 1) {
    const int CV = g.C / (dtype == 0 ? 8 : 4);
    const int blocks = (ntok + 7) / 8;   // 8 warps (tokens) per block
#define UW(T, CVV)                                                                                        \
    if (CV == CVV) {                                                                                      \
      pdl_launch(unfold_warp_kernel<T, CVV, 7, 7, 8>, dim3(blocks), dim3(256), 0, st, (const T*)in, (T*)out, g, ntok, timing); \
      return cudaGetLastError();                                                                          \
    }
    if (dtype == 0) { UW(bf16, 16) UW(bf16, 5) }
    else { UW(float, 10) UW(float, 32) }
#undef UW
  }
  if (g.kh == 7 && g.kw == 7) {
    const int CV = g.C / (dtype == 0 ? 8 : 4);
    const long long total = (long long)ntok * 49 * CV;
    // 4 vectors per thread in flight when that still leaves >= 4 blocks per SM (C3: yes; one
    // frame per step: no, there every vector gets its own thread)
    const long long threads = (total + 3) / 4 >= 148LL * 4 * 256 ? (total + 3) / 4 : total;
#define UF(T, V, CVV)                                                                                     \
    if (CV == CVV) {                                                                                      \
      pdl_launch(unfold_fixed_kernel<T, V, CVV, 7, 7>, dim3(grid_cap(threads)), dim3(256), 0, st, (const T*)in, (T*)out, g, ntok, timing); \
      return cudaGetLastError();                                                                          \
    }
    if (dtype == 0) { UF(bf16, 8, 16) UF(bf16, 8, 5) UF(bf16, 8, 32) }
    else { UF(float, 4, 4) UF(float, 4, 10) UF(float, 4, 32) }
#undef UF
  }
  const int per = g.kh * g.kw * (g.C / (dtype == 0 ? 8 : 4));
  const int tpb = (per >= 512) ? 1 : (512 + per - 1) / per;
  const int blocks = (ntok + tpb - 1) / tpb;
  if (dtype == 0)
    pdl_launch(unfold_kernel<bf16, 8>, dim3(blocks), dim3(256), 0, st, (const bf16*)in, (bf16*)out, g, ntok);
  else
    pdl_launch(unfold_kernel<float, 4>, dim3(blocks), dim3(256), 0, st, (const float*)in, (float*)out, g, ntok);
  return cudaGetLastError();
}

cudaError_t launch_fold(const void* in, int in_dtype, void* out, int out_dtype, int n, const Geom& g, bool gelu,
                        cudaStream_t st, unsigned long long* timing) {
  const int blocks = n * g.H;
  if (g.kh == 7 && g.kw == 7 && g.sh == 3 && g.sw == 3) {
    const int ncell = n * g.H * g.W;
    // the memory step's map (60 x 108, padding 3): compile-time geometry, 32-bit offsets
    const bool c3 = g.H == 60 && g.W == 108 && g.ph == 3 && g.pw == 3 && g.oh == 20 && g.ow == 36 &&
                    (long long)n * g.oh * g.ow * 49 * g.C < (1ll << 31) && patch_variant() == 1;
#define FF(TI, TO, V, CVV)                                                                                    \
    if (g.C == CVV * V) {                                                                                     \
      const long long total = (long long)ncell * CVV;                                                        \
      if (c3 && gelu)                                                                                         \
        pdl_launch(fold_fixed_kernel<TI, TO, V, CVV, 7, 7, 3, 3, true, 60, 108>, dim3(grid_cap(total)), dim3(256), 0, st, (const TI*)in, (TO*)out, g, ncell, timing); \
      else if (c3)                                                                                            \
        pdl_launch(fold_fixed_kernel<TI, TO, V, CVV, 7, 7, 3, 3, false, 60, 108>, dim3(grid_cap(total)), dim3(256), 0, st, (const TI*)in, (TO*)out, g, ncell, timing); \
      else if (gelu)                                                                                          \
        pdl_launch(fold_fixed_kernel<TI, TO, V, CVV, 7, 7, 3, 3, true>, dim3(grid_cap(total)), dim3(256), 0, st, (const TI*)in, (TO*)out, g, ncell, timing); \
      else                                                                                                    \
        pdl_launch(fold_fixed_kernel<TI, TO, V, CVV, 7, 7, 3, 3, false>, dim3(grid_cap(total)), dim3(256), 0, st, (const TI*)in, (TO*)out, g, ncell, timing); \
      return cudaGetLastError();                                                                              \
    }
    if (in_dtype == 1 && out_dtype == 0) { FF(float, bf16, 4, 10) FF(float, bf16, 4, 32) }
    if (in_dtype == 1 && out_dtype == 1) { FF(float, float, 4, 10) FF(float, float, 4, 4) FF(float, float, 4, 32) }
    if (in_dtype == 0 && out_dtype == 0) { FF(bf16, bf16, 8, 16) FF(bf16, bf16, 8, 5) }
#undef FF
  }
#define FOLD(TI, TO, V)                                                                              \
  (gelu ? (pdl_launch(fold_kernel<TI, TO, V, true>, dim3(blocks), dim3(256), 0, st, (const TI*)in, (TO*)out, g), 0)        \
        : (pdl_launch(fold_kernel<TI, TO, V, false>, dim3(blocks), dim3(256), 0, st, (const TI*)in, (TO*)out, g), 0))
  if (in_dtype == 0 && out_dtype == 0) FOLD(bf16, bf16, 8);
  else if (in_dtype == 0) FOLD(bf16, float, 8);
  else if (out_dtype == 1) FOLD(float, float, 4);
  else FOLD(float, bf16, 8);
#undef FOLD
  return cudaGetLastError();
}

}  // namespace vi
