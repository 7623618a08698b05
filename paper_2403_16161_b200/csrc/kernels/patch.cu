// Soft split / soft composite / Fusion-FFN fold-unfold gather kernels (HBM-bound).
//
// Geometry (reading Q6): nn.Unfold semantics with symmetric zero padding; the patch
// vector of token (oy, ox) is ordered (ky, kx, c); feature maps are channels-last.
//   unfold: Tp[t][oy*ow+ox][(ky*kw+kx)*C + c] = F[t][oy*sh-ph+ky][ox*sw-pw+kx][c] (0 if outside)
//   fold:   out[t][y][x][c] = (sum over windows covering (y,x), in token order) / count
// Both are written as GATHERS with one thread per 16-byte vector of the output, so
// every output byte is written once, coalesced, without atomics (deterministic), and
// the overlapping reads (each input cell is read by up to 9 windows) hit L1/L2.
// The fold sums in fp32 and divides with IEEE round-to-nearest (no fast-math).
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

// Pure copy (bit-exact) unfold: one thread per output vector.
template <typename T, int VEC>
__global__ void unfold_kernel(const T* __restrict__ in, T* __restrict__ out, int n, Geom g) {
  const int CV = g.C / VEC, KK = g.kh * g.kw, P = g.oh * g.ow;
  const size_t total = (size_t)n * P * KK * CV;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const int cv = int(i % CV);
    size_t r = i / CV;
    const int j = int(r % KK); r /= KK;
    const int tok = int(r % P);
    const int t = int(r / P);
    const int oy = tok / g.ow, ox = tok - oy * g.ow;
    const int ky = j / g.kw, kx = j - ky * g.kw;
    const int y = oy * g.sh - g.ph + ky, x = ox * g.sw - g.pw + kx;
    T* dst = out + i * VEC;
    if (y < 0 || y >= g.H || x < 0 || x >= g.W) {
      Vec<T, VEC>::zero(dst);
    } else {
      const T* src = in + (((size_t)t * g.H + y) * g.W + x) * g.C + cv * VEC;
      if constexpr (sizeof(T) == 2)
        *reinterpret_cast<uint4*>(dst) = __ldg(reinterpret_cast<const uint4*>(src));
      else
        *reinterpret_cast<float4*>(dst) = __ldg(reinterpret_cast<const float4*>(src));
    }
  }
}

// F3N: GELU(unfold(folded fp32 map)) -> Tout.
template <typename Tout, int VEC>
__global__ void unfold_gelu_kernel(const float* __restrict__ in, Tout* __restrict__ out, int n, Geom g) {
  const int CV = g.C / VEC, KK = g.kh * g.kw, P = g.oh * g.ow;
  const size_t total = (size_t)n * P * KK * CV;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const int cv = int(i % CV);
    size_t r = i / CV;
    const int j = int(r % KK); r /= KK;
    const int tok = int(r % P);
    const int t = int(r / P);
    const int oy = tok / g.ow, ox = tok - oy * g.ow;
    const int ky = j / g.kw, kx = j - ky * g.kw;
    const int y = oy * g.sh - g.ph + ky, x = ox * g.sw - g.pw + kx;
    float f[VEC];
    if (y < 0 || y >= g.H || x < 0 || x >= g.W) {
#pragma unroll
      for (int v = 0; v < VEC; ++v) f[v] = 0.f;      // GELU(0) = 0
    } else {
      Vec<float, VEC>::ld(in + (((size_t)t * g.H + y) * g.W + x) * g.C + cv * VEC, f);
#pragma unroll
      for (int v = 0; v < VEC; ++v) f[v] = gelu_erf(f[v]);
    }
    Vec<Tout, VEC>::st(out + i * VEC, f);
  }
}

// Fold with cover-count normalisation, gather formulation.
template <typename Tin, typename Tout, int VEC>
__global__ void fold_kernel(const Tin* __restrict__ in, Tout* __restrict__ out, int n, Geom g) {
  const int CV = g.C / VEC, KK = g.kh * g.kw, P = g.oh * g.ow;
  const size_t total = (size_t)n * g.H * g.W * CV;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const int cv = int(i % CV);
    size_t r = i / CV;
    const int x = int(r % g.W); r /= g.W;
    const int y = int(r % g.H);
    const int t = int(r / g.H);
    // windows oy with oy*sh - ph <= y <= oy*sh - ph + kh - 1
    const int yy = y + g.ph, xx = x + g.pw;
    int oy0 = yy - g.kh + 1; oy0 = oy0 <= 0 ? 0 : (oy0 + g.sh - 1) / g.sh;
    int oy1 = yy / g.sh; if (oy1 > g.oh - 1) oy1 = g.oh - 1;
    int ox0 = xx - g.kw + 1; ox0 = ox0 <= 0 ? 0 : (ox0 + g.sw - 1) / g.sw;
    int ox1 = xx / g.sw; if (ox1 > g.ow - 1) ox1 = g.ow - 1;
    float acc[VEC];
#pragma unroll
    for (int v = 0; v < VEC; ++v) acc[v] = 0.f;
    int cnt = 0;
    for (int oy = oy0; oy <= oy1; ++oy) {
      const int ky = yy - oy * g.sh;
      for (int ox = ox0; ox <= ox1; ++ox) {
        const int kx = xx - ox * g.sw;
        const Tin* src = in + (((size_t)t * P + oy * g.ow + ox) * KK + ky * g.kw + kx) * g.C + cv * VEC;
        float f[VEC];
        Vec<Tin, VEC>::ld(src, f);
#pragma unroll
        for (int v = 0; v < VEC; ++v) acc[v] += f[v];
        ++cnt;
      }
    }
    const float c = (float)cnt;
#pragma unroll
    for (int v = 0; v < VEC; ++v) acc[v] = __fdiv_rn(acc[v], c);
    Vec<Tout, VEC>::st(out + i * VEC, acc);
  }
}

static int grid_for(size_t total) {
  size_t b = (total + 255) / 256;
  const size_t cap = 148 * 16;
  return int(b < cap ? (b ? b : 1) : cap);
}

cudaError_t launch_unfold(const void* in, void* out, int n, const Geom& g, int dtype, cudaStream_t st) {
  const int VEC = dtype == 0 ? 8 : 4;
  const size_t total = (size_t)n * g.oh * g.ow * g.kh * g.kw * (g.C / VEC);
  if (dtype == 0)
    unfold_kernel<bf16, 8><<<grid_for(total), 256, 0, st>>>((const bf16*)in, (bf16*)out, n, g);
  else
    unfold_kernel<float, 4><<<grid_for(total), 256, 0, st>>>((const float*)in, (float*)out, n, g);
  return cudaGetLastError();
}

cudaError_t launch_unfold_gelu(const float* in, void* out, int n, const Geom& g, int out_dtype, cudaStream_t st) {
  const int VEC = out_dtype == 0 ? 8 : 4;
  const size_t total = (size_t)n * g.oh * g.ow * g.kh * g.kw * (g.C / VEC);
  if (out_dtype == 0)
    unfold_gelu_kernel<bf16, 8><<<grid_for(total), 256, 0, st>>>(in, (bf16*)out, n, g);
  else
    unfold_gelu_kernel<float, 4><<<grid_for(total), 256, 0, st>>>(in, (float*)out, n, g);
  return cudaGetLastError();
}

cudaError_t launch_fold(const void* in, int in_dtype, void* out, int out_dtype, int n, const Geom& g,
                        cudaStream_t st) {
  if (in_dtype == 0) {
    const size_t total = (size_t)n * g.H * g.W * (g.C / 8);
    if (out_dtype == 0)
      fold_kernel<bf16, bf16, 8><<<grid_for(total), 256, 0, st>>>((const bf16*)in, (bf16*)out, n, g);
    else
      fold_kernel<bf16, float, 8><<<grid_for(total), 256, 0, st>>>((const bf16*)in, (float*)out, n, g);
  } else if (out_dtype == 1) {
    const size_t total = (size_t)n * g.H * g.W * (g.C / 4);
    fold_kernel<float, float, 4><<<grid_for(total), 256, 0, st>>>((const float*)in, (float*)out, n, g);
  } else {
    const size_t total = (size_t)n * g.H * g.W * (g.C / 8);
    fold_kernel<float, bf16, 8><<<grid_for(total), 256, 0, st>>>((const float*)in, (bf16*)out, n, g);
  }
  return cudaGetLastError();
}

}  // namespace vi
