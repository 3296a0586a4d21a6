#include <algorithm>
#include <cstdlib>
// train_kernels.cu -- non-GEMM kernels of the decoder trainer step (see
// train.cuh).  Correctness-first CUDA-core implementations; every reduction
// over rows that feeds a weight gradient uses fp32 atomics (gradients are
// compared within tolerance, not bit-exactly).
#include <cmath>

#include "decoder.cuh"
#include "gemm.cuh"
#include "train.cuh"

namespace srl {
namespace {

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ double block_sum_dd(double v, double* red) {
  v = warp_sum_d(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double t = threadIdx.x < (blockDim.x >> 5) ? red[l] : 0.0;
  if (w == 0) {
    t = warp_sum_d(t);
    if (l == 0) red[32] = t;
  }
  __syncthreads();
  return red[32];
}

template <typename In>
__global__ void transpose_kernel(const In* __restrict__ src, const float* __restrict__ row_scale,
                                 int rows, int cols, __nv_bfloat16* __restrict__ dst, int ld) {
  __shared__ float tile[32][33];
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int r = r0 + i, c = c0 + threadIdx.x;
    float v = 0.f;
    if (r < rows && c < cols) {
      if constexpr (sizeof(In) == 2) v = __bfloat162float(src[(size_t)r * cols + c]);
      else v = src[(size_t)r * cols + c];
      if (row_scale) v *= row_scale[r];
    }
    tile[i][threadIdx.x] = v;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int c = c0 + i, r = r0 + threadIdx.x;
    if (r < rows && c < cols) dst[(size_t)c * ld + r] = __float2bfloat16(tile[threadIdx.x][i]);
  }
}

__global__ void f32_to_bf16_kernel(const float* __restrict__ s, size_t n, __nv_bfloat16* __restrict__ d) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    d[i] = __float2bfloat16(s[i]);
}
// 4 elements per step (16-byte loads, 8-byte stores; n % 4 == 0, aligned)
__global__ void f32_to_bf16_x4_kernel(const float4* __restrict__ s, size_t n4, uint2* __restrict__ d) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    const float4 v = s[i];
    const __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
    d[i] = make_uint2(*reinterpret_cast<const uint32_t*>(&a), *reinterpret_cast<const uint32_t*>(&b));
  }
}
__global__ void bf16_to_f32_kernel(const __nv_bfloat16* __restrict__ s, size_t n, float* __restrict__ d) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    d[i] = __bfloat162float(s[i]);
}
// dst[r, :] = bf16(scale[r] * src[r, :]), 8 columns per thread (cols % 8 == 0)
__global__ void scale_rows_kernel(const __nv_bfloat16* __restrict__ src, const float* __restrict__ scale,
                                  int rows, int cols, __nv_bfloat16* __restrict__ dst) {
  const int c8 = cols / 8;
  const size_t n = (size_t)rows * c8;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const float sc = scale[i / c8];
    uint4 v = reinterpret_cast<const uint4*>(src)[i];
    __nv_bfloat16* b = reinterpret_cast<__nv_bfloat16*>(&v);
#pragma unroll
    for (int j = 0; j < 8; ++j) b[j] = __float2bfloat16(sc * __bfloat162float(b[j]));
    reinterpret_cast<uint4*>(dst)[i] = v;
  }
}
__global__ void zero_kernel(float* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = 0.f;
}

constexpr int kRowThreads = 256;

__global__ void __launch_bounds__(kRowThreads)
    loss_dlogits_kernel(const float* __restrict__ logits, const float* __restrict__ pmax,
                        const double* __restrict__ psum, int V, const int32_t* __restrict__ targets,
                        const float* __restrict__ coef, double* __restrict__ logprob,
                        __nv_bfloat16* __restrict__ dlogits) {
  __shared__ float fred[33];
  __shared__ double dred[33];
  const int r = blockIdx.x;
  const int T = (V + 127) / 128;
  const float* pm = pmax + (size_t)r * T;
  const double* ps = psum + (size_t)r * T;
  float mx = -INFINITY;
  for (int t = threadIdx.x; t < T; t += blockDim.x) mx = fmaxf(mx, pm[t]);
  mx = warp_max(mx);
  if ((threadIdx.x & 31) == 0) fred[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? fred[threadIdx.x] : -INFINITY;
    v = warp_max(v);
    if (threadIdx.x == 0) fred[32] = v;
  }
  __syncthreads();
  const double M = (double)fred[32];
  double part = 0.0;
  for (int t = threadIdx.x; t < T; t += blockDim.x) part += ps[t] * exp((double)pm[t] - M);
  const double lse = M + log(block_sum_dd(part, dred));
  const int tgt = targets[r];
  const float* x = logits + (size_t)r * V;
  const float c = coef[r];
  const float lsef = (float)lse;
  for (int v = threadIdx.x; v < V; v += blockDim.x) {
    const float p = __expf(x[v] - lsef);
    dlogits[(size_t)r * V + v] = __float2bfloat16(c * ((v == tgt ? 1.f : 0.f) - p));
  }
  if (threadIdx.x == 0) logprob[r] = (double)x[tgt] - lse;
}

// Per row: lse = log-sum-exp of the LM-head logits from the per-128-column
// (max, fp64 sum) partials (same combination as loss_dlogits_kernel) and
// log pi(target) = logit(target) - lse.
__global__ void __launch_bounds__(kRowThreads)
    lse_logprob_kernel(const float* __restrict__ pmax, const double* __restrict__ psum, int V,
                       const float* __restrict__ tgt_logit, double* __restrict__ lse_out,
                       double* __restrict__ logprob) {
  __shared__ float fred[33];
  __shared__ double dred[33];
  const int r = blockIdx.x;
  const int T = (V + 127) / 128;
  const float* pm = pmax + (size_t)r * T;
  const double* ps = psum + (size_t)r * T;
  float mx = -INFINITY;
  for (int t = threadIdx.x; t < T; t += blockDim.x) mx = fmaxf(mx, pm[t]);
  mx = warp_max(mx);
  if ((threadIdx.x & 31) == 0) fred[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? fred[threadIdx.x] : -INFINITY;
    v = warp_max(v);
    if (threadIdx.x == 0) fred[32] = v;
  }
  __syncthreads();
  const double M = (double)fred[32];
  double part = 0.0;
  for (int t = threadIdx.x; t < T; t += blockDim.x) part += ps[t] * exp((double)pm[t] - M);
  const double lse = M + log(block_sum_dd(part, dred));
  if (threadIdx.x == 0) {
    lse_out[r] = lse;
    logprob[r] = (double)tgt_logit[r] - lse;
  }
}

// One warp per row, float4 loads (H % 4 == 0).
__global__ void row_rstd_kernel(const float* __restrict__ x, int T, int H, float eps,
                                float* __restrict__ rstd) {
  const int lane = threadIdx.x & 31;
  const int H4 = H / 4;
  for (int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < T; r += gridDim.x * (blockDim.x >> 5)) {
    const float4* xr = reinterpret_cast<const float4*>(x + (size_t)r * H);
    float s = 0.f;
    for (int k = lane; k < H4; k += 32) {
      const float4 v = xr[k];
      s += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) rstd[r] = rsqrtf(s / (float)H + eps);
  }
}

// dx += rstd (g * dzw) - rstd^3 / H * (sum_k dzw x g) x, dg += sum_rows rstd dzw x.
// One warp per row (float4, H % 4 == 0); the gain gradient is summed per block
// in shared memory and added to dg once per block.
__global__ void rmsnorm_bwd_kernel(const float* __restrict__ dzw, const float* __restrict__ x,
                                   const __nv_bfloat16* __restrict__ g, const float* __restrict__ rstd,
                                   int T, int H, float* __restrict__ dx, float* __restrict__ dg, int pre) {
  extern __shared__ float s_dg[];
  for (int k = threadIdx.x; k < H; k += blockDim.x) s_dg[k] = 0.f;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int H4 = H / 4;
  for (int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < T; r += gridDim.x * (blockDim.x >> 5)) {
    const float4* dz4 = reinterpret_cast<const float4*>(dzw + (size_t)r * H);
    const float4* x4 = reinterpret_cast<const float4*>(x + (size_t)r * H);
    float4* dx4 = reinterpret_cast<float4*>(dx + (size_t)r * H);
    const float rstd_r = rstd[r];
    const float rs = pre ? 1.f : rstd_r;  // prescaled dzw carries rstd already
    float dr = 0.f;
    for (int k = lane; k < H4; k += 32) {
      const float4 d = dz4[k], v = x4[k];
      const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(g + 4 * k);
      const float2 ga = __bfloat1622float2(g2[0]), gb = __bfloat1622float2(g2[1]);
      dr += d.x * v.x * ga.x + d.y * v.y * ga.y + d.z * v.z * gb.x + d.w * v.w * gb.y;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) dr += __shfl_xor_sync(0xffffffffu, dr, o);
    const float coef = -rstd_r * rstd_r * rs / (float)H * dr;
    for (int k = lane; k < H4; k += 32) {
      const float4 d = dz4[k], v = x4[k];
      const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(g + 4 * k);
      const float2 ga = __bfloat1622float2(g2[0]), gb = __bfloat1622float2(g2[1]);
      float4 o = dx4[k];
      o.x += rs * d.x * ga.x + coef * v.x;
      o.y += rs * d.y * ga.y + coef * v.y;
      o.z += rs * d.z * gb.x + coef * v.z;
      o.w += rs * d.w * gb.y + coef * v.w;
      dx4[k] = o;
      atomicAdd(&s_dg[4 * k], rs * d.x * v.x);
      atomicAdd(&s_dg[4 * k + 1], rs * d.y * v.y);
      atomicAdd(&s_dg[4 * k + 2], rs * d.z * v.z);
      atomicAdd(&s_dg[4 * k + 3], rs * d.w * v.w);
    }
  }
  __syncthreads();
  for (int k = threadIdx.x; k < H; k += blockDim.x) atomicAdd(&dg[k], s_dg[k]);
}

// The same for H <= 32 * 4 * NV: a lane keeps its columns' dz, x, gain and the
// gain-gradient partials in registers (one pass over the row, one shared
// atomic per column per warp instead of one per element).
template <int NV>
__global__ void __launch_bounds__(256)
    rmsnorm_bwd_reg_kernel(const float* __restrict__ dzw, const float* __restrict__ x,
                           const __nv_bfloat16* __restrict__ g, const float* __restrict__ rstd, int T,
                           int H, float* __restrict__ dx, float* __restrict__ dg, int pre) {
  extern __shared__ float s_dg[];
  for (int k = threadIdx.x; k < H; k += blockDim.x) s_dg[k] = 0.f;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int H4 = H / 4;
  float4 gv[NV], acc[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int k = lane + 32 * i;
    acc[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    gv[i] = acc[i];
    if (k < H4) {
      const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(g + 4 * k);
      const float2 ga = __bfloat1622float2(g2[0]), gb = __bfloat1622float2(g2[1]);
      gv[i] = make_float4(ga.x, ga.y, gb.x, gb.y);
    }
  }
  for (int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < T; r += gridDim.x * (blockDim.x >> 5)) {
    const float4* dz4 = reinterpret_cast<const float4*>(dzw + (size_t)r * H);
    const float4* x4 = reinterpret_cast<const float4*>(x + (size_t)r * H);
    float4* dx4 = reinterpret_cast<float4*>(dx + (size_t)r * H);
    const float rstd_r = rstd[r];
    const float rs = pre ? 1.f : rstd_r;
    float4 d[NV], v[NV], o[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int k = lane + 32 * i;
      const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
      d[i] = k < H4 ? dz4[k] : z;
      v[i] = k < H4 ? x4[k] : z;
      o[i] = k < H4 ? dx4[k] : z;
    }
    float dr = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i)
      dr += d[i].x * v[i].x * gv[i].x + d[i].y * v[i].y * gv[i].y + d[i].z * v[i].z * gv[i].z +
            d[i].w * v[i].w * gv[i].w;
#pragma unroll
    for (int s = 16; s; s >>= 1) dr += __shfl_xor_sync(0xffffffffu, dr, s);
    const float coef = -rstd_r * rstd_r * rs / (float)H * dr;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int k = lane + 32 * i;
      if (k >= H4) continue;
      o[i].x += rs * d[i].x * gv[i].x + coef * v[i].x;
      o[i].y += rs * d[i].y * gv[i].y + coef * v[i].y;
      o[i].z += rs * d[i].z * gv[i].z + coef * v[i].z;
      o[i].w += rs * d[i].w * gv[i].w + coef * v[i].w;
      dx4[k] = o[i];
      acc[i].x += rs * d[i].x * v[i].x;
      acc[i].y += rs * d[i].y * v[i].y;
      acc[i].z += rs * d[i].z * v[i].z;
      acc[i].w += rs * d[i].w * v[i].w;
    }
  }
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int k = lane + 32 * i;
    if (k >= H4) continue;
    atomicAdd(&s_dg[4 * k], acc[i].x);
    atomicAdd(&s_dg[4 * k + 1], acc[i].y);
    atomicAdd(&s_dg[4 * k + 2], acc[i].z);
    atomicAdd(&s_dg[4 * k + 3], acc[i].w);
  }
  __syncthreads();
  for (int k = threadIdx.x; k < H; k += blockDim.x) atomicAdd(&dg[k], s_dg[k]);
}

// The same for 1024 < H <= 32 * 4 * NV (1.5B: H = 1536, NV = 12): only the
// gain-gradient partials stay in registers; dz and x are read twice (the
// second pass from L1 / L2) so the kernel runs at ~80 registers, 3 blocks
// (24 warps) per SM -- it is latency-bound, and a register-resident row
// (168 registers, 8 warps per SM) measured no faster than the generic kernel
// above (two passes, a shared atomic per element): 173 vs 166 us per
// 20480-row call at H = 1536.
template <int NV>
__global__ void __launch_bounds__(256, 3)
    rmsnorm_bwd_reg2_kernel(const float* __restrict__ dzw, const float* __restrict__ x,
                            const __nv_bfloat16* __restrict__ g, const float* __restrict__ rstd, int T,
                            int H, float* __restrict__ dx, float* __restrict__ dg, int pre) {
  extern __shared__ float s_dg[];
  for (int k = threadIdx.x; k < H; k += blockDim.x) s_dg[k] = 0.f;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int H4 = H / 4;
  float4 acc[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) acc[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  auto gain = [&](int k) {
    const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(g + 4 * k);
    const float2 ga = __bfloat1622float2(g2[0]), gb = __bfloat1622float2(g2[1]);
    return make_float4(ga.x, ga.y, gb.x, gb.y);
  };
  for (int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < T; r += gridDim.x * (blockDim.x >> 5)) {
    const float4* dz4 = reinterpret_cast<const float4*>(dzw + (size_t)r * H);
    const float4* x4 = reinterpret_cast<const float4*>(x + (size_t)r * H);
    float4* dx4 = reinterpret_cast<float4*>(dx + (size_t)r * H);
    const float rstd_r = rstd[r];
    const float rs = pre ? 1.f : rstd_r;
    float dr = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int k = lane + 32 * i;
      if (k >= H4) continue;
      const float4 d = dz4[k], v = x4[k], gv = gain(k);
      dr += d.x * v.x * gv.x + d.y * v.y * gv.y + d.z * v.z * gv.z + d.w * v.w * gv.w;
    }
#pragma unroll
    for (int s = 16; s; s >>= 1) dr += __shfl_xor_sync(0xffffffffu, dr, s);
    const float coef = -rstd_r * rstd_r * rs / (float)H * dr;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int k = lane + 32 * i;
      if (k >= H4) continue;
      const float4 d = dz4[k], v = x4[k], gv = gain(k);
      float4 o = dx4[k];
      o.x += rs * d.x * gv.x + coef * v.x;
      o.y += rs * d.y * gv.y + coef * v.y;
      o.z += rs * d.z * gv.z + coef * v.z;
      o.w += rs * d.w * gv.w + coef * v.w;
      dx4[k] = o;
      acc[i].x += rs * d.x * v.x;
      acc[i].y += rs * d.y * v.y;
      acc[i].z += rs * d.z * v.z;
      acc[i].w += rs * d.w * v.w;
    }
  }
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int k = lane + 32 * i;
    if (k >= H4) continue;
    atomicAdd(&s_dg[4 * k], acc[i].x);
    atomicAdd(&s_dg[4 * k + 1], acc[i].y);
    atomicAdd(&s_dg[4 * k + 2], acc[i].z);
    atomicAdd(&s_dg[4 * k + 3], acc[i].w);
  }
  __syncthreads();
  for (int k = threadIdx.x; k < H; k += blockDim.x) atomicAdd(&dg[k], s_dg[k]);
}

__global__ void swiglu_bwd_kernel(const float* __restrict__ dact, const __nv_bfloat16* __restrict__ gu,
                                  int T, int I, __nv_bfloat16* __restrict__ dgu,
                                  float* __restrict__ dgu_f32) {
  const size_t n = (size_t)T * I;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n;
       e += (size_t)gridDim.x * blockDim.x) {
    const size_t t = e / I;
    const int j = (int)(e % I);
    const int blk = j >> 6, c = j & 63;
    const size_t gi = t * 2 * I + (size_t)blk * 128 + c, ui = gi + 64;
    const float gv = __bfloat162float(gu[gu_index(t, (size_t)blk * 128 + c, 2 * (size_t)I)]);
    const float uv = __bfloat162float(gu[gu_index(t, (size_t)blk * 128 + c + 64, 2 * (size_t)I)]);
    const float da = dact[e];
    const float sg = 1.f / (1.f + expf(-gv));
    const float silu = gv * sg;
    const float dg = da * uv * (sg * (1.f + gv * (1.f - sg)));
    const float du = da * silu;
    dgu[gi] = __float2bfloat16(dg);
    dgu[ui] = __float2bfloat16(du);
    if (dgu_f32) {
      dgu_f32[gi] = dg;
      dgu_f32[ui] = du;
    }
  }
}

__global__ void swiglu_fwd_kernel(const float* __restrict__ gu, int T, int I,
                                  __nv_bfloat16* __restrict__ act) {
  const size_t n = (size_t)T * I;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n;
       e += (size_t)gridDim.x * blockDim.x) {
    const size_t t = e / I;
    const int j = (int)(e % I);
    const size_t gi = t * 2 * I + (size_t)(j >> 6) * 128 + (j & 63);
    const float g = gu[gi], u = gu[gi + 64];
    act[e] = __float2bfloat16(g / (1.f + expf(-g)) * u);
  }
}

// D[t,h] = sum_d dO[t,h,d] * O[t,h,d]
__global__ void attn_bwd_dot_kernel(const float* __restrict__ d_o, const __nv_bfloat16* __restrict__ o,
                                    int T, int nq, int hd, float* __restrict__ D) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= T * nq) return;
  const size_t base = (size_t)warp * hd;
  float s = 0.f;
  for (int d = lane; d < hd; d += 32) s += d_o[base + d] * __bfloat162float(o[base + d]);
  s = warp_sum(s);
  if (lane == 0) D[warp] = s;
}
// Split bf16 pair (hi | lo per row) of src * row_scale * col_gain, 4 columns per thread.
__global__ void split_bf16_kernel(const float* __restrict__ src, int rows, int cols,
                                  const float* __restrict__ row_scale, const __nv_bfloat16* __restrict__ col_gain,
                                  __nv_bfloat16* __restrict__ dst) {
  const int c4 = cols / 4;
  const size_t n4 = (size_t)rows * c4;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    const int r = (int)(i / c4), c = (int)(i % c4) * 4;
    float4 v = reinterpret_cast<const float4*>(src)[i];
    if (row_scale) {
      const float s = row_scale[r];
      v.x *= s; v.y *= s; v.z *= s; v.w *= s;
    }
    if (col_gain) {
      const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(col_gain + c);
      const float2 ga = __bfloat1622float2(g2[0]), gb = __bfloat1622float2(g2[1]);
      v.x *= ga.x; v.y *= ga.y; v.z *= gb.x; v.w *= gb.y;
    }
    const __nv_bfloat162 h0 = __floats2bfloat162_rn(v.x, v.y), h1 = __floats2bfloat162_rn(v.z, v.w);
    const float2 f0 = __bfloat1622float2(h0), f1 = __bfloat1622float2(h1);
    const __nv_bfloat162 l0 = __floats2bfloat162_rn(v.x - f0.x, v.y - f0.y);
    const __nv_bfloat162 l1 = __floats2bfloat162_rn(v.z - f1.x, v.w - f1.y);
    __nv_bfloat16* row = dst + (size_t)r * 2 * cols + c;
    *reinterpret_cast<__nv_bfloat162*>(row) = h0;
    *reinterpret_cast<__nv_bfloat162*>(row + 2) = h1;
    *reinterpret_cast<__nv_bfloat162*>(row + cols) = l0;
    *reinterpret_cast<__nv_bfloat162*>(row + cols + 2) = l1;
  }
}

// D = rowsum(dO * O) per (row, head) with L = hd / 8 lanes per pair, 8 elements
// per lane (two float4 of dO, one 16-byte load of O); hd in {32, 64, 128, 256}
// o_lo > 0: O is split, rows [hi (nq hd) | lo] (stride nq hd + o_lo), D uses hi + lo.
template <int L>
__global__ void attn_bwd_dot_v_kernel(const float* __restrict__ d_o, const __nv_bfloat16* __restrict__ o,
                                      int pairs, int hd, float* __restrict__ D, int nq, int o_lo,
                                      __nv_bfloat16* __restrict__ dob, __nv_bfloat16* __restrict__ dol) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x, p = t / L, j = t % L;
  float s = 0.f;
  if (p < pairs) {
    const size_t base = (size_t)p * hd + j * 8;
    const size_t obase = o_lo ? (size_t)(p / nq) * (nq * hd + o_lo) + (size_t)(p % nq) * hd + j * 8 : base;
    const float4 a = *reinterpret_cast<const float4*>(d_o + base);
    const float4 b = *reinterpret_cast<const float4*>(d_o + base + 4);
    if (dob) {  // dO as bf16 (+ the lo residual): the attention backward streams it by cp.async
      const float f[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
      uint32_t hw[4], lw[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const __nv_bfloat162 hv = __floats2bfloat162_rn(f[2 * e], f[2 * e + 1]);
        const float2 hf = __bfloat1622float2(hv);
        const __nv_bfloat162 lv = __floats2bfloat162_rn(f[2 * e] - hf.x, f[2 * e + 1] - hf.y);
        hw[e] = *reinterpret_cast<const uint32_t*>(&hv);
        lw[e] = *reinterpret_cast<const uint32_t*>(&lv);
      }
      *reinterpret_cast<uint4*>(dob + base) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
      if (dol) *reinterpret_cast<uint4*>(dol + base) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
    }
    for (int part = 0; part < (o_lo ? 2 : 1); ++part) {
      const uint4 ov = *reinterpret_cast<const uint4*>(o + obase + (part ? o_lo : 0));
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&ov);
      const float2 o0 = __bfloat1622float2(h[0]), o1 = __bfloat1622float2(h[1]), o2 = __bfloat1622float2(h[2]),
                   o3 = __bfloat1622float2(h[3]);
      s += a.x * o0.x + a.y * o0.y + a.z * o1.x + a.w * o1.y + b.x * o2.x + b.y * o2.y + b.z * o3.x + b.w * o3.y;
    }
  }
#pragma unroll
  for (int w = L / 2; w; w >>= 1) s += __shfl_xor_sync(0xffffffffu, s, w);
  if (p < pairs && j == 0) D[p] = s;
}

__device__ __forceinline__ const __nv_bfloat16* kv_row(const __nv_bfloat16* c, const int32_t* bt,
                                                       int pps, int slot, int pos, int nkv, int kh,
                                                       int hd) {
  const int page = bt[(size_t)slot * pps + pos / kPageTokens];
  return c + (((size_t)page * nkv + kh) * kPageTokens + (pos % kPageTokens)) * hd;
}

// dq: one warp per (row t, q head h); lane holds hd/32 dims.
__global__ void attn_bwd_dq_kernel(const __nv_bfloat16* __restrict__ q, const float* __restrict__ d_o,
                                   const float* __restrict__ lse, const float* __restrict__ D,
                                   const __nv_bfloat16* __restrict__ kc,
                                   const __nv_bfloat16* __restrict__ vc,
                                   const int32_t* __restrict__ row_slot,
                                   const int32_t* __restrict__ row_pos,
                                   const int32_t* __restrict__ bt, int pps, int T, int nq, int nkv,
                                   int hd, float scale, float* __restrict__ dqkv) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= T * nq) return;
  const int t = warp / nq, h = warp % nq, kh = h / (nq / nkv);
  const int slot = row_slot[t], pos = row_pos[t];
  const int dpl = hd / 32;
  float qv[4], dov[4], dq[4] = {0.f, 0.f, 0.f, 0.f};
  for (int i = 0; i < dpl; ++i) {
    qv[i] = __bfloat162float(q[((size_t)t * nq + h) * hd + lane * dpl + i]);
    dov[i] = d_o[((size_t)t * nq + h) * hd + lane * dpl + i];
  }
  const float l = lse[(size_t)t * nq + h], Dv = D[(size_t)t * nq + h];
  for (int j = 0; j <= pos; ++j) {
    const __nv_bfloat16* kr = kv_row(kc, bt, pps, slot, j, nkv, kh, hd);
    const __nv_bfloat16* vr = kv_row(vc, bt, pps, slot, j, nkv, kh, hd);
    float s = 0.f, dp = 0.f, kvv[4];
    for (int i = 0; i < dpl; ++i) {
      kvv[i] = __bfloat162float(kr[lane * dpl + i]);
      s += qv[i] * kvv[i];
      dp += dov[i] * __bfloat162float(vr[lane * dpl + i]);
    }
    s = warp_sum(s) * scale;
    dp = warp_sum(dp);
    const float p = __expf(s - l);
    const float ds = p * (dp - Dv) * scale;
    for (int i = 0; i < dpl; ++i) dq[i] += ds * kvv[i];
  }
  const int qkv = (nq + 2 * nkv) * hd;
  for (int i = 0; i < dpl; ++i) dqkv[(size_t)t * qkv + h * hd + lane * dpl + i] = dq[i];
}

// dk, dv: one warp per (row t = the key, kv head kh); loops over the query
// rows of the same sequence at positions >= pos(t) and the G heads.
__global__ void attn_bwd_dkv_kernel(const __nv_bfloat16* __restrict__ q, const float* __restrict__ d_o,
                                    const float* __restrict__ lse, const float* __restrict__ D,
                                    const __nv_bfloat16* __restrict__ kc,
                                    const __nv_bfloat16* __restrict__ vc,
                                    const int32_t* __restrict__ row_slot,
                                    const int32_t* __restrict__ row_pos,
                                    const int32_t* __restrict__ seq_start,
                                    const int32_t* __restrict__ seq_len,
                                    const int32_t* __restrict__ bt, int pps, int T, int nq, int nkv,
                                    int hd, float scale, float* __restrict__ dqkv) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= T * nkv) return;
  const int t = warp / nkv, kh = warp % nkv;
  const int slot = row_slot[t], pos = row_pos[t];
  const int G = nq / nkv, dpl = hd / 32;
  const __nv_bfloat16* kr = kv_row(kc, bt, pps, slot, pos, nkv, kh, hd);
  const __nv_bfloat16* vr = kv_row(vc, bt, pps, slot, pos, nkv, kh, hd);
  float kvv[4], vvv[4], dk[4] = {0.f, 0.f, 0.f, 0.f}, dv[4] = {0.f, 0.f, 0.f, 0.f};
  for (int i = 0; i < dpl; ++i) {
    kvv[i] = __bfloat162float(kr[lane * dpl + i]);
    vvv[i] = __bfloat162float(vr[lane * dpl + i]);
  }
  const int s0 = seq_start[slot], L = seq_len[slot];
  for (int p = pos; p < L; ++p) {
    const int r = s0 + p;
    for (int g = 0; g < G; ++g) {
      const int h = kh * G + g;
      float qv[4], dov[4], s = 0.f, dp = 0.f;
      for (int i = 0; i < dpl; ++i) {
        qv[i] = __bfloat162float(q[((size_t)r * nq + h) * hd + lane * dpl + i]);
        dov[i] = d_o[((size_t)r * nq + h) * hd + lane * dpl + i];
        s += qv[i] * kvv[i];
        dp += dov[i] * vvv[i];
      }
      s = warp_sum(s) * scale;
      dp = warp_sum(dp);
      const float pr = __expf(s - lse[(size_t)r * nq + h]);
      const float ds = pr * (dp - D[(size_t)r * nq + h]) * scale;
      for (int i = 0; i < dpl; ++i) {
        dk[i] += ds * qv[i];
        dv[i] += pr * dov[i];
      }
    }
  }
  const int qkv = (nq + 2 * nkv) * hd;
  for (int i = 0; i < dpl; ++i) {
    dqkv[(size_t)t * qkv + nq * hd + kh * hd + lane * dpl + i] = dk[i];
    dqkv[(size_t)t * qkv + (nq + nkv) * hd + kh * hd + lane * dpl + i] = dv[i];
  }
}

__global__ void rope_bwd_kernel(float* __restrict__ dqkv, const int32_t* __restrict__ row_pos,
                                const float* __restrict__ cs, int nq, int nkv, int hd) {
  const int t = blockIdx.x, half = hd / 2;
  const int pos = row_pos[t];
  float* row = dqkv + (size_t)t * (nq + 2 * nkv) * hd;
  for (int idx = threadIdx.x; idx < (nq + nkv) * half; idx += blockDim.x) {
    const int h = idx / half, j = idx % half;
    const float co = cs[(size_t)pos * hd + j], si = cs[(size_t)pos * hd + half + j];
    const float d1 = row[h * hd + j], d2 = row[h * hd + j + half];
    // forward y1 = x1 c - x2 s, y2 = x2 c + x1 s  =>  dx1 = d1 c + d2 s, dx2 = d2 c - d1 s
    row[h * hd + j] = d1 * co + d2 * si;
    row[h * hd + j + half] = d2 * co - d1 * si;
  }
}

__global__ void colsum_kernel(const float* __restrict__ src, int rows, int cols, float* __restrict__ out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cols) return;
  const int chunk = (rows + gridDim.y - 1) / gridDim.y;
  const int r0 = blockIdx.y * chunk, r1 = min(rows, r0 + chunk);
  float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};  // 8 loads in flight
  int r = r0;
  for (; r + 8 <= r1; r += 8) {
#pragma unroll
    for (int u = 0; u < 8; ++u) a[u] += src[(size_t)(r + u) * cols + c];
  }
  for (; r < r1; ++r) a[0] += src[(size_t)r * cols + c];
  const float s = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
  atomicAdd(&out[c], s);
}

__global__ void embed_bwd_kernel(const float* __restrict__ dx, const int32_t* __restrict__ tokens,
                                 int H, float* __restrict__ dE) {
  const int r = blockIdx.x, tok = tokens[r];
  for (int k = threadIdx.x; k < H; k += blockDim.x) atomicAdd(&dE[(size_t)tok * H + k], dx[(size_t)r * H + k]);
}

__global__ void adam_kernel(float* __restrict__ master, __nv_bfloat16* __restrict__ w,
                            const float* __restrict__ g, float* __restrict__ m, float* __restrict__ v,
                            size_t n, float lr, float b1, float b2, float eps, float bc1, float bc2,
                            float sign) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const float gi = g[i];
    const float mi = b1 * m[i] + (1.f - b1) * gi;
    const float vi = b2 * v[i] + (1.f - b2) * gi * gi;
    m[i] = mi;
    v[i] = vi;
    const float upd = (mi / bc1) / (sqrtf(vi / bc2) + eps);
    const float nw = master[i] + sign * lr * upd;
    master[i] = nw;
    w[i] = __float2bfloat16(nw);
  }
}

// Adam on 4 parameters per step (16-byte fp32 streams, 8-byte bf16 store);
// the same arithmetic as adam_kernel, element by element.
__global__ void adam_x4_kernel(float4* __restrict__ master, uint2* __restrict__ w, const float4* __restrict__ g,
                               float4* __restrict__ m, float4* __restrict__ v, size_t n4, float lr, float b1,
                               float b2, float eps, float bc1, float bc2, float sign) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    const float4 gi = g[i], mo = m[i], vo = v[i], wo = master[i];
    float gg[4] = {gi.x, gi.y, gi.z, gi.w}, mm[4] = {mo.x, mo.y, mo.z, mo.w}, vv[4] = {vo.x, vo.y, vo.z, vo.w},
          ww[4] = {wo.x, wo.y, wo.z, wo.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float mi = b1 * mm[e] + (1.f - b1) * gg[e];
      const float vi = b2 * vv[e] + (1.f - b2) * gg[e] * gg[e];
      mm[e] = mi;
      vv[e] = vi;
      const float upd = (mi / bc1) / (sqrtf(vi / bc2) + eps);
      ww[e] = ww[e] + sign * lr * upd;
    }
    m[i] = make_float4(mm[0], mm[1], mm[2], mm[3]);
    v[i] = make_float4(vv[0], vv[1], vv[2], vv[3]);
    master[i] = make_float4(ww[0], ww[1], ww[2], ww[3]);
    const __nv_bfloat162 a = __floats2bfloat162_rn(ww[0], ww[1]), b = __floats2bfloat162_rn(ww[2], ww[3]);
    w[i] = make_uint2(*reinterpret_cast<const uint32_t*>(&a), *reinterpret_cast<const uint32_t*>(&b));
  }
}

int num_sms() {
  static int n = [] {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

int grid_for(size_t n, int threads) {
  size_t b = (n + threads - 1) / threads;
  return (int)(b > 8192 ? 8192 : (b < 1 ? 1 : b));
}

}  // namespace

void launch_transpose_bf16(const __nv_bfloat16* src, int rows, int cols, __nv_bfloat16* dst,
                           int ld, cudaStream_t st) {
  transpose_kernel<__nv_bfloat16><<<dim3((cols + 31) / 32, (rows + 31) / 32), dim3(32, 8), 0, st>>>(
      src, nullptr, rows, cols, dst, ld);
}
void launch_transpose_f32_bf16(const float* src, int rows, int cols, __nv_bfloat16* dst, int ld,
                               cudaStream_t st) {
  transpose_kernel<float><<<dim3((cols + 31) / 32, (rows + 31) / 32), dim3(32, 8), 0, st>>>(
      src, nullptr, rows, cols, dst, ld);
}
void launch_scale_transpose_bf16(const __nv_bfloat16* src, const float* row_scale, int rows,
                                 int cols, __nv_bfloat16* dst, int ld, cudaStream_t st) {
  transpose_kernel<__nv_bfloat16><<<dim3((cols + 31) / 32, (rows + 31) / 32), dim3(32, 8), 0, st>>>(
      src, row_scale, rows, cols, dst, ld);
}
void launch_swiglu_fwd(const float* gu, int T, int I, __nv_bfloat16* act, cudaStream_t st) {
  swiglu_fwd_kernel<<<grid_for((size_t)T * I, 256), 256, 0, st>>>(gu, T, I, act);
}
void launch_f32_to_bf16(const float* src, size_t n, __nv_bfloat16* dst, cudaStream_t st) {
  if (n % 4 == 0 && (reinterpret_cast<uintptr_t>(src) & 15) == 0 && (reinterpret_cast<uintptr_t>(dst) & 7) == 0) {
    const size_t n4 = n / 4;
    f32_to_bf16_x4_kernel<<<(int)std::min<size_t>((n4 + 255) / 256, (size_t)num_sms() * 16), 256, 0, st>>>(
        reinterpret_cast<const float4*>(src), n4, reinterpret_cast<uint2*>(dst));
    return;
  }
  f32_to_bf16_kernel<<<grid_for(n, 256), 256, 0, st>>>(src, n, dst);
}
void launch_scale_rows_bf16(const __nv_bfloat16* src, const float* row_scale, int rows, int cols,
                            __nv_bfloat16* dst, cudaStream_t st) {
  scale_rows_kernel<<<grid_for((size_t)rows * (cols / 8), 256), 256, 0, st>>>(src, row_scale, rows, cols, dst);
}
void launch_bf16_to_f32(const __nv_bfloat16* src, size_t n, float* dst, cudaStream_t st) {
  bf16_to_f32_kernel<<<grid_for(n, 256), 256, 0, st>>>(src, n, dst);
}
void launch_zero(float* p, size_t n, cudaStream_t st) {
  zero_kernel<<<grid_for(n, 256), 256, 0, st>>>(p, n);
}
void launch_lse_logprob(const float* pmax, const double* psum, int V, int rows, const float* tgt_logit,
                        double* lse, double* logprob, cudaStream_t st) {
  if (rows > 0) lse_logprob_kernel<<<rows, kRowThreads, 0, st>>>(pmax, psum, V, tgt_logit, lse, logprob);
}
void launch_loss_dlogits(const float* logits, const float* pmax, const double* psum, int V,
                         int rows, const int32_t* targets, const float* coef, double* logprob,
                         __nv_bfloat16* dlogits, cudaStream_t st) {
  if (rows > 0)
    loss_dlogits_kernel<<<rows, kRowThreads, 0, st>>>(logits, pmax, psum, V, targets, coef, logprob,
                                                      dlogits);
}
void launch_rmsnorm_bwd(const float* dzw, const float* x, const __nv_bfloat16* g,
                        const float* rstd, int T, int H, float* dx, float* dg, cudaStream_t st,
                        bool prescaled) {
  const int pre = prescaled ? 1 : 0;
  if (T < 1) return;
  const int blocks = std::min((T + 7) / 8, 3 * num_sms());
  const size_t sm = sizeof(float) * H;
  switch ((H / 4 + 31) / 32) {  // float4 columns per lane
    case 1: rmsnorm_bwd_reg_kernel<1><<<blocks, 256, sm, st>>>(dzw, x, g, rstd, T, H, dx, dg, pre); return;
    case 2: rmsnorm_bwd_reg_kernel<2><<<blocks, 256, sm, st>>>(dzw, x, g, rstd, T, H, dx, dg, pre); return;
    case 3: rmsnorm_bwd_reg_kernel<3><<<blocks, 256, sm, st>>>(dzw, x, g, rstd, T, H, dx, dg, pre); return;
    case 4: rmsnorm_bwd_reg_kernel<4><<<blocks, 256, sm, st>>>(dzw, x, g, rstd, T, H, dx, dg, pre); return;
    case 5: rmsnorm_bwd_reg_kernel<5><<<blocks, 256, sm, st>>>(dzw, x, g, rstd, T, H, dx, dg, pre); return;
    case 6: rmsnorm_bwd_reg_kernel<6><<<blocks, 256, sm, st>>>(dzw, x, g, rstd, T, H, dx, dg, pre); return;
    case 7: rmsnorm_bwd_reg_kernel<7><<<blocks, 256, sm, st>>>(dzw, x, g, rstd, T, H, dx, dg, pre); return;
    case 8: rmsnorm_bwd_reg_kernel<8><<<blocks, 256, sm, st>>>(dzw, x, g, rstd, T, H, dx, dg, pre); return;
    case 9: case 10: case 11: case 12:
      rmsnorm_bwd_reg2_kernel<12><<<blocks, 256, sm, st>>>(dzw, x, g, rstd, T, H, dx, dg, pre); return;
    case 13: case 14: case 15: case 16:
      rmsnorm_bwd_reg2_kernel<16><<<blocks, 256, sm, st>>>(dzw, x, g, rstd, T, H, dx, dg, pre); return;
    default: rmsnorm_bwd_kernel<<<blocks, 256, sm, st>>>(dzw, x, g, rstd, T, H, dx, dg, pre);
  }
}
void launch_split_bf16(const float* src, int rows, int cols, const float* row_scale,
                       const __nv_bfloat16* col_gain, __nv_bfloat16* dst, cudaStream_t st) {
  const size_t n4 = (size_t)rows * cols / 4;
  if (n4 == 0) return;
  split_bf16_kernel<<<(int)std::min<size_t>((n4 + 255) / 256, (size_t)num_sms() * 16), 256, 0, st>>>(
      src, rows, cols, row_scale, col_gain, dst);
}
void launch_row_rstd(const float* x, int T, int H, float eps, float* rstd, cudaStream_t st) {
  if (T > 0) row_rstd_kernel<<<(T + 7) / 8, 256, 0, st>>>(x, T, H, eps, rstd);
}
void launch_swiglu_bwd(const float* dact, const __nv_bfloat16* gu, int T, int I, __nv_bfloat16* dgu,
                       float* dgu_f32, cudaStream_t st) {
  swiglu_bwd_kernel<<<grid_for((size_t)T * I, 256), 256, 0, st>>>(dact, gu, T, I, dgu, dgu_f32);
}
void launch_attention_bwd(const __nv_bfloat16* q, const __nv_bfloat16* o, const float* d_o,
                          const float* lse, const __nv_bfloat16* kc, const __nv_bfloat16* vc,
                          const int32_t* row_slot, const int32_t* row_pos,
                          const int32_t* seq_start, const int32_t* seq_len,
                          const int32_t* block_table, int pages_per_seq, int T, int n_seq, int nq,
                          int nkv, int hd, float* dqkv, cudaStream_t st, bool split) {
  float* D = nullptr;
  cudaMallocAsync(&D, sizeof(float) * (size_t)T * nq, st);
  const int w1 = T * nq;
  const int o_lo = split ? nq * hd : 0;  // split: O rows are [hi | lo]
  static const bool scalar = std::getenv("SRL_ATTN_BWD_SCALAR") != nullptr;  // A/B: the CUDA-core path
  const bool tc = (!scalar || split) && (hd == 64 || hd == 128);
  __nv_bfloat16* dob = nullptr;  // dO as bf16 [T x nq x hd] (+ lo), for the tensor-core kernels
  if (tc) cudaMallocAsync(&dob, sizeof(__nv_bfloat16) * (size_t)w1 * hd * (split ? 2 : 1), st);
  __nv_bfloat16* dol = split && dob ? dob + (size_t)w1 * hd : nullptr;
  if (hd == 64)
    attn_bwd_dot_v_kernel<8><<<(w1 * 8 + 255) / 256, 256, 0, st>>>(d_o, o, w1, hd, D, nq, o_lo, dob, dol);
  else if (hd == 128)
    attn_bwd_dot_v_kernel<16><<<(w1 * 16 + 255) / 256, 256, 0, st>>>(d_o, o, w1, hd, D, nq, o_lo, dob, dol);
  else
    attn_bwd_dot_kernel<<<(w1 * 32 + 255) / 256, 256, 0, st>>>(d_o, o, T, nq, hd, D);
  if (tc) {
    launch_attention_bwd_mma(q, dob, dol, lse, D, kc, vc, seq_start, seq_len, block_table, pages_per_seq,
                             n_seq, nq, nkv, hd, dqkv, st, split);
    cudaFreeAsync(dob, st);
  } else {
    const float scale = 1.0f / sqrtf((float)hd);
    const int w2 = T * nkv;
    attn_bwd_dq_kernel<<<(w1 * 32 + 255) / 256, 256, 0, st>>>(q, d_o, lse, D, kc, vc, row_slot, row_pos,
                                                               block_table, pages_per_seq, T, nq, nkv,
                                                               hd, scale, dqkv);
    attn_bwd_dkv_kernel<<<(w2 * 32 + 255) / 256, 256, 0, st>>>(q, d_o, lse, D, kc, vc, row_slot,
                                                                row_pos, seq_start, seq_len,
                                                                block_table, pages_per_seq, T, nq,
                                                                nkv, hd, scale, dqkv);
  }
  cudaFreeAsync(D, st);
}
void launch_rope_bwd(float* dqkv, const int32_t* row_pos, const float* cos_sin, int T, int nq,
                     int nkv, int hd, cudaStream_t st) {
  if (T > 0) rope_bwd_kernel<<<T, 128, 0, st>>>(dqkv, row_pos, cos_sin, nq, nkv, hd);
}
void launch_colsum_accum(const float* src, int rows, int cols, float* out, cudaStream_t st) {
  dim3 grid((cols + 255) / 256, rows > 1024 ? 64 : (rows + 15) / 16);
  colsum_kernel<<<grid, 256, 0, st>>>(src, rows, cols, out);
}
void launch_embed_bwd(const float* dx, const int32_t* tokens, int T, int H, float* dE,
                      cudaStream_t st) {
  if (T > 0) embed_bwd_kernel<<<T, 256, 0, st>>>(dx, tokens, H, dE);
}
void launch_adam(float* master, __nv_bfloat16* w, const float* grad, float* m, float* v, size_t n,
                 float lr, float beta1, float beta2, float eps, float bias1, float bias2,
                 float sign, cudaStream_t st) {
  const bool vec = n % 4 == 0 && ((reinterpret_cast<uintptr_t>(master) | reinterpret_cast<uintptr_t>(grad) |
                                    reinterpret_cast<uintptr_t>(m) | reinterpret_cast<uintptr_t>(v)) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(w) & 7) == 0;
  if (vec) {
    const size_t n4 = n / 4;
    adam_x4_kernel<<<(int)std::min<size_t>((n4 + 255) / 256, (size_t)num_sms() * 16), 256, 0, st>>>(
        reinterpret_cast<float4*>(master), reinterpret_cast<uint2*>(w), reinterpret_cast<const float4*>(grad),
        reinterpret_cast<float4*>(m), reinterpret_cast<float4*>(v), n4, lr, beta1, beta2, eps, bias1, bias2, sign);
    return;
  }
  adam_kernel<<<grid_for(n, 256), 256, 0, st>>>(master, w, grad, m, v, n, lr, beta1, beta2, eps,
                                                bias1, bias2, sign);
}

}  // namespace srl
