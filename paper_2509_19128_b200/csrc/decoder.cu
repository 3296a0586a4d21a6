// decoder.cu -- non-GEMM kernels of a decoder round: weight init/drift,
// embedding + first RMSNorm statistics, RoPE + paged-KV append, causal paged
// GQA attention (split-KV, deterministic combine), last-row gather, the fp64
// log-softmax/SplitMix64 sampler, and device lag statistics.
#include <algorithm>
#include <cfloat>
#include <cstdlib>
#include <cmath>
#include <cstring>

#include "decoder.cuh"
#include "sm100.cuh"

namespace srl {

namespace {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ULL;

__host__ __device__ __forceinline__ uint64_t splitmix_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
// n-th draw (0-based) of SplitMix64(seed): state = seed + (n+1)*golden
// (rng.hpp:18-28); the engine draws exactly one uniform per emitted token.
__device__ __forceinline__ double splitmix_uniform(uint64_t seed, uint64_t n) {
  const uint64_t z = splitmix_mix(seed + (n + 1) * kGolden);
  return (double)(z >> 11) * 0x1.0p-53;
}
// derive_stream(seed, idx) then two draws -> Box-Muller (rng.hpp:39-57).
__device__ __forceinline__ double counter_gaussian(uint64_t seed, uint64_t idx) {
  const uint64_t s0 = splitmix_mix((seed ^ (kGolden * (idx + 1))) + kGolden);
  const double u1 = 1.0 - (double)(splitmix_mix(s0 + kGolden) >> 11) * 0x1.0p-53;
  const double u2 = (double)(splitmix_mix(s0 + 2 * kGolden) >> 11) * 0x1.0p-53;
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586476925286766559 * u2);
}

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

// ------------------------------------------------------------ weights ---
__global__ void init_segment_kernel(__nv_bfloat16* w, size_t n, size_t global_off, uint64_t seed,
                                    double scale, int ones) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    const float v = ones ? 1.0f : (float)(scale * counter_gaussian(seed, global_off + i));
    w[i] = __float2bfloat16(v);
  }
}

__global__ void perturb_kernel(__nv_bfloat16* w, size_t n, uint64_t seed, double mag) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    const float v = __bfloat162float(w[i]) + (float)(mag * counter_gaussian(seed, i));
    w[i] = __float2bfloat16(v);
  }
}

__global__ void rope_table_kernel(float* cs, int max_pos, int hd, double theta) {
  const int half = hd / 2;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < max_pos * half;
       i += gridDim.x * blockDim.x) {
    const int p = i / half, j = i % half;
    const double inv = pow(theta, -2.0 * j / (double)hd);
    const double a = (double)p * inv;
    cs[(size_t)p * hd + j] = (float)cos(a);
    cs[(size_t)p * hd + half + j] = (float)sin(a);
  }
}

// ------------------------------------------------------------- embed ---
__global__ void embed_kernel(const __nv_bfloat16* __restrict__ E, const __nv_bfloat16* __restrict__ g,
                             const int32_t* __restrict__ row_token, int H, int V, float* __restrict__ x,
                             __nv_bfloat16* __restrict__ xg, float* __restrict__ ssq) {
  __shared__ float red[4];
  sm100::griddep_wait();
  const int m = blockIdx.x;
  int tok = row_token[m];
  const bool ok = tok >= 0 && tok < V;
  const int parts = (H + 127) / 128;
  for (int p = 0; p < parts; ++p) {
    const int c = p * 128 + threadIdx.x;
    float v = 0.f;
    if (c < H) {
      v = ok ? __bfloat162float(E[(size_t)tok * H + c]) : 0.f;
      x[(size_t)m * H + c] = v;
      xg[(size_t)m * H + c] = __float2bfloat16(v * __bfloat162float(g[c]));
    }
    float s = warp_sum(v * v);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) ssq[(size_t)m * parts + p] = red[0] + red[1] + red[2] + red[3];
    __syncthreads();
  }
}

// -------------------------------------------------------- rope/append ---
__global__ void rope_append_kernel(const float* __restrict__ qkv, int nq, int nkv, int hd,
                                   const int32_t* __restrict__ row_slot,
                                   const int32_t* __restrict__ row_pos, const float* __restrict__ cs,
                                   const int32_t* __restrict__ block_table, int pages_per_seq,
                                   __nv_bfloat16* __restrict__ kc, __nv_bfloat16* __restrict__ vc,
                                   __nv_bfloat16* __restrict__ q_out) {
  sm100::griddep_wait();
  const int m = blockIdx.x;
  const int slot = row_slot[m];
  if (slot < 0) return;
  const int pos = row_pos[m];
  const int half = hd / 2;
  const int qkv_dim = (nq + 2 * nkv) * hd;
  const float* row = qkv + (size_t)m * qkv_dim;
  const float* c = cs + (size_t)pos * hd;
  const int page = block_table[(size_t)slot * pages_per_seq + pos / kPageTokens];
  const int off = pos % kPageTokens;
  // q and k heads: rotate pairs (j, j + hd/2)
  for (int idx = threadIdx.x; idx < (nq + nkv) * half; idx += blockDim.x) {
    const int h = idx / half, j = idx % half;
    const float x1 = row[h * hd + j], x2 = row[h * hd + j + half];
    const float co = c[j], si = c[half + j];
    const float y1 = x1 * co - x2 * si, y2 = x2 * co + x1 * si;
    if (h < nq) {
      q_out[(size_t)m * nq * hd + h * hd + j] = __float2bfloat16(y1);
      q_out[(size_t)m * nq * hd + h * hd + j + half] = __float2bfloat16(y2);
    } else {
      const int kh = h - nq;
      __nv_bfloat16* dst = kc + (((size_t)page * nkv + kh) * kPageTokens + off) * hd;
      dst[j] = __float2bfloat16(y1);
      dst[j + half] = __float2bfloat16(y2);
    }
  }
  for (int idx = threadIdx.x; idx < nkv * hd; idx += blockDim.x) {
    const int kh = idx / hd, j = idx % hd;
    vc[(((size_t)page * nkv + kh) * kPageTokens + off) * hd + j] =
        __float2bfloat16(row[(nq + nkv) * hd + idx]);
  }
}

// --------------------------------------------------------- attention ---
// One CTA per (row, kv head, key split) -- splits sized by attention_splits;
// 4 warps, each streaming 32-key tiles w, w + 4, ... of the split.  A warp stages its tile's K and V rows (contiguous inside a KV page) with
// coalesced 16-B loads into shared memory, scores all G = nq/nkv query heads
// of the group (lane = key), runs an online softmax per head and accumulates
// P.V with lane = head dims.  Split partials are combined by the last CTA of
// the (row, head) in split order (deterministic).
constexpr int kAttnWarps = 4;
constexpr int kAttnKeyStep = 32 * kAttnWarps;  // a split is a multiple of this many keys
constexpr int kAttnMinChunk = 512;             // smallest split (sizes the merge workspace)
constexpr int kAttnTargetCtas = 600;           // ~1.4 waves of 148 SMs x 3 resident CTAs
// SRL_ATTN_CHUNK: a fixed split size instead of the heuristic (read once)
int attn_chunk_override() {
  static const int c = [] {
    const char* v = std::getenv("SRL_ATTN_CHUNK");
    const int k = v ? std::atoi(v) : 0;
    return k <= 0 ? 0 : std::max(kAttnMinChunk, (k + kAttnKeyStep - 1) / kAttnKeyStep * kAttnKeyStep);
  }();
  return c;
}
__device__ __forceinline__ void att_cp16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
               "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void att_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void att_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void att_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ void att_mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t att_ld32(const void* p) { return *reinterpret_cast<const uint32_t*>(p); }
__device__ __forceinline__ void att_split(float x, float y, uint32_t& hi, uint32_t& lo) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(x, y);
  const float2 hf = __bfloat1622float2(h);
  hi = *reinterpret_cast<const uint32_t*>(&h);
  const __nv_bfloat162 l = __floats2bfloat162_rn(x - hf.x, y - hf.y);
  lo = *reinterpret_cast<const uint32_t*>(&l);
}

template <int G, int HD>
__global__ void __launch_bounds__(32 * kAttnWarps)
    attention_kernel(const __nv_bfloat16* __restrict__ q, int nq, int nkv,
                     const int32_t* __restrict__ row_slot, const int32_t* __restrict__ row_pos,
                     const int32_t* __restrict__ block_table, int pages_per_seq,
                     const __nv_bfloat16* __restrict__ kc, const __nv_bfloat16* __restrict__ vc,
                     float scale, float* __restrict__ ws, int* __restrict__ counters,
                     __nv_bfloat16* __restrict__ out, float* __restrict__ lse_out, int out_lo,
                     int chunk) {
  // S = Q K^T and O = P V on the tensor cores (mma.sync m16n8k16): the G
  // query heads of the KV head are the A rows (padded to 16), each warp one
  // 32-key tile; P enters as hi + lo bf16 halves (fp32-class accuracy)
  constexpr int ROW = HD * 2 + 16;       // padded K / V rows in smem (bytes): conflict-free
  constexpr int V4 = HD / 8;             // uint4 per K/V row
  constexpr int QP = HD + 8;             // bf16 q tile pitch (elements)
  constexpr int NDT = HD / 8;
  extern __shared__ __align__(16) uint8_t att_smem[];
  using SqT = __nv_bfloat16[16][QP];
  using SkT = uint8_t[kAttnWarps][32 * ROW];
  using SvT = uint8_t[kAttnWarps][32 * ROW];
  using SmT = float[kAttnWarps][G];
  using SaT = float[kAttnWarps][G][HD];
  SqT& sq = *reinterpret_cast<SqT*>(att_smem);
  SkT& sk = *reinterpret_cast<SkT*>(att_smem + sizeof(SqT));
  SvT& sv = *reinterpret_cast<SvT*>(att_smem + sizeof(SqT) + sizeof(SkT));
  SmT& sm_m = *reinterpret_cast<SmT*>(att_smem + sizeof(SqT) + sizeof(SkT) + sizeof(SvT));
  SmT& sm_l = *reinterpret_cast<SmT*>(att_smem + sizeof(SqT) + sizeof(SkT) + sizeof(SvT) + sizeof(SmT));
  SaT& sm_acc = *reinterpret_cast<SaT*>(att_smem + sizeof(SqT));  // aliases sk after the tiles
  static_assert(sizeof(SaT) <= sizeof(SkT), "accumulator alias must fit in the K staging area");
  __shared__ int s_last;
  const int m = blockIdx.x, kh = blockIdx.y, split = blockIdx.z, splits = gridDim.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  sm100::griddep_wait();
  const int slot = row_slot[m];
  if (slot < 0) return;  // padding / finished row
  const int ctx = row_pos[m] + 1;
  const int k_begin = split * chunk;
  if (k_begin >= ctx && splits == 1) return;


  float m_lo = -INFINITY, m_hi = -INFINITY, l_lo = 0.f, l_hi = 0.f;  // heads lane/4, lane/4 + 8
  float o[NDT][4];
#pragma unroll
  for (int n = 0; n < NDT; ++n)
#pragma unroll
    for (int i = 0; i < 4; ++i) o[n][i] = 0.f;

  // keys [k_begin, k_end) in 32-key tiles, warp w takes tiles w, w + 4, ...; K and
  // V of a tile are two cp.async groups: the next tile's K streams in under this
  // tile's softmax and P.V, its V under the next Q K^T (online softmax per warp)
  const int k_end = min(ctx, k_begin + chunk);
  const int ntiles = k_end > k_begin ? (k_end - k_begin + 31) / 32 : 0;
  uint8_t* kb = sk[warp];
  uint8_t* vb = sv[warp];
  auto tile_src = [&](int t, const __nv_bfloat16* c) {
    const int t0 = k_begin + t * 32;  // 32 keys inside one 64-token page
    const int page = block_table[(size_t)slot * pages_per_seq + t0 / kPageTokens];
    return reinterpret_cast<const uint4*>(c + (((size_t)page * nkv + kh) * kPageTokens + (t0 % kPageTokens)) * HD);
  };
  auto load_k = [&](int t) {
    const int nv = min(32, k_end - (k_begin + t * 32));
    const uint4* g = tile_src(t, kc);
#pragma unroll
    for (int i = 0; i < V4; ++i) {
      const int e = lane + 32 * i, r = e / V4, c = e % V4;
      if (r < nv) att_cp16(kb + r * ROW + c * 16, g + e);
    }
    att_commit();
  };
  auto load_v = [&](int t) {
    const int nv = min(32, k_end - (k_begin + t * 32));
    const uint4* g = tile_src(t, vc);
#pragma unroll
    for (int i = 0; i < V4; ++i) {
      const int e = lane + 32 * i, r = e / V4, c = e % V4;
      if (r < nv) att_cp16(vb + r * ROW + c * 16, g + e);
      else *reinterpret_cast<uint4*>(vb + r * ROW + c * 16) = make_uint4(0u, 0u, 0u, 0u);  // 0 x NaN is NaN
    }
    att_commit();
  };
  for (int i = threadIdx.x; i < 16 * HD; i += blockDim.x)
    sq[i / HD][i % HD] = i < G * HD ? q[(size_t)m * nq * HD + (kh * G) * HD + i] : __float2bfloat16(0.f);
  if (warp < ntiles) {
    load_k(warp);
    load_v(warp);
  }
  __syncthreads();  // the q tile
  for (int t = warp; t < ntiles; t += kAttnWarps) {
    const int nvalid = min(32, k_end - (k_begin + t * 32));
    const bool has_next = t + kAttnWarps < ntiles;
    att_wait1();  // K(t) landed (V(t) may still be in flight)
    __syncwarp();
    float sc[4][4];
#pragma unroll
    for (int n = 0; n < 4; ++n)
#pragma unroll
      for (int i = 0; i < 4; ++i) sc[n][i] = 0.f;
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk) {
      uint32_t a[4];
      const __nv_bfloat16* qa = &sq[lane >> 2][kk * 16 + (lane & 3) * 2];
      a[0] = att_ld32(qa);
      a[1] = att_ld32(qa + 8 * QP);
      a[2] = att_ld32(qa + 8);
      a[3] = att_ld32(qa + 8 * QP + 8);
#pragma unroll
      for (int n = 0; n < 4; ++n) {
        const uint8_t* kp = kb + (n * 8 + (lane >> 2)) * ROW + (kk * 16 + (lane & 3) * 2) * 2;
        att_mma16816(sc[n], a, att_ld32(kp), att_ld32(kp + 16));
      }
    }
    __syncwarp();
    if (has_next) load_k(t + kAttnWarps);
    float mx_lo = m_lo, mx_hi = m_hi;
#pragma unroll
    for (int n = 0; n < 4; ++n)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int key = n * 8 + (lane & 3) * 2 + (i & 1);
        sc[n][i] = key < nvalid ? sc[n][i] * scale : -INFINITY;
        if (i < 2) mx_lo = fmaxf(mx_lo, sc[n][i]);
        else mx_hi = fmaxf(mx_hi, sc[n][i]);
      }
#pragma unroll
    for (int off = 1; off <= 2; off <<= 1) {
      mx_lo = fmaxf(mx_lo, __shfl_xor_sync(0xffffffffu, mx_lo, off));
      mx_hi = fmaxf(mx_hi, __shfl_xor_sync(0xffffffffu, mx_hi, off));
    }
    const float c_lo = m_lo == -INFINITY ? 0.f : __expf(m_lo - mx_lo);
    const float c_hi = m_hi == -INFINITY ? 0.f : __expf(m_hi - mx_hi);
    m_lo = mx_lo;
    m_hi = mx_hi;
    float sum_lo = 0.f, sum_hi = 0.f;
#pragma unroll
    for (int n = 0; n < 4; ++n)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float pv = sc[n][i] == -INFINITY ? 0.f : __expf(sc[n][i] - (i < 2 ? m_lo : m_hi));
        sc[n][i] = pv;
        if (i < 2) sum_lo += pv;
        else sum_hi += pv;
      }
#pragma unroll
    for (int off = 1; off <= 2; off <<= 1) {
      sum_lo += __shfl_xor_sync(0xffffffffu, sum_lo, off);
      sum_hi += __shfl_xor_sync(0xffffffffu, sum_hi, off);
    }
    l_lo = l_lo * c_lo + sum_lo;
    l_hi = l_hi * c_hi + sum_hi;
#pragma unroll
    for (int n = 0; n < NDT; ++n) {
      o[n][0] *= c_lo; o[n][1] *= c_lo;
      o[n][2] *= c_hi; o[n][3] *= c_hi;
    }
    if (has_next) att_wait1();  // V(t) landed (K(t + 4) may still be in flight)
    else att_wait0();
    __syncwarp();
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      uint32_t ah[4], al[4];
      att_split(sc[2 * ks][0], sc[2 * ks][1], ah[0], al[0]);
      att_split(sc[2 * ks][2], sc[2 * ks][3], ah[1], al[1]);
      att_split(sc[2 * ks + 1][0], sc[2 * ks + 1][1], ah[2], al[2]);
      att_split(sc[2 * ks + 1][2], sc[2 * ks + 1][3], ah[3], al[3]);
#pragma unroll
      for (int n = 0; n < NDT; ++n) {
        uint32_t b0, b1;
        const uint8_t* vp = vb + (ks * 16 + (lane & 15)) * ROW + n * 16;
        asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0, %1}, [%2];"
                     : "=r"(b0), "=r"(b1)
                     : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(vp))));
        att_mma16816(o[n], ah, b0, b1);
        att_mma16816(o[n], al, b0, b1);
      }
    }
    __syncwarp();
    if (has_next) load_v(t + kAttnWarps);
  }
  // combine the warps of this CTA (sm_acc aliases the K tiles: wait for all warps)
  __syncthreads();
  {
    const int h_lo = lane >> 2, h_hi = h_lo + 8;
    if ((lane & 3) == 0) {
      if (h_lo < G) { sm_m[warp][h_lo] = m_lo; sm_l[warp][h_lo] = l_lo; }
      if (h_hi < G) { sm_m[warp][h_hi] = m_hi; sm_l[warp][h_hi] = l_hi; }
    }
#pragma unroll
    for (int n = 0; n < NDT; ++n) {
      const int d = n * 8 + (lane & 3) * 2;
      if (h_lo < G) { sm_acc[warp][h_lo][d] = o[n][0]; sm_acc[warp][h_lo][d + 1] = o[n][1]; }
      if (h_hi < G) { sm_acc[warp][h_hi][d] = o[n][2]; sm_acc[warp][h_hi][d + 1] = o[n][3]; }
    }
  }
  __syncthreads();

  constexpr size_t rec = (size_t)G * (HD + 2);
  // out row stride nq HD + out_lo; split (out_lo > 0): lo = bf16(o - hi) at + out_lo
  auto put_out = [&](int g, int d, float v) {
    const size_t at = (size_t)m * (nq * HD + out_lo) + (kh * G + g) * HD + d;
    const __nv_bfloat16 h = __float2bfloat16(v);
    out[at] = h;
    if (out_lo) out[at + out_lo] = __float2bfloat16(v - __bfloat162float(h));
  };
  float* my_ws = ws + (((size_t)m * nkv + kh) * splits + split) * rec;
  for (int i = threadIdx.x; i < G * HD; i += blockDim.x) {
    const int g = i / HD, d = i % HD;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < kAttnWarps; ++w) M = fmaxf(M, sm_m[w][g]);
    float L = 0.f, A = 0.f;
#pragma unroll
    for (int w = 0; w < kAttnWarps; ++w) {
      const float a = (sm_m[w][g] == -INFINITY) ? 0.f : __expf(sm_m[w][g] - M);
      L += sm_l[w][g] * a;
      A += sm_acc[w][g][d] * a;
    }
    if (splits == 1) {
      put_out(g, d, L > 0.f ? A / L : 0.f);
      if (lse_out != nullptr && d == 0) lse_out[(size_t)m * nq + kh * G + g] = M + logf(L);
    } else {
      my_ws[g * (HD + 2) + 2 + d] = A;
      if (d == 0) {
        my_ws[g * (HD + 2)] = M;
        my_ws[g * (HD + 2) + 1] = L;
      }
    }
  }
  if (splits == 1) return;
  __threadfence();
  __syncthreads();
  const int cidx = m * nkv + kh;
  if (threadIdx.x == 0) s_last = (atomicAdd(&counters[cidx], 1) == splits - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const float* base = ws + ((size_t)m * nkv + kh) * splits * rec;
  const int used = min(splits, (ctx + chunk - 1) / chunk);  // later splits are empty
  for (int i = threadIdx.x; i < G * HD; i += blockDim.x) {
    const int g = i / HD, d = i % HD;
    float M = -INFINITY;
    for (int sp2 = 0; sp2 < used; ++sp2) M = fmaxf(M, __ldcg(&base[sp2 * rec + g * (HD + 2)]));
    float L = 0.f, A = 0.f;
    for (int sp2 = 0; sp2 < used; ++sp2) {
      const float ms = __ldcg(&base[sp2 * rec + g * (HD + 2)]);
      const float a = (ms == -INFINITY) ? 0.f : __expf(ms - M);
      L += __ldcg(&base[sp2 * rec + g * (HD + 2) + 1]) * a;
      A += __ldcg(&base[sp2 * rec + g * (HD + 2) + 2 + d]) * a;
    }
    put_out(g, d, L > 0.f ? A / L : 0.f);
    if (lse_out != nullptr && d == 0) lse_out[(size_t)m * nq + kh * G + g] = M + logf(L);
  }
  if (threadIdx.x == 0) counters[cidx] = 0;
}

// Key splits of a launch.  Few long splits beat many short ones (each split
// pays the q load, the first tile's latency and the workspace merge): as few
// as give ~kAttnTargetCtas CTAs, none shorter than kAttnMinChunk keys.
// 7B, 256 rows x 4 KV heads, 1088-key contexts: one split (merge-free) --
// attention 3.31 -> 2.07 ms per round against 512-key splits.
int attention_splits(const DecoderDims& d, int M, int max_ctx) {
  const int most = std::max(1, (max_ctx + kAttnMinChunk - 1) / kAttnMinChunk);
  if (const int c = attn_chunk_override()) return std::min(most, std::max(1, (max_ctx + c - 1) / c));
  const int units = std::max(1, M * d.nkv);
  return std::min(most, std::max(1, (kAttnTargetCtas + units - 1) / units));
}
// keys per split for `splits` splits (a multiple of kAttnKeyStep)
static int attention_chunk(int max_ctx, int splits) {
  const int c = (max_ctx + splits - 1) / splits;
  return std::max(kAttnKeyStep, (c + kAttnKeyStep - 1) / kAttnKeyStep * kAttnKeyStep);
}

// ------------------------------------------------------------- gather ---
__global__ void gather_rows_kernel(const __nv_bfloat16* __restrict__ xg, const float* __restrict__ ssq,
                                   const int32_t* __restrict__ last_row, int H, int parts,
                                   __nv_bfloat16* __restrict__ xg_out, float* __restrict__ ssq_out) {
  sm100::griddep_wait();
  const int s = blockIdx.x;
  const int r = last_row[s];
  for (int c = threadIdx.x; c < H; c += blockDim.x)
    xg_out[(size_t)s * H + c] = r >= 0 ? xg[(size_t)r * H + c] : __float2bfloat16(0.f);
  for (int p = threadIdx.x; p < parts; p += blockDim.x)
    ssq_out[(size_t)s * parts + p] = r >= 0 ? ssq[(size_t)r * parts + p] : 1.f;
}

// ------------------------------------------------------------- sample ---
constexpr int kSampleThreads = 512;

__device__ double block_sum_d(double v, double* red) {
  // fixed-order reduction: warp tree, then warp 0 over the 32 warp sums
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double t = (threadIdx.x < (blockDim.x >> 5)) ? red[l] : 0.0;  // only warps that exist
  if (w == 0) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (l == 0) red[32] = t;
  }
  __syncthreads();
  return red[32];
}

constexpr int kTile = 128;  // LM-head GEMM tile width (columns per partial)

struct SampleShared {
  double red[33];
  float fred[32];
  int ired[32];
  double scan[kSampleThreads];
  int tile;
  int tok;
};

// Per (row, 128-column tile): max and fp64 sum of exp(x - max).  The LM-head
// GEMM epilogue (EPI_LOGITS) produces the same statistics; this kernel serves
// raw logits handed to srl_kernel_sample_logits.
__global__ void tile_stats_kernel(const float* __restrict__ logits, int V, float* __restrict__ pmax,
                                  double* __restrict__ psum) {
  const int row = blockIdx.y, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int T = (V + kTile - 1) / kTile;
  const int t = blockIdx.x * (blockDim.x >> 5) + warp;
  if (t >= T) return;
  const float* x = logits + (size_t)row * V + (size_t)t * kTile;
  float v[4];
  float mx = -INFINITY;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int k = t * kTile + lane * 4 + i;
    v[i] = k < V ? x[lane * 4 + i] : -INFINITY;
    mx = fmaxf(mx, v[i]);
  }
  mx = warp_max(mx);
  double s = 0.0;
  if (mx != -INFINITY)
    for (int i = 0; i < 4; ++i) s += exp((double)v[i] - (double)mx);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) {
    pmax[(size_t)row * T + t] = mx;
    psum[(size_t)row * T + t] = s;
  }
}

// Block-wide sampling of one logits row from its tile partials.
//   lse = M + log(sum_t s_t * exp(m_t - M))                 (numeric.hpp:13-20)
//   tile masses q_t = s_t * exp(m_t - lse), inclusive scan over thread chunks
//   the first tile whose walk may cross u is walked element by element with
//   p_k = exp(x_k - lse) in fp64: the inverse CDF of rng.hpp:61-69 with a
//   fixed-order (tile, lane) summation; rounding slack past the last element
//   falls back to V-1 like the reference.
// Greedy: argmax over the row, lowest index on ties.
__device__ int sample_row(const float* __restrict__ x, int V, const float* __restrict__ pmax,
                          const double* __restrict__ psum, double u, int greedy, SampleShared& sh,
                          double* lse_out) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int T = (V + kTile - 1) / kTile;
  const int C = (T + kSampleThreads - 1) / kSampleThreads;  // tiles per thread (contiguous)
  const int t0 = tid * C, t1 = min(T, t0 + C);
  float mx = -INFINITY;
  int mt = 0x7fffffff;
  for (int t = t0; t < t1; ++t) {
    const float v = pmax[t];
    if (v > mx) { mx = v; mt = t; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float om = __shfl_xor_sync(0xffffffffu, mx, o);
    const int oi = __shfl_xor_sync(0xffffffffu, mt, o);
    if (om > mx || (om == mx && oi < mt)) { mx = om; mt = oi; }
  }
  if (lane == 0) { sh.fred[warp] = mx; sh.ired[warp] = mt; }
  __syncthreads();
  if (tid < 32) {
    mx = tid < kSampleThreads / 32 ? sh.fred[tid] : -INFINITY;
    mt = tid < kSampleThreads / 32 ? sh.ired[tid] : 0x7fffffff;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float om = __shfl_xor_sync(0xffffffffu, mx, o);
      const int oi = __shfl_xor_sync(0xffffffffu, mt, o);
      if (om > mx || (om == mx && oi < mt)) { mx = om; mt = oi; }
    }
    if (tid == 0) { sh.fred[0] = mx; sh.ired[0] = mt; }
  }
  __syncthreads();
  const float Mf = sh.fred[0];
  const double M = (double)Mf;
  const int mtile = sh.ired[0];
  double part = 0.0;
  for (int t = t0; t < t1; ++t) part += psum[t] * exp((double)pmax[t] - M);
  const double lse = M + log(block_sum_d(part, sh.red));
  *lse_out = lse;

  if (greedy) {  // first element equal to the max inside the first max tile
    if (warp == 0) {
      int best = 0x7fffffff;
      for (int i = lane; i < kTile; i += 32) {
        const int k = mtile * kTile + i;
        if (k < V && x[k] == Mf) best = min(best, k);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
      if (lane == 0) sh.tok = best == 0x7fffffff ? mtile * kTile : best;
    }
    __syncthreads();
    return sh.tok;
  }

  double mass = 0.0;
  for (int t = t0; t < t1; ++t) mass += psum[t] * exp((double)pmax[t] - lse);
  sh.scan[tid] = mass;
  __syncthreads();
  for (int o = 1; o < kSampleThreads; o <<= 1) {  // Hillis-Steele, fixed order
    const double add = tid >= o ? sh.scan[tid - o] : 0.0;
    __syncthreads();
    sh.scan[tid] += add;
    __syncthreads();
  }
  // first tile whose [base, base + mass + margin) may contain u
  int cand = 0x7fffffff;
  {
    double base = tid == 0 ? 0.0 : sh.scan[tid - 1];
    if (u < sh.scan[tid] + 1e-12) {
      for (int t = t0; t < t1; ++t) {
        const double q = psum[t] * exp((double)pmax[t] - lse);
        if (u < base + q + 1e-12) { cand = t; break; }
        base += q;
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cand = min(cand, __shfl_xor_sync(0xffffffffu, cand, o));
  __syncthreads();
  if (lane == 0) sh.ired[warp] = cand;
  __syncthreads();
  if (tid < 32) {
    int c = tid < kSampleThreads / 32 ? sh.ired[tid] : 0x7fffffff;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c = min(c, __shfl_xor_sync(0xffffffffu, c, o));
    if (tid == 0) sh.tile = c;
  }
  __syncthreads();
  // warp 0 walks from the candidate tile; base = prefix of tile masses in the
  // same (thread chunk, tile) order as the scan
  if (warp == 0) {
    int tok = V - 1;
    int t = sh.tile;
    if (t != 0x7fffffff) {
      const int owner = t / C;
      double base = owner == 0 ? 0.0 : sh.scan[owner - 1];
      for (int tt = owner * C; tt < t; ++tt) base += psum[tt] * exp((double)pmax[tt] - lse);
      bool done = false;
      for (; t < T && !done; ++t) {
        double p[4];
        double ls = 0.0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int k = t * kTile + lane * 4 + i;
          p[i] = k < V ? exp((double)x[k] - lse) : 0.0;
          ls += p[i];
        }
        double incl = ls;  // inclusive warp scan of lane sums (fixed order)
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const double n = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += n;
        }
        double cum = base + (incl - ls);
        int found = 0x7fffffff;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          cum += p[i];
          const int k = t * kTile + lane * 4 + i;
          if (found == 0x7fffffff && k < V && u < cum) found = k;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) found = min(found, __shfl_xor_sync(0xffffffffu, found, o));
        if (found != 0x7fffffff) {
          tok = found;
          done = true;
        }
        base += __shfl_sync(0xffffffffu, incl, 31);
      }
    }
    if (lane == 0) sh.tok = tok;
  }
  __syncthreads();
  return sh.tok;
}

__global__ void __launch_bounds__(kSampleThreads)
    sample_kernel(const float* __restrict__ logits, const float* __restrict__ pmax,
                  const double* __restrict__ psum, int V, int slots, RoundPlan plan,
                  RoundPlan next, SlotState ss, EventRing ring, const int32_t* __restrict__ round_ctr,
                  const int32_t* __restrict__ version, int greedy) {
  __shared__ SampleShared sh;
  sm100::griddep_wait();
  const int s = blockIdx.x;
  const int tid = threadIdx.x;
  const int ri = (*round_ctr - 1) % ring.rounds;
  const size_t ev = (size_t)ri * slots + s;
  const int r = plan.last_row[s];
  if (r < 0 || ss.live[s] == 0) {
    if (tid == 0) {
      ring.ev[ev].flag = 0;
      next.row_slot[s] = -1;
      next.last_row[s] = -1;
      next.row_pos[s] = 0;
      next.row_token[s] = 0;
    }
    return;
  }
  const float* x = logits + (size_t)s * V;
  const int T = (V + kTile - 1) / kTile;
  const double u = splitmix_uniform(ss.seed[s], (uint64_t)ss.gen_count[s]);
  double lse;
  const int tok = sample_row(x, V, pmax + (size_t)s * T, psum + (size_t)s * T, u, greedy, sh, &lse);

  if (tid == 0) {
    const int pos_row = plan.row_pos[r];
    const int new_len = pos_row + 1;
    const int gen = ss.gen_count[s];
    int flag = 1;
    if (tok == ss.terminator[s]) flag = 3;                    // Terminator (engine.cpp:146)
    else if (gen + 1 >= ss.max_tokens[s]) flag = 2;           // Length (engine.cpp:148)
    else if (new_len + 1 > ss.max_seq) flag = 2;              // KV capacity (guarded at open)
    DevEvent e;
    e.flag = flag;
    e.token = tok;
    e.position = gen;
    e.version = *version;
    e.logprob = (double)x[tok] - lse;
    ring.ev[ev] = e;
    ss.seq_len[s] = new_len;
    ss.gen_count[s] = gen + 1;
    if (new_len < ss.max_seq) ss.history[(size_t)s * ss.max_seq + new_len] = tok;
    const int alive = flag == 1;
    ss.live[s] = alive;
    next.row_slot[s] = alive ? s : -1;
    next.row_pos[s] = new_len;
    next.row_token[s] = tok;
    next.last_row[s] = alive ? s : -1;
  }
}


// log pi(target | row) = logit[target] - logsumexp(row), fp64 (rl_math.cpp:128-142)
__global__ void __launch_bounds__(kSampleThreads)
    row_logprobs_kernel(const float* __restrict__ logits, int V, const int32_t* __restrict__ targets,
                        double* __restrict__ out) {
  __shared__ double red[33];
  __shared__ float fred[32];
  const int row = blockIdx.x, tid = threadIdx.x;
  const float* x = logits + (size_t)row * V;
  float mx = -INFINITY;
  for (int k = tid; k < V; k += kSampleThreads) mx = fmaxf(mx, x[k]);
  mx = warp_max(mx);
  if ((tid & 31) == 0) fred[tid >> 5] = mx;
  __syncthreads();
  if (tid < 32) {
    float v = warp_max(tid < (kSampleThreads >> 5) ? fred[tid] : -INFINITY);
    if (tid == 0) fred[0] = v;
  }
  __syncthreads();
  const double M = (double)fred[0];
  double part = 0.0;
  for (int k = tid; k < V; k += kSampleThreads) part += exp((double)x[k] - M);
  const double lse = M + log(block_sum_d(part, red));
  if (tid == 0) out[row] = (double)x[targets[row]] - lse;
}

// Exact categorical KL(p || q) per row from two logits rows (numeric.hpp:34-46:
// terms with p = 0 skipped, +inf where q has no support, clamped at 0); fp64
// log-sum-exp of both rows, fp64 accumulation.
__global__ void __launch_bounds__(kSampleThreads)
    row_kl_kernel(const float* __restrict__ lp, const float* __restrict__ lq, int V, double* __restrict__ out) {
  __shared__ double red[33];
  __shared__ float fred[32];
  const int row = blockIdx.x, tid = threadIdx.x;
  const float* x = lp + (size_t)row * V;
  const float* y = lq + (size_t)row * V;
  double lse[2];
  for (int side = 0; side < 2; ++side) {
    const float* z = side ? y : x;
    float mx = -INFINITY;
    for (int k = tid; k < V; k += kSampleThreads) mx = fmaxf(mx, z[k]);
    mx = warp_max(mx);
    if ((tid & 31) == 0) fred[tid >> 5] = mx;
    __syncthreads();
    if (tid < 32) {
      float v = warp_max(tid < (kSampleThreads >> 5) ? fred[tid] : -INFINITY);
      if (tid == 0) fred[0] = v;
    }
    __syncthreads();
    const double M = (double)fred[0];
    __syncthreads();
    double part = 0.0;
    for (int k = tid; k < V; k += kSampleThreads) part += exp((double)z[k] - M);
    lse[side] = M + log(block_sum_d(part, red));
  }
  double part = 0.0;
  int inf = 0;
  for (int k = tid; k < V; k += kSampleThreads) {
    const double a = (double)x[k] - lse[0], b = (double)y[k] - lse[1];
    const double p = exp(a);
    if (p == 0.0) continue;
    if (!isfinite(b)) inf = 1;
    part += p * (a - b);
  }
  const int any_inf = __syncthreads_or(inf);
  const double kl = block_sum_d(part, red);
  if (tid == 0) out[row] = any_inf ? INFINITY : fmax(kl, 0.0);
}

__global__ void __launch_bounds__(kSampleThreads)
    sample_logits_kernel(const float* __restrict__ logits, const float* __restrict__ pmax,
                         const double* __restrict__ psum, int V, const uint64_t* __restrict__ seeds,
                         const int32_t* __restrict__ draw, int greedy, int32_t* __restrict__ tok_out,
                         double* __restrict__ lp_out) {
  __shared__ SampleShared sh;
  const int r = blockIdx.x;
  const float* x = logits + (size_t)r * V;
  const int T = (V + kTile - 1) / kTile;
  const double u = splitmix_uniform(seeds[r], (uint64_t)draw[r]);
  double lse;
  const int tok = sample_row(x, V, pmax + (size_t)r * T, psum + (size_t)r * T, u, greedy, sh, &lse);
  if (threadIdx.x == 0) {
    tok_out[r] = tok;
    lp_out[r] = (double)x[tok] - lse;
  }
}

__global__ void plan_copy_kernel(RoundPlan dst, RoundPlan src, int rows, int slots,
                                 int32_t* round_ctr) {
  sm100::griddep_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0) *round_ctr += 1;
  if (i < rows) {
    dst.row_slot[i] = src.row_slot[i];
    dst.row_pos[i] = src.row_pos[i];
    dst.row_token[i] = src.row_token[i];
  }
  if (i < slots) dst.last_row[i] = src.last_row[i];
}

// ---------------------------------------------------------------- lag ---
__global__ void lag_stats_kernel(const int32_t* __restrict__ versions,
                                 const int64_t* __restrict__ offs, int version_before,
                                 unsigned long long* __restrict__ hist, int cap,
                                 int64_t* __restrict__ seq_sums, unsigned long long* __restrict__ totals) {
  __shared__ unsigned long long red[32];
  __shared__ int red_max[32];
  const int sidx = blockIdx.x;
  const int64_t b = offs[sidx], e = offs[sidx + 1];
  unsigned long long sum = 0;
  int mx = 0, bad = 0;
  for (int64_t t = b + threadIdx.x; t < e; t += blockDim.x) {
    const int lag = version_before - versions[t];
    if (lag < 0 || lag >= cap) { bad = 1; continue; }
    atomicAdd(&hist[lag], 1ull);
    sum += (unsigned long long)lag;
    mx = max(mx, lag);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sum += __shfl_xor_sync(0xffffffffu, sum, o);
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    bad |= __shfl_xor_sync(0xffffffffu, bad, o);
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
  if (l == 0) { red[w] = sum; red_max[w] = mx | (bad << 30); }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long s2 = 0;
    int m2 = 0, b2 = 0;
    for (int i = 0; i < nw; ++i) {
      s2 += red[i];
      m2 = max(m2, red_max[i] & ~(1 << 30));
      b2 |= red_max[i] >> 30;
    }
    seq_sums[sidx] = (int64_t)s2;
    atomicAdd(&totals[0], (unsigned long long)(e - b));
    atomicAdd(&totals[1], s2);
    atomicMax(&totals[2], (unsigned long long)m2);
    if (b2) atomicAdd(&totals[3], 1ull);
  }
}

}  // namespace

// ----------------------------------------------------------- host side ---
DecoderDims dims_from(const srl_decoder_config& c) {
  DecoderDims d;
  d.V = c.vocab_size; d.H = c.hidden; d.L = c.layers; d.nq = c.q_heads; d.nkv = c.kv_heads;
  d.hd = c.head_dim; d.I = c.intermediate; d.tie = c.tie_embeddings; d.bos = c.bos_token;
  d.max_pos = c.max_positions; d.theta = (float)c.rope_theta; d.eps = (float)c.rms_eps;
  return d;
}

bool dims_valid(const DecoderDims& d, const char** why) {
  auto fail = [&](const char* w) { if (why) *why = w; return false; };
  if (d.V < 1 || d.H < 64 || d.L < 1 || d.nq < 1 || d.nkv < 1 || d.I < 64) return fail("non-positive dims");
  if (d.H % 64 || d.I % 64) return fail("hidden and intermediate must be multiples of 64");
  if (d.hd != 64 && d.hd != 128) return fail("head_dim must be 64 or 128");
  if (d.nq % d.nkv || d.nq / d.nkv > 8) return fail("q_heads / kv_heads must be an integer <= 8");
  if ((d.nq * d.hd) % 64) return fail("q_heads * head_dim must be a multiple of 64");
  if (d.bos < 0 || d.bos >= d.V) return fail("bos_token out of vocab");
  if (d.max_pos < 2) return fail("max_positions must be >= 2");
  return true;
}

size_t make_layout(const DecoderDims& d, WeightLayout& out) {
  size_t cur = 0;
  auto take = [&](size_t n) {
    const size_t at = cur;
    cur += (n + 63) / 64 * 64;  // 128-byte alignment of every tensor
    return at;
  };
  out.embed = take((size_t)d.V * d.H);
  out.layers = new LayerOffsets[d.L];
  for (int l = 0; l < d.L; ++l) {
    LayerOffsets& o = out.layers[l];
    o.ln1 = take(d.H);
    o.qkv_w = take((size_t)d.qkv() * d.H);
    o.qkv_b = take(d.qkv());
    o.o_w = take((size_t)d.H * d.qdim());
    o.ln2 = take(d.H);
    o.gate_up_w = take((size_t)2 * d.I * d.H);
    o.down_w = take((size_t)d.H * d.I);
  }
  out.final_norm = take(d.H);
  out.lm_head = d.tie ? out.embed : take((size_t)d.V * d.H);
  out.total = cur;
  return cur;
}

void launch_init_weights(__nv_bfloat16* w, const DecoderDims& d, const WeightLayout& lay,
                         uint64_t seed, double scale, cudaStream_t st) {
  cudaMemsetAsync(w, 0, lay.total * sizeof(__nv_bfloat16), st);
  auto seg = [&](size_t off, size_t n, int ones) {
    const int blocks = (int)std::min<size_t>((n + 255) / 256, 4096);
    init_segment_kernel<<<blocks, 256, 0, st>>>(w + off, n, off, seed, scale, ones);
  };
  seg(lay.embed, (size_t)d.V * d.H, 0);
  for (int l = 0; l < d.L; ++l) {
    const LayerOffsets& o = lay.layers[l];
    seg(o.ln1, d.H, 1);
    seg(o.qkv_w, (size_t)d.qkv() * d.H, 0);
    seg(o.qkv_b, d.qkv(), 0);
    seg(o.o_w, (size_t)d.H * d.qdim(), 0);
    seg(o.ln2, d.H, 1);
    seg(o.gate_up_w, (size_t)2 * d.I * d.H, 0);
    seg(o.down_w, (size_t)d.H * d.I, 0);
  }
  seg(lay.final_norm, d.H, 1);
  if (!d.tie) seg(lay.lm_head, (size_t)d.V * d.H, 0);
}

void launch_perturb(__nv_bfloat16* w, size_t n, uint64_t seed, double magnitude, cudaStream_t st) {
  const int blocks = (int)std::min<size_t>((n + 255) / 256, 8192);
  perturb_kernel<<<blocks, 256, 0, st>>>(w, n, seed, magnitude);
}

void launch_rope_table(float* cs, int max_pos, int hd, double theta, cudaStream_t st) {
  const int n = max_pos * hd / 2;
  rope_table_kernel<<<(n + 255) / 256, 256, 0, st>>>(cs, max_pos, hd, theta);
}

void launch_embed(const __nv_bfloat16* embed, const __nv_bfloat16* gain, const int32_t* row_token,
                  int M, int H, int V, float* x, __nv_bfloat16* xg, float* ssq, cudaStream_t st) {
  // rows with an out-of-range token (padding / finished slots) embed to zero
  launch_pdl(embed_kernel, dim3(M), dim3(128), 0, st, dim3(1, 1, 1), embed, gain, row_token, H, V,
             x, xg, ssq);
}

void launch_rope_append(const float* qkv, const DecoderDims& d, const RoundPlan& plan, int M,
                        const float* cos_sin, const int32_t* block_table, int pages_per_seq,
                        __nv_bfloat16* kc, __nv_bfloat16* vc, __nv_bfloat16* q_out,
                        cudaStream_t st) {
  launch_pdl(rope_append_kernel, dim3(M), dim3(128), 0, st, dim3(1, 1, 1), qkv, d.nq, d.nkv, d.hd,
             (const int32_t*)plan.row_slot, (const int32_t*)plan.row_pos, cos_sin, block_table,
             pages_per_seq, kc, vc, q_out);
}

size_t attention_ws_floats(const DecoderDims& d, int M, int max_ctx) {
  // any launch of <= M rows: at most one split per kAttnMinChunk keys
  const int splits = std::max(1, (max_ctx + kAttnMinChunk - 1) / kAttnMinChunk);
  return (size_t)M * d.nkv * splits * (d.nq / d.nkv) * (d.hd + 2);
}

template <int G, int HD>
constexpr size_t attention_smem() {
  // bf16 q tile [16][HD + 8], K and V tiles (padded rows), m, l: 74 KB at hd 128, three CTAs
  // per SM (with the unused P area of the CUDA-core version it was 78 KB, two CTAs: the 7B
  // batch-256 decode attention ran at 27% of the HBM peak, 12% warps active)
  return sizeof(__nv_bfloat16) * 16 * (HD + 8) + 2 * (size_t)kAttnWarps * 32 * (HD * 2 + 16) +
         2 * sizeof(float) * kAttnWarps * G;
}

template <int G, int HD>
void attention_launch_t(dim3 grid, cudaStream_t st, const __nv_bfloat16* q, int nq, int nkv,
                        const RoundPlan& plan, const int32_t* bt, int pps, const __nv_bfloat16* kc,
                        const __nv_bfloat16* vc, float scale, float* ws, int* counters,
                        __nv_bfloat16* out, float* lse_out, int out_lo, int chunk) {
  constexpr size_t smem = attention_smem<G, HD>();
  static bool once = [] {
    cudaFuncSetAttribute(attention_kernel<G, HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    return true;
  }();
  (void)once;
  launch_pdl(attention_kernel<G, HD>, grid, dim3(32 * kAttnWarps), smem, st, dim3(1, 1, 1), q, nq,
             nkv, (const int32_t*)plan.row_slot, (const int32_t*)plan.row_pos, bt, pps, kc, vc,
             scale, ws, counters, out, lse_out, out_lo, chunk);
}

template <int HD>
void attention_dispatch_g(int G, dim3 grid, cudaStream_t st, const __nv_bfloat16* q, int nq,
                          int nkv, const RoundPlan& plan, const int32_t* bt, int pps,
                          const __nv_bfloat16* kc, const __nv_bfloat16* vc, float scale, float* ws,
                          int* counters, __nv_bfloat16* out, float* lse_out, int out_lo, int chunk) {
  switch (G) {
#define SRL_ATTN_G(g) \
  case g: attention_launch_t<g, HD>(grid, st, q, nq, nkv, plan, bt, pps, kc, vc, scale, ws, counters, out, lse_out, out_lo, chunk); break;
    SRL_ATTN_G(1) SRL_ATTN_G(2) SRL_ATTN_G(3) SRL_ATTN_G(4)
    SRL_ATTN_G(5) SRL_ATTN_G(6) SRL_ATTN_G(7) SRL_ATTN_G(8)
#undef SRL_ATTN_G
    default: break;
  }
}

void launch_attention(const __nv_bfloat16* q, const DecoderDims& d, const RoundPlan& plan, int M,
                      const int32_t* block_table, int pages_per_seq, const __nv_bfloat16* kc,
                      const __nv_bfloat16* vc, int max_ctx, float* ws, int* counters,
                      size_t ws_floats, __nv_bfloat16* out, cudaStream_t st, float* lse_out, int out_lo) {
  const int splits = attention_splits(d, M, max_ctx);
  const int chunk = attention_chunk(max_ctx, splits);
  (void)ws_floats;
  dim3 grid(M, d.nkv, splits);
  const float scale = 1.0f / sqrtf((float)d.hd);
  const int G = d.nq / d.nkv;
  if (d.hd == 64)
    attention_dispatch_g<64>(G, grid, st, q, d.nq, d.nkv, plan, block_table, pages_per_seq, kc,
                             vc, scale, ws, counters, out, lse_out, out_lo, chunk);
  else
    attention_dispatch_g<128>(G, grid, st, q, d.nq, d.nkv, plan, block_table, pages_per_seq, kc,
                              vc, scale, ws, counters, out, lse_out, out_lo, chunk);
}

// Slot bookkeeping written by a one-thread kernel (values travel as kernel
// parameters: no pinned staging to keep alive, no stream synchronisation).
__global__ void slot_set_kernel(SlotState ss, int slot, int live, int reset, int max_tokens, int terminator,
                                unsigned long long seed) {
  ss.live[slot] = live;
  if (reset) {
    ss.seq_len[slot] = 0;
    ss.gen_count[slot] = 0;
    ss.max_tokens[slot] = max_tokens;
    ss.terminator[slot] = terminator;
    ss.seed[slot] = seed;
  }
}
void launch_slot_set(const SlotState& ss, int slot, int live, int reset, int max_tokens, int terminator,
                     uint64_t seed, cudaStream_t st) {
  slot_set_kernel<<<1, 1, 0, st>>>(ss, slot, live, reset, max_tokens, terminator, (unsigned long long)seed);
}

void launch_gather_rows(const __nv_bfloat16* xg, const float* ssq, const int32_t* last_row,
                        int slots, int H, int parts, __nv_bfloat16* xg_out, float* ssq_out,
                        cudaStream_t st) {
  launch_pdl(gather_rows_kernel, dim3(slots), dim3(256), 0, st, dim3(1, 1, 1), xg, ssq, last_row, H,
             parts, xg_out, ssq_out);
}

void launch_sample(const float* logits, const float* pmax, const double* psum, int V, int slots,
                   const RoundPlan& plan, RoundPlan next_plan, SlotState ss, EventRing ring,
                   const int32_t* round_ctr, const int32_t* version, int greedy, cudaStream_t st) {
  launch_pdl(sample_kernel, dim3(slots), dim3(kSampleThreads), 0, st, dim3(1, 1, 1), logits, pmax,
             psum, V, slots, plan, next_plan, ss, ring, round_ctr, version, greedy);
}

void launch_row_logprobs(const float* logits, int V, int rows, const int32_t* targets, double* out,
                         cudaStream_t st) {
  if (rows > 0) row_logprobs_kernel<<<rows, kSampleThreads, 0, st>>>(logits, V, targets, out);
}

void launch_row_kl(const float* logits_p, const float* logits_q, int V, int rows, double* out, cudaStream_t st) {
  if (rows > 0) row_kl_kernel<<<rows, kSampleThreads, 0, st>>>(logits_p, logits_q, V, out);
}

void launch_sample_logits(const float* logits, int V, int rows, const uint64_t* seeds,
                          const int32_t* draw, int greedy, int32_t* tok, double* lp, cudaStream_t st) {
  if (rows <= 0) return;
  const int T = (V + kTile - 1) / kTile;
  float* pmax = nullptr;
  double* psum = nullptr;
  cudaMallocAsync(&pmax, sizeof(float) * (size_t)rows * T, st);
  cudaMallocAsync(&psum, sizeof(double) * (size_t)rows * T, st);
  tile_stats_kernel<<<dim3((T + 7) / 8, rows), 256, 0, st>>>(logits, V, pmax, psum);
  sample_logits_kernel<<<rows, kSampleThreads, 0, st>>>(logits, pmax, psum, V, seeds, draw, greedy,
                                                        tok, lp);
  cudaFreeAsync(pmax, st);
  cudaFreeAsync(psum, st);
}

void launch_plan_copy(RoundPlan dst, RoundPlan src, int rows, int slots, int32_t* round_ctr,
                      cudaStream_t st) {
  const int n = rows > slots ? rows : slots;
  launch_pdl(plan_copy_kernel, dim3((n + 255) / 256), dim3(256), 0, st, dim3(1, 1, 1), dst, src,
             rows, slots, round_ctr);
}

void launch_lag_stats(const int32_t* versions, const int64_t* seq_offsets, int n_seq,
                      int version_before, int64_t* hist, int hist_cap, int64_t* seq_lag_sums,
                      int64_t* totals, cudaStream_t st) {
  cudaMemsetAsync(hist, 0, sizeof(int64_t) * hist_cap, st);
  cudaMemsetAsync(totals, 0, sizeof(int64_t) * 4, st);
  if (n_seq > 0)
    lag_stats_kernel<<<n_seq, 256, 0, st>>>(versions, seq_offsets, version_before,
                                            reinterpret_cast<unsigned long long*>(hist), hist_cap,
                                            seq_lag_sums,
                                            reinterpret_cast<unsigned long long*>(totals));
}

}  // namespace srl
