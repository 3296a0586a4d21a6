// decoder.cu -- non-GEMM kernels of a decoder round: weight init/drift,
// embedding + first RMSNorm statistics, RoPE + paged-KV append, causal paged
// GQA attention (split-KV, deterministic combine), last-row gather, the fp64
// log-softmax/SplitMix64 sampler, and device lag statistics.
#include <cfloat>
#include <cmath>
#include <cstring>

#include "decoder.cuh"

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
constexpr int kMaxG = 8;

template <int HD>
__global__ void __launch_bounds__(128)
    attention_kernel(const __nv_bfloat16* __restrict__ q, int nq, int nkv,
                     const int32_t* __restrict__ row_slot, const int32_t* __restrict__ row_pos,
                     const int32_t* __restrict__ block_table, int pages_per_seq,
                     const __nv_bfloat16* __restrict__ kc, const __nv_bfloat16* __restrict__ vc,
                     int chunk, float scale, float* __restrict__ ws, int* __restrict__ counters,
                     __nv_bfloat16* __restrict__ out) {
  constexpr int DPL = HD / 32;  // dims per lane in the PV phase
  const int m = blockIdx.x, kh = blockIdx.y, split = blockIdx.z, splits = gridDim.z;
  const int G = nq / nkv;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ float sq[kMaxG][HD];
  __shared__ float sm_m[4][kMaxG], sm_l[4][kMaxG];
  __shared__ float sm_acc[4][kMaxG][HD];
  __shared__ int s_last;

  const int slot = row_slot[m];
  if (slot < 0) return;  // padding / finished row: nothing to attend
  const int ctx = row_pos[m] + 1;
  const int k_begin = split * chunk;
  const int k_end = min(ctx, k_begin + chunk);

  for (int i = threadIdx.x; i < G * HD; i += blockDim.x) {
    const int g = i / HD, d = i % HD;
    sq[g][d] = __bfloat162float(q[(size_t)m * nq * HD + (kh * G + g) * HD + d]) * scale;
  }
  __syncthreads();

  float mrun[kMaxG], lrun[kMaxG], acc[kMaxG][DPL];
#pragma unroll
  for (int g = 0; g < kMaxG; ++g) {
    mrun[g] = -INFINITY;
    lrun[g] = 0.f;
#pragma unroll
    for (int d = 0; d < DPL; ++d) acc[g][d] = 0.f;
  }
  const int32_t* bt = block_table + (size_t)slot * pages_per_seq;

  for (int t0 = k_begin + warp * 32; t0 < k_end; t0 += 128) {
    const int key = t0 + lane;
    const bool valid = key < k_end;
    float s[kMaxG];
    if (valid) {
      const int page = bt[key / kPageTokens];
      const __nv_bfloat16* krow =
          kc + (((size_t)page * nkv + kh) * kPageTokens + (key % kPageTokens)) * HD;
      float kf[HD];
#pragma unroll
      for (int v = 0; v < HD / 8; ++v) {
        const uint4 raw = reinterpret_cast<const uint4*>(krow)[v];
        const __nv_bfloat162* p2 = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = __bfloat1622float2(p2[e]);
          kf[v * 8 + 2 * e] = f.x;
          kf[v * 8 + 2 * e + 1] = f.y;
        }
      }
#pragma unroll
      for (int g = 0; g < kMaxG; ++g) {
        float a = 0.f;
        if (g < G) {
#pragma unroll
          for (int d = 0; d < HD; ++d) a += sq[g][d] * kf[d];
        }
        s[g] = a;
      }
    }
#pragma unroll
    for (int g = 0; g < kMaxG; ++g) {
      if (g >= G) break;
      const float sv = valid ? s[g] : -INFINITY;
      const float tmax = warp_max(sv);
      const float mnew = fmaxf(mrun[g], tmax);
      const float alpha = (mrun[g] == -INFINITY) ? 0.f : __expf(mrun[g] - mnew);
      const float p = valid ? __expf(sv - mnew) : 0.f;
      lrun[g] = lrun[g] * alpha + warp_sum(p);
      mrun[g] = mnew;
#pragma unroll
      for (int d = 0; d < DPL; ++d) acc[g][d] *= alpha;
      s[g] = p;
    }
    const int nvalid = min(32, k_end - t0);
    for (int j = 0; j < nvalid; ++j) {
      const int kj = t0 + j;
      const int page = bt[kj / kPageTokens];
      const __nv_bfloat16* vrow =
          vc + (((size_t)page * nkv + kh) * kPageTokens + (kj % kPageTokens)) * HD + lane * DPL;
      float vf[DPL];
      if constexpr (DPL == 2) {
        const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(vrow));
        vf[0] = f.x;
        vf[1] = f.y;
      } else {
        const uint2 raw = *reinterpret_cast<const uint2*>(vrow);
        const __nv_bfloat162* p2 = reinterpret_cast<const __nv_bfloat162*>(&raw);
        const float2 a = __bfloat1622float2(p2[0]), b = __bfloat1622float2(p2[1]);
        vf[0] = a.x; vf[1] = a.y; vf[2] = b.x; vf[3] = b.y;
      }
#pragma unroll
      for (int g = 0; g < kMaxG; ++g) {
        if (g >= G) break;
        const float pj = __shfl_sync(0xffffffffu, s[g], j);
#pragma unroll
        for (int d = 0; d < DPL; ++d) acc[g][d] += pj * vf[d];
      }
    }
  }

  // combine the 4 warps of this CTA
  if (lane == 0)
    for (int g = 0; g < G; ++g) {
      sm_m[warp][g] = mrun[g];
      sm_l[warp][g] = lrun[g];
    }
  for (int g = 0; g < G; ++g)
#pragma unroll
    for (int d = 0; d < DPL; ++d) sm_acc[warp][g][lane * DPL + d] = acc[g][d];
  __syncthreads();

  const size_t rec = (size_t)G * (HD + 2);
  float* my_ws = ws + (((size_t)m * nkv + kh) * splits + split) * rec;
  for (int i = threadIdx.x; i < G * HD; i += blockDim.x) {
    const int g = i / HD, d = i % HD;
    float M = -INFINITY;
    for (int w = 0; w < 4; ++w) M = fmaxf(M, sm_m[w][g]);
    float L = 0.f, A = 0.f;
    for (int w = 0; w < 4; ++w) {
      const float a = (sm_m[w][g] == -INFINITY) ? 0.f : __expf(sm_m[w][g] - M);
      L += sm_l[w][g] * a;
      A += sm_acc[w][g][d] * a;
    }
    if (splits == 1) {
      out[(size_t)m * nq * HD + (kh * G + g) * HD + d] = __float2bfloat16(L > 0.f ? A / L : 0.f);
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
  for (int i = threadIdx.x; i < G * HD; i += blockDim.x) {
    const int g = i / HD, d = i % HD;
    float M = -INFINITY;
    for (int sp = 0; sp < splits; ++sp) M = fmaxf(M, __ldcg(&base[sp * rec + g * (HD + 2)]));
    float L = 0.f, A = 0.f;
    for (int sp = 0; sp < splits; ++sp) {
      const float ms = __ldcg(&base[sp * rec + g * (HD + 2)]);
      const float a = (ms == -INFINITY) ? 0.f : __expf(ms - M);
      L += __ldcg(&base[sp * rec + g * (HD + 2) + 1]) * a;
      A += __ldcg(&base[sp * rec + g * (HD + 2) + 2 + d]) * a;
    }
    out[(size_t)m * nq * HD + (kh * G + g) * HD + d] = __float2bfloat16(L > 0.f ? A / L : 0.f);
  }
  if (threadIdx.x == 0) counters[cidx] = 0;
}

int attention_splits(const DecoderDims& d, int M, int max_ctx) {
  const int ctas = M * d.nkv;
  int want = (2 * 148 + ctas - 1) / ctas;
  int cap = (max_ctx + 127) / 128;
  int s = want < cap ? want : cap;
  return s < 1 ? 1 : s;
}

// ------------------------------------------------------------- gather ---
__global__ void gather_rows_kernel(const __nv_bfloat16* __restrict__ xg, const float* __restrict__ ssq,
                                   const int32_t* __restrict__ last_row, int H, int parts,
                                   __nv_bfloat16* __restrict__ xg_out, float* __restrict__ ssq_out) {
  const int s = blockIdx.x;
  const int r = last_row[s];
  for (int c = threadIdx.x; c < H; c += blockDim.x)
    xg_out[(size_t)s * H + c] = r >= 0 ? xg[(size_t)r * H + c] : __float2bfloat16(0.f);
  for (int p = threadIdx.x; p < parts; p += blockDim.x)
    ssq_out[(size_t)s * parts + p] = r >= 0 ? ssq[(size_t)r * parts + p] : 1.f;
}

// ------------------------------------------------------------- sample ---
constexpr int kSampleThreads = 1024;

__device__ double block_sum_d(double v, double* red) {
  // fixed-order reduction: warp tree, then warp 0 over the 32 warp sums
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double t = (threadIdx.x < 32) ? red[l] : 0.0;
  if (w == 0) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (l == 0) red[32] = t;
  }
  __syncthreads();
  return red[32];
}

struct SampleShared {
  double red[33];
  float fred[32];
  int ired[32];
  double scan[kSampleThreads];
  int tok;
};

// Block-wide: log-softmax statistics of one logits row in fp64 and the
// SplitMix64 inverse-CDF draw with uniform u (rng.hpp:61-69), or greedy
// argmax (lowest index on ties).  Returns the token; *lse_out = logsumexp.
__device__ int sample_row(const float* __restrict__ x, int V, double u, int greedy,
                          SampleShared& sh, double* lse_out) {
  const int tid = threadIdx.x;
  // pass 1: max (+argmax), then fp64 sum of exp(x - max)  (numeric.hpp:13-20)
  float mx = -INFINITY;
  int amax = 0x7fffffff;
  for (int k = tid; k < V; k += kSampleThreads) {
    const float v = x[k];
    if (v > mx) { mx = v; amax = k; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float om = __shfl_xor_sync(0xffffffffu, mx, o);
    const int oi = __shfl_xor_sync(0xffffffffu, amax, o);
    if (om > mx || (om == mx && oi < amax)) { mx = om; amax = oi; }
  }
  if ((tid & 31) == 0) { sh.fred[tid >> 5] = mx; sh.ired[tid >> 5] = amax; }
  __syncthreads();
  if (tid < 32) {
    mx = sh.fred[tid];
    amax = sh.ired[tid];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float om = __shfl_xor_sync(0xffffffffu, mx, o);
      const int oi = __shfl_xor_sync(0xffffffffu, amax, o);
      if (om > mx || (om == mx && oi < amax)) { mx = om; amax = oi; }
    }
    if (tid == 0) { sh.fred[0] = mx; sh.ired[0] = amax; }
  }
  __syncthreads();
  const double M = (double)sh.fred[0];
  const int argmax = sh.ired[0];
  double part = 0.0;
  for (int k = tid; k < V; k += kSampleThreads) part += exp((double)x[k] - M);
  const double lse = M + log(block_sum_d(part, sh.red));
  *lse_out = lse;
  if (greedy) return argmax;

  // pass 2: contiguous chunk per thread, inclusive scan of chunk masses
  const int C = (V + kSampleThreads - 1) / kSampleThreads;
  const int k0 = tid * C, k1 = min(V, k0 + C);
  double mass = 0.0;
  for (int k = k0; k < k1; ++k) mass += exp((double)x[k] - lse);
  sh.scan[tid] = mass;
  __syncthreads();
  for (int o = 1; o < kSampleThreads; o <<= 1) {  // Hillis-Steele, fixed order
    const double add = tid >= o ? sh.scan[tid - o] : 0.0;
    __syncthreads();
    sh.scan[tid] += add;
    __syncthreads();
  }
  // Every thread's result equals a full walk of its chunk from `base`:
  // u < base means the walk stops at k0; u past the chunk's mass (plus a
  // margin far above the fp64 rounding of the two summation orders) means
  // it never stops; otherwise walk.  The first chunk that stops wins.
  const double base = tid == 0 ? 0.0 : sh.scan[tid - 1];
  int found = 0x7fffffff;
  if (k0 < k1) {
    if (u < base) {
      found = k0;
    } else if (u < sh.scan[tid] + 1e-12) {
      double cum = base;
      for (int k = k0; k < k1; ++k) {
        cum += exp((double)x[k] - lse);
        if (u < cum) { found = k; break; }
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) found = min(found, __shfl_xor_sync(0xffffffffu, found, o));
  __syncthreads();
  if ((tid & 31) == 0) sh.ired[tid >> 5] = found;
  __syncthreads();
  if (tid < 32) {
    int f = sh.ired[tid];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) f = min(f, __shfl_xor_sync(0xffffffffu, f, o));
    if (tid == 0) sh.tok = (f == 0x7fffffff) ? V - 1 : f;  // rounding slack -> V-1
  }
  __syncthreads();
  return sh.tok;
}

__global__ void __launch_bounds__(kSampleThreads)
    sample_kernel(const float* __restrict__ logits, int V, int slots, RoundPlan plan,
                  RoundPlan next, SlotState ss, EventRing ring, const int32_t* __restrict__ round_ctr,
                  const int32_t* __restrict__ version, int greedy) {
  __shared__ SampleShared sh;
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
  const double u = splitmix_uniform(ss.seed[s], (uint64_t)ss.gen_count[s]);
  double lse;
  const int tok = sample_row(x, V, u, greedy, sh, &lse);

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
    float v = warp_max(fred[tid]);
    if (tid == 0) fred[0] = v;
  }
  __syncthreads();
  const double M = (double)fred[0];
  double part = 0.0;
  for (int k = tid; k < V; k += kSampleThreads) part += exp((double)x[k] - M);
  const double lse = M + log(block_sum_d(part, red));
  if (tid == 0) out[row] = (double)x[targets[row]] - lse;
}

__global__ void __launch_bounds__(kSampleThreads)
    sample_logits_kernel(const float* __restrict__ logits, int V, const uint64_t* __restrict__ seeds,
                         const int32_t* __restrict__ draw, int greedy, int32_t* __restrict__ tok_out,
                         double* __restrict__ lp_out) {
  __shared__ SampleShared sh;
  const int r = blockIdx.x;
  const float* x = logits + (size_t)r * V;
  const double u = splitmix_uniform(seeds[r], (uint64_t)draw[r]);
  double lse;
  const int tok = sample_row(x, V, u, greedy, sh, &lse);
  if (threadIdx.x == 0) {
    tok_out[r] = tok;
    lp_out[r] = (double)x[tok] - lse;
  }
}

__global__ void plan_copy_kernel(RoundPlan dst, RoundPlan src, int rows, int slots,
                                 int32_t* round_ctr) {
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
  embed_kernel<<<M, 128, 0, st>>>(embed, gain, row_token, H, V, x, xg, ssq);
}

void launch_rope_append(const float* qkv, const DecoderDims& d, const RoundPlan& plan, int M,
                        const float* cos_sin, const int32_t* block_table, int pages_per_seq,
                        __nv_bfloat16* kc, __nv_bfloat16* vc, __nv_bfloat16* q_out,
                        cudaStream_t st) {
  rope_append_kernel<<<M, 128, 0, st>>>(qkv, d.nq, d.nkv, d.hd, plan.row_slot, plan.row_pos,
                                        cos_sin, block_table, pages_per_seq, kc, vc, q_out);
}

size_t attention_ws_floats(const DecoderDims& d, int M, int max_ctx) {
  const int splits = attention_splits(d, M, max_ctx);
  return (size_t)M * d.nkv * splits * (d.nq / d.nkv) * (d.hd + 2);
}

void launch_attention(const __nv_bfloat16* q, const DecoderDims& d, const RoundPlan& plan, int M,
                      const int32_t* block_table, int pages_per_seq, const __nv_bfloat16* kc,
                      const __nv_bfloat16* vc, int max_ctx, float* ws, int* counters,
                      size_t ws_floats, __nv_bfloat16* out, cudaStream_t st) {
  int splits = attention_splits(d, M, max_ctx);
  if ((size_t)M * d.nkv * splits * (d.nq / d.nkv) * (d.hd + 2) > ws_floats) splits = 1;
  int chunk = (max_ctx + splits - 1) / splits;
  chunk = (chunk + 31) / 32 * 32;
  dim3 grid(M, d.nkv, splits);
  const float scale = 1.0f / sqrtf((float)d.hd);
  if (d.hd == 64)
    attention_kernel<64><<<grid, 128, 0, st>>>(q, d.nq, d.nkv, plan.row_slot, plan.row_pos,
                                               block_table, pages_per_seq, kc, vc, chunk, scale,
                                               ws, counters, out);
  else
    attention_kernel<128><<<grid, 128, 0, st>>>(q, d.nq, d.nkv, plan.row_slot, plan.row_pos,
                                                block_table, pages_per_seq, kc, vc, chunk, scale,
                                                ws, counters, out);
}

void launch_gather_rows(const __nv_bfloat16* xg, const float* ssq, const int32_t* last_row,
                        int slots, int H, int parts, __nv_bfloat16* xg_out, float* ssq_out,
                        cudaStream_t st) {
  gather_rows_kernel<<<slots, 256, 0, st>>>(xg, ssq, last_row, H, parts, xg_out, ssq_out);
}

void launch_sample(const float* logits, int V, int slots, const RoundPlan& plan,
                   RoundPlan next_plan, SlotState ss, EventRing ring, const int32_t* round_ctr,
                   const int32_t* version, int greedy, cudaStream_t st) {
  sample_kernel<<<slots, kSampleThreads, 0, st>>>(logits, V, slots, plan, next_plan, ss, ring,
                                                  round_ctr, version, greedy);
}

void launch_row_logprobs(const float* logits, int V, int rows, const int32_t* targets, double* out,
                         cudaStream_t st) {
  if (rows > 0) row_logprobs_kernel<<<rows, kSampleThreads, 0, st>>>(logits, V, targets, out);
}

void launch_sample_logits(const float* logits, int V, int rows, const uint64_t* seeds,
                          const int32_t* draw, int greedy, int32_t* tok, double* lp, cudaStream_t st) {
  if (rows > 0)
    sample_logits_kernel<<<rows, kSampleThreads, 0, st>>>(logits, V, seeds, draw, greedy, tok, lp);
}

void launch_plan_copy(RoundPlan dst, RoundPlan src, int rows, int slots, int32_t* round_ctr,
                      cudaStream_t st) {
  const int n = rows > slots ? rows : slots;
  plan_copy_kernel<<<(n + 255) / 256, 256, 0, st>>>(dst, src, rows, slots, round_ctr);
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
