// decode_mk.cu -- persistent decode-round megakernel (see decode_mk.cuh).
#include <cmath>
#include <cstdio>

#include "decode_mk.cuh"
#include "sm100.cuh"

namespace srl {
using namespace sm100;

namespace {

constexpr int kTok = 64;   // rows (UMMA N): decode batch <= 64
constexpr int kBN = 128;   // weight rows per tile (UMMA M)
constexpr int kBK = 64;    // k-block (128-B swizzle row)
constexpr int kThreads = 256;
constexpr int kCT = 128;   // compute threads (warps 4..7)
constexpr int kABytes = kBN * kBK * 2;
constexpr int kBBytes = kTok * kBK * 2;
constexpr int kStageBytes = kABytes + kBBytes;
constexpr int kPitch = kBN + 4;
constexpr int kTileFloats = kTok * kBN;
constexpr int kLmTile = 128;
constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ULL;

__device__ __forceinline__ void csync() { asm volatile("bar.sync 1, 128;" ::: "memory"); }
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Bounded spins: a broken schedule traps (the launch fails loudly) instead of
// hanging the device.
constexpr long long kSpinLimit = 1ll << 26;
__device__ __forceinline__ void wait_count(const unsigned* p, unsigned target) {
  long long n = 0;
  while ((int)(ld_acquire(p) - target) < 0) {
    __nanosleep(32);
    if (++n > kSpinLimit) __trap();
  }
}
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, 1000000;\n\t"
      "selp.u32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mk_wait(uint64_t* bar, uint32_t parity) {
  long long n = 0;
  while (!mbar_try(bar, parity))
    if (++n > kSpinLimit) __trap();
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ float bf2f(__nv_bfloat16 v) { return __bfloat162float(v); }
__device__ __forceinline__ float wsum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double wsum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float wmax(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double uniform_draw(uint64_t seed, uint64_t n) {
  uint64_t z = seed + (n + 1) * kGolden;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  z ^= z >> 31;
  return (double)(z >> 11) * 0x1.0p-53;
}

// item index k of CTA c in a phase with `n` items and rotation `rot`
__device__ __forceinline__ int first_item(int c, int rot, int G) { return ((c - rot) % G + G) % G; }

template <int HD, int G>
struct AttnSmem {
  static constexpr int ROW = HD * 2 + 16;
  static constexpr int VROW = HD * 2;
  static constexpr size_t sq = sizeof(float) * G * HD;
  static constexpr size_t sk = (size_t)4 * 32 * ROW;
  static constexpr size_t sv = (size_t)4 * 32 * VROW;
  static constexpr size_t sp = sizeof(float) * 4 * G * 32;
  static constexpr size_t sml = sizeof(float) * 2 * 4 * G;
  static constexpr size_t total = sq + sk + sv + sp + sml;
};

template <int HD, int G>
struct MkLayout {
  static constexpr int STAGES = HD == 64 ? 7 : 5;
  static constexpr size_t ring = (size_t)STAGES * kStageBytes;
  static constexpr size_t epi = sizeof(float) * kTok * kPitch;
  static constexpr size_t att = AttnSmem<HD, G>::total;
  static constexpr size_t smp = sizeof(double) * (kCT + 33) + 256;
  static constexpr size_t scratch = epi > att ? (epi > smp ? epi : smp) : (att > smp ? att : smp);
  static constexpr size_t bar = ring + scratch;
  static constexpr size_t misc = bar + (2 * STAGES + 4) * 8;
  static constexpr size_t rstd = misc + 32;
  static constexpr size_t rowm = rstd + kTok * 4;
  static constexpr size_t total = rowm + kTok * 16;
  static constexpr size_t alloc = total + 1024;
};

// ----------------------------------------------------------- compute ---
// Per-row metadata for the current GEMM phase: rstd (deferred RMSNorm) and,
// for QKV, the KV-cache coordinates of the row.
__device__ void mk_rows(const MkParams& P, int kind, float* s_rstd, int4* s_row, int ct) {
  for (int j = ct; j < kTok; j += kCT) {
    float r = 1.f;
    if ((kind == MK_QKV || kind == MK_GU || kind == MK_LM) && j < P.S) {
      float s = 0.f;
      for (int p = 0; p < P.parts; ++p) s += P.ssq[(size_t)j * P.parts + p];
      r = rsqrtf(s * P.inv_h + P.eps);
    }
    s_rstd[j] = r;
    if (kind == MK_QKV) {
      int4 rc = make_int4(-1, 0, 0, 0);
      if (j < P.S) {
        rc.x = P.plan.row_slot[j];
        rc.y = P.plan.row_pos[j];
        if (rc.x >= 0) {
          rc.z = P.block_table[(size_t)rc.x * P.pps + rc.y / kPageTokens];
          rc.w = rc.y % kPageTokens;
        }
      }
      s_row[j] = rc;
    }
  }
}

// Fused epilogues on the reduced [64 x 128] tile (rows = tokens, cols = n0..).
// Rows [r0, r1) of the tile belong to this CTA (split-K row slices).
__device__ void mk_epilogue(const MkParams& P, const MkPhase& ph, int n_tile, float* tile,
                            const float* s_rstd, const int4* s_row, int ct, int r0, int r1) {
  const int n0 = n_tile * kBN, N = ph.N, M = r1;
  const int nr = r1 - r0;
  const int cw = ct >> 5, lane = ct & 31;
  const __nv_bfloat16* w = P.w;
  if (ph.kind == MK_QKV) {
    const __nv_bfloat16* bias = w + P.layers[ph.layer].qkv_b;
#pragma unroll 4
    for (int idx = ct; idx < nr * kBN; idx += kCT) {
      const int j = r0 + (idx >> 7), c = idx & 127, n = n0 + c;
      float v = 0.f;
      if (n < N) v = tile[j * kPitch + c] * s_rstd[j] + bf2f(bias[n]);
      tile[j * kPitch + c] = v;
    }
    csync();
    const int hd = P.hd, half = hd >> 1;
    const int qend = P.nq * hd, kend = (P.nq + P.nkv) * hd;
    __nv_bfloat16* kc = P.kc + P.kv_layer_elems * ph.layer;
    __nv_bfloat16* vc = P.vc + P.kv_layer_elems * ph.layer;
#pragma unroll 4
    for (int idx = ct; idx < nr * kBN; idx += kCT) {
      const int j = r0 + (idx >> 7), c = idx & 127, n = n0 + c;
      const int4 rc = s_row[j];
      if (n >= N || rc.x < 0) continue;
      const int jj = n % hd;
      const float* row = &tile[j * kPitch + (c - jj)];
      float y;
      if (n < kend) {
        const int i = jj < half ? jj : jj - half;
        const float co = P.cos_sin[(size_t)rc.y * hd + i];
        const float si = P.cos_sin[(size_t)rc.y * hd + half + i];
        const float x1 = row[i], x2 = row[i + half];
        y = jj < half ? x1 * co - x2 * si : x2 * co + x1 * si;
      } else {
        y = row[jj];
      }
      const __nv_bfloat16 b = __float2bfloat16(y);
      if (n < qend) {
        P.q[(size_t)j * qend + n] = b;
      } else {
        const int kv = n < kend ? n - qend : n - kend;
        const size_t at = (((size_t)rc.z * P.nkv + kv / hd) * kPageTokens + rc.w) * hd + (kv % hd);
        if (n < kend) kc[at] = b;
        else vc[at] = b;
      }
    }
  } else if (ph.kind == MK_O || ph.kind == MK_DOWN) {
    const __nv_bfloat16* gain =
        w + (ph.kind == MK_O ? P.layers[ph.layer].ln2
                             : (ph.layer + 1 < P.L ? P.layers[ph.layer + 1].ln1 : P.off_final_norm));
#pragma unroll 4
    for (int idx = ct; idx < nr * kBN; idx += kCT) {
      const int j = r0 + (idx >> 7), c = idx & 127, n = n0 + c;
      float x = 0.f;
      if (n < N) {
        const size_t o = (size_t)j * N + n;
        x = P.x[o] + tile[j * kPitch + c];
        P.x[o] = x;
        P.xg[o] = __float2bfloat16(x * bf2f(gain[n]));
      }
      tile[j * kPitch + c] = x;
    }
    csync();
    for (int j = r0 + cw; j < M; j += kCT / 32) {
      float s = 0.f;
      for (int c = lane; c < kBN; c += 32) {
        const float xv = tile[j * kPitch + c];
        s += xv * xv;
      }
      s = wsum(s);
      if (lane == 0) P.ssq[(size_t)j * P.parts + n_tile] = s;
    }
  } else if (ph.kind == MK_GU) {
#pragma unroll 4
    for (int idx = ct; idx < nr * (kBN / 2); idx += kCT) {
      const int j = r0 + (idx >> 6), c = idx & 63;
      const float g = tile[j * kPitch + c] * s_rstd[j];
      const float u = tile[j * kPitch + 64 + c] * s_rstd[j];
      P.act[(size_t)j * P.I + (n0 >> 1) + c] = __float2bfloat16(g / (1.f + expf(-g)) * u);
    }
  } else if (ph.kind == MK_LM) {
#pragma unroll 4
    for (int idx = ct; idx < nr * kBN; idx += kCT) {
      const int j = r0 + (idx >> 7), c = idx & 127, n = n0 + c;
      float v = -INFINITY;
      if (n < N) {
        v = tile[j * kPitch + c] * s_rstd[j];
        P.logits[(size_t)j * N + n] = v;
      }
      tile[j * kPitch + c] = v;
    }
    csync();
    const int T = (N + kLmTile - 1) / kLmTile;
    for (int j = r0 + cw; j < M; j += kCT / 32) {
      const float4 x = *reinterpret_cast<const float4*>(&tile[j * kPitch + lane * 4]);
      const float mx = wmax(fmaxf(fmaxf(x.x, x.y), fmaxf(x.z, x.w)));
      double s = 0.0;
      if (mx != -INFINITY) {
        const double md = (double)mx;
        s = exp((double)x.x - md) + exp((double)x.y - md) + exp((double)x.z - md) +
            exp((double)x.w - md);
      }
      s = wsum_d(s);
      if (lane == 0) {
        P.lse_max[(size_t)j * T + n_tile] = mx;
        P.lse_sum[(size_t)j * T + n_tile] = s;
      }
    }
  }
}

// Causal paged GQA attention for (row m, kv head kh, 128-key split) on the 4
// compute warps (same algorithm as attention_kernel in decoder.cu).
template <int HD, int G>
__device__ void mk_attention(const MkParams& P, int layer, int m, int kh, int split, uint8_t* scr,
                             unsigned* ctr, unsigned ep1, float* ws, int ct, int* s_flag) {
  using A = AttnSmem<HD, G>;
  constexpr int DPL = HD / 32, V4 = HD / 8;
  float(*sq)[HD] = reinterpret_cast<float(*)[HD]>(scr);
  uint8_t(*sk)[32 * A::ROW] = reinterpret_cast<uint8_t(*)[32 * A::ROW]>(scr + A::sq);
  uint8_t(*sv)[32 * A::VROW] = reinterpret_cast<uint8_t(*)[32 * A::VROW]>(scr + A::sq + A::sk);
  float(*sp)[G][32] = reinterpret_cast<float(*)[G][32]>(scr + A::sq + A::sk + A::sv);
  float(*sm_m)[G] = reinterpret_cast<float(*)[G]>(scr + A::sq + A::sk + A::sv + A::sp);
  float(*sm_l)[G] = reinterpret_cast<float(*)[G]>(scr + A::sq + A::sk + A::sv + A::sp + sizeof(float) * 4 * G);
  float(*sm_acc)[G][HD] = reinterpret_cast<float(*)[G][HD]>(scr + A::sq);  // aliases sk
  const int warp = ct >> 5, lane = ct & 31;
  const int splits = P.attn_splits, nq = P.nq, nkv = P.nkv;
  const int slot = P.plan.row_slot[m];
  if (slot < 0) {  // every split still arrives: the counters are monotonic
    if (splits > 1 && ct == 0) atomicAdd(&ctr[m * nkv + kh], 1u);
    return;
  }
  const int ctx = P.plan.row_pos[m] + 1;
  const int k_begin = split * 128;
  const __nv_bfloat16* kc = P.kc + P.kv_layer_elems * layer;
  const __nv_bfloat16* vc = P.vc + P.kv_layer_elems * layer;
  for (int i = ct; i < G * HD; i += kCT)
    sq[i / HD][i % HD] = bf2f(P.q[(size_t)m * nq * HD + (kh * G) * HD + i]) * P.scale;
  csync();
  float mrun[G], lrun[G], acc[G][DPL];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    mrun[g] = -INFINITY;
    lrun[g] = 0.f;
#pragma unroll
    for (int d = 0; d < DPL; ++d) acc[g][d] = 0.f;
  }
  const int t0 = k_begin + warp * 32;
  const int nvalid = max(0, min(32, ctx - t0));
  if (nvalid > 0) {
    const int page = P.block_table[(size_t)slot * P.pps + t0 / kPageTokens];
    const size_t base = (((size_t)page * nkv + kh) * kPageTokens + (t0 % kPageTokens)) * HD;
    const uint4* kg = reinterpret_cast<const uint4*>(kc + base);
    const uint4* vg = reinterpret_cast<const uint4*>(vc + base);
    uint4 kr[V4], vr[V4];
#pragma unroll
    for (int i = 0; i < V4; ++i) {
      const int e = lane + 32 * i, r = e / V4;
      if (r < nvalid) { kr[i] = kg[e]; vr[i] = vg[e]; }
    }
#pragma unroll
    for (int i = 0; i < V4; ++i) {
      const int e = lane + 32 * i, r = e / V4, c = e % V4;
      if (r < nvalid) {
        *reinterpret_cast<uint4*>(&sk[warp][r * A::ROW + c * 16]) = kr[i];
        *reinterpret_cast<uint4*>(&sv[warp][r * A::VROW + c * 16]) = vr[i];
      }
    }
    __syncwarp();
    float s[G];
#pragma unroll
    for (int g = 0; g < G; ++g) s[g] = 0.f;
    if (lane < nvalid) {
#pragma unroll
      for (int c = 0; c < V4; ++c) {
        const uint4 raw = *reinterpret_cast<const uint4*>(&sk[warp][lane * A::ROW + c * 16]);
        const __nv_bfloat162* p2 = reinterpret_cast<const __nv_bfloat162*>(&raw);
        float kf[8];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = __bfloat1622float2(p2[e]);
          kf[2 * e] = f.x;
          kf[2 * e + 1] = f.y;
        }
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const float4 qa = *reinterpret_cast<const float4*>(&sq[g][c * 8]);
          const float4 qb = *reinterpret_cast<const float4*>(&sq[g][c * 8 + 4]);
          s[g] += qa.x * kf[0] + qa.y * kf[1] + qa.z * kf[2] + qa.w * kf[3] + qb.x * kf[4] +
                  qb.y * kf[5] + qb.z * kf[6] + qb.w * kf[7];
        }
      }
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const float sv_ = lane < nvalid ? s[g] : -INFINITY;
      const float mx = wmax(sv_);
      const float p = lane < nvalid ? __expf(sv_ - mx) : 0.f;
      mrun[g] = mx;
      lrun[g] = wsum(p);
      sp[warp][g][lane] = p;
    }
    __syncwarp();
    for (int j = 0; j < nvalid; ++j) {
      float vf[DPL];
      const uint8_t* vrow = &sv[warp][j * A::VROW + lane * DPL * 2];
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
      for (int g = 0; g < G; ++g) {
        const float pj = sp[warp][g][j];
#pragma unroll
        for (int d = 0; d < DPL; ++d) acc[g][d] += pj * vf[d];
      }
    }
  }
  csync();  // sm_acc aliases the K tiles
  if (lane == 0) {
#pragma unroll
    for (int g = 0; g < G; ++g) {
      sm_m[warp][g] = mrun[g];
      sm_l[warp][g] = lrun[g];
    }
  }
#pragma unroll
  for (int g = 0; g < G; ++g)
#pragma unroll
    for (int d = 0; d < DPL; ++d) sm_acc[warp][g][lane * DPL + d] = acc[g][d];
  csync();
  constexpr size_t rec = (size_t)G * (HD + 2);
  float* my_ws = ws + (((size_t)m * nkv + kh) * splits + split) * rec;
  for (int i = ct; i < G * HD; i += kCT) {
    const int g = i / HD, d = i % HD;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < 4; ++w) M = fmaxf(M, sm_m[w][g]);
    float L = 0.f, Acc = 0.f;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const float a = (sm_m[w][g] == -INFINITY) ? 0.f : __expf(sm_m[w][g] - M);
      L += sm_l[w][g] * a;
      Acc += sm_acc[w][g][d] * a;
    }
    if (splits == 1) {
      P.attn[(size_t)m * nq * HD + (kh * G + g) * HD + d] = __float2bfloat16(L > 0.f ? Acc / L : 0.f);
    } else {
      __stcg(&my_ws[g * (HD + 2) + 2 + d], Acc);
      if (d == 0) {
        __stcg(&my_ws[g * (HD + 2)], M);
        __stcg(&my_ws[g * (HD + 2) + 1], L);
      }
    }
  }
  if (splits == 1) {
    csync();
    return;
  }
  csync();
  if (ct == 0) {
    __threadfence();
    *s_flag = (atomicAdd(&ctr[m * nkv + kh], 1u) + 1u == ep1 * (unsigned)splits);
  }
  csync();
  const bool last = *s_flag;
  if (last) {
    __threadfence();
    const float* base = ws + ((size_t)m * nkv + kh) * splits * rec;
    const int used = min(splits, (ctx + 127) / 128);
    for (int i = ct; i < G * HD; i += kCT) {
      const int g = i / HD, d = i % HD;
      float M = -INFINITY;
      for (int q = 0; q < used; ++q) M = fmaxf(M, __ldcg(&base[q * rec + g * (HD + 2)]));
      float L = 0.f, Acc = 0.f;
      for (int q = 0; q < used; ++q) {
        const float ms = __ldcg(&base[q * rec + g * (HD + 2)]);
        const float a = (ms == -INFINITY) ? 0.f : __expf(ms - M);
        L += __ldcg(&base[q * rec + g * (HD + 2) + 1]) * a;
        Acc += __ldcg(&base[q * rec + g * (HD + 2) + 2 + d]) * a;
      }
      P.attn[(size_t)m * nq * HD + (kh * G + g) * HD + d] = __float2bfloat16(L > 0.f ? Acc / L : 0.f);
    }
  }
  csync();
}

// plan copy + embedding + first RMSNorm statistics for row m
__device__ void mk_embed(const MkParams& P, int m, int ct, float* red) {
  if (ct == 0) {
    P.plan.row_slot[m] = P.next.row_slot[m];
    P.plan.row_pos[m] = P.next.row_pos[m];
    P.plan.row_token[m] = P.next.row_token[m];
    P.plan.last_row[m] = P.next.last_row[m];
  }
  const int tok = P.next.row_token[m];
  const bool ok = tok >= 0 && tok < P.V;
  const __nv_bfloat16* E = P.w + P.off_embed;
  const __nv_bfloat16* g = P.w + P.layers[0].ln1;
  for (int p = 0; p < P.parts; ++p) {
    const int c = p * 128 + ct;
    float v = 0.f;
    if (c < P.H) {
      v = ok ? bf2f(E[(size_t)tok * P.H + c]) : 0.f;
      P.x[(size_t)m * P.H + c] = v;
      P.xg[(size_t)m * P.H + c] = __float2bfloat16(v * bf2f(g[c]));
    }
    const float s = wsum(v * v);
    if ((ct & 31) == 0) red[ct >> 5] = s;
    csync();
    if (ct == 0) P.ssq[(size_t)m * P.parts + p] = red[0] + red[1] + red[2] + red[3];
    csync();
  }
}

// Sampling of slot s from the LM-head tile partials (128 threads): same
// algorithm as sample_row in decoder.cu.
__device__ void mk_sample(const MkParams& P, int s, int ct, uint8_t* scr) {
  double* scan = reinterpret_cast<double*>(scr);
  double* red = scan + kCT;
  int* iv = reinterpret_cast<int*>(red + 33);
  float* fv = reinterpret_cast<float*>(iv + 8);
  const int warp = ct >> 5, lane = ct & 31;
  const int V = P.V;
  const int ri = (*P.round_ctr - 1) % P.ring.rounds;
  const size_t ev = (size_t)ri * P.S + s;
  const int r = P.plan.last_row[s];
  if (r < 0 || P.ss.live[s] == 0) {
    if (ct == 0) {
      P.ring.ev[ev].flag = 0;
      P.next.row_slot[s] = -1;
      P.next.last_row[s] = -1;
      P.next.row_pos[s] = 0;
      P.next.row_token[s] = 0;
    }
    return;
  }
  const float* x = P.logits + (size_t)s * V;
  const int T = (V + kLmTile - 1) / kLmTile;
  const float* pmax = P.lse_max + (size_t)s * T;
  const double* psum = P.lse_sum + (size_t)s * T;
  const int C = (T + kCT - 1) / kCT;
  const int t0 = ct * C, t1 = min(T, t0 + C);
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
  if (lane == 0) { fv[warp] = mx; iv[warp] = mt; }
  csync();
  if (ct == 0) {
    for (int w = 1; w < 4; ++w)
      if (fv[w] > fv[0] || (fv[w] == fv[0] && iv[w] < iv[0])) { fv[0] = fv[w]; iv[0] = iv[w]; }
  }
  csync();
  const float Mf = fv[0];
  const double M = (double)Mf;
  const int mtile = iv[0];
  double part = 0.0;
  for (int t = t0; t < t1; ++t) part += psum[t] * exp((double)pmax[t] - M);
  part = wsum_d(part);
  if (lane == 0) red[warp] = part;
  csync();
  const double lse = M + log(red[0] + red[1] + red[2] + red[3]);
  csync();
  const double u = uniform_draw(P.ss.seed[s], (uint64_t)P.ss.gen_count[s]);
  int tok;
  if (P.greedy) {
    if (warp == 0) {
      int best = 0x7fffffff;
      for (int i = lane; i < kLmTile; i += 32) {
        const int k = mtile * kLmTile + i;
        if (k < V && x[k] == Mf) best = min(best, k);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
      if (lane == 0) iv[4] = best == 0x7fffffff ? mtile * kLmTile : best;
    }
    csync();
    tok = iv[4];
  } else {
    double mass = 0.0;
    for (int t = t0; t < t1; ++t) mass += psum[t] * exp((double)pmax[t] - lse);
    scan[ct] = mass;
    csync();
    for (int o = 1; o < kCT; o <<= 1) {
      const double add = ct >= o ? scan[ct - o] : 0.0;
      csync();
      scan[ct] += add;
      csync();
    }
    int cand = 0x7fffffff;
    {
      double base = ct == 0 ? 0.0 : scan[ct - 1];
      if (u < scan[ct] + 1e-12) {
        for (int t = t0; t < t1; ++t) {
          const double q = psum[t] * exp((double)pmax[t] - lse);
          if (u < base + q + 1e-12) { cand = t; break; }
          base += q;
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cand = min(cand, __shfl_xor_sync(0xffffffffu, cand, o));
    if (lane == 0) iv[warp] = cand;
    csync();
    if (warp == 0) {
      int t = min(min(iv[0], iv[1]), min(iv[2], iv[3]));
      int tk = V - 1;
      if (t != 0x7fffffff) {
        const int owner = t / C;
        double base = owner == 0 ? 0.0 : scan[owner - 1];
        for (int tt = owner * C; tt < t; ++tt) base += psum[tt] * exp((double)pmax[tt] - lse);
        bool done = false;
        for (; t < T && !done; ++t) {
          double p[4];
          double ls = 0.0;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int k = t * kLmTile + lane * 4 + i;
            p[i] = k < V ? exp((double)x[k] - lse) : 0.0;
            ls += p[i];
          }
          double incl = ls;
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
            const int k = t * kLmTile + lane * 4 + i;
            if (found == 0x7fffffff && k < V && u < cum) found = k;
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) found = min(found, __shfl_xor_sync(0xffffffffu, found, o));
          if (found != 0x7fffffff) {
            tk = found;
            done = true;
          }
          base += __shfl_sync(0xffffffffu, incl, 31);
        }
      }
      if (lane == 0) iv[4] = tk;
    }
    csync();
    tok = iv[4];
  }
  if (ct == 0) {
    const int pos_row = P.plan.row_pos[r];
    const int new_len = pos_row + 1;
    const int gen = P.ss.gen_count[s];
    int flag = 1;
    if (tok == P.ss.terminator[s]) flag = 3;
    else if (gen + 1 >= P.ss.max_tokens[s]) flag = 2;
    else if (new_len + 1 > P.ss.max_seq) flag = 2;
    DevEvent e;
    e.flag = flag;
    e.token = tok;
    e.position = gen;
    e.version = *P.version;
    e.logprob = (double)x[tok] - lse;
    P.ring.ev[ev] = e;
    P.ss.seq_len[s] = new_len;
    P.ss.gen_count[s] = gen + 1;
    if (new_len < P.ss.max_seq) P.ss.history[(size_t)s * P.ss.max_seq + new_len] = tok;
    const int alive = flag == 1;
    P.ss.live[s] = alive;
    P.next.row_slot[s] = alive ? s : -1;
    P.next.row_pos[s] = new_len;
    P.next.row_token[s] = tok;
    P.next.last_row[s] = alive ? s : -1;
  }
  csync();
}

// ------------------------------------------------------------ kernel ---
template <int HD, int G>
__global__ void __launch_bounds__(kThreads, 1) decode_megakernel(const __grid_constant__ MkParams P) {
  using Lo = MkLayout<HD, G>;
  constexpr int STAGES = Lo::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* scratch = smem + Lo::ring;
  float* tile = reinterpret_cast<float*>(scratch);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Lo::bar);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + Lo::misc);
  int* s_flag = reinterpret_cast<int*>(smem + Lo::misc + 4);
  float* s_red = reinterpret_cast<float*>(smem + Lo::misc + 8);  // 4 floats
  float* s_rstd = reinterpret_cast<float*>(smem + Lo::rstd);
  int4* s_row = reinterpret_cast<int4*>(smem + Lo::rowm);

  const int warp = threadIdx.x >> 5;
  const int GR = gridDim.x, c = blockIdx.x;
  const unsigned ep1 = *P.epoch + 1u;
  const unsigned target = ep1 * (unsigned)GR;

  if (warp == 0) {
    tmem_alloc<128>(tmem_slot);  // two 64-column fp32 accumulators
  } else if (warp == 1) {
    if (elect_one()) {
      for (int s = 0; s < STAGES; ++s) {
        mbar_init(&full[s], 1);
        mbar_init(&empty[s], 1);
      }
      for (int a = 0; a < 2; ++a) {
        mbar_init(&tfull[a], 1);
        mbar_init(&tempty[a], kCT);
      }
      fence_barrier_init();
    }
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------------------------------------------- TMA producer
    if (elect_one()) {
      const uint64_t pol = policy_evict_first();
      int stage = 0;
      uint32_t ph = 0;
      for (int p = 0; p < P.n_phases; ++p) {
        const MkPhase& F = P.phases[p];
        if (F.kind == MK_EMBED || F.kind == MK_ATTN || F.kind == MK_SAMPLE) continue;
        const CUtensorMap* tw = &P.wmaps[F.wmap];
        const CUtensorMap* tx = &P.xmaps[F.xmap];
        bool dep_ok = false;
        const int kb_total = F.K / kBK;
        for (int i = first_item(c, F.rot, GR); i < F.n_items; i += GR) {
          const int tile_n = i / F.cs, split = i % F.cs;
          const int kb0 = (split * kb_total) / F.cs;
          const int nkb = ((split + 1) * kb_total) / F.cs - kb0;
          const int n0 = tile_n * kBN;
          const int pre = nkb < STAGES ? nkb : STAGES;
          const int s0 = stage;
          for (int k = 0; k < pre; ++k) {  // weights: independent of the previous phase
            mk_wait(&empty[stage], ph ^ 1);
            mbar_arrive_expect_tx(&full[stage], kStageBytes);
            tma_load_2d_hint(smem + stage * kStageBytes, tw, &full[stage], (kb0 + k) * kBK, n0, pol);
            if (++stage == STAGES) { stage = 0; ph ^= 1; }
          }
          if (!dep_ok) {
            wait_count(&P.phase_done[p - 1], target);
            fence_proxy_async_global();  // generic-proxy results -> TMA reads
            dep_ok = true;
          }
          for (int k = 0; k < pre; ++k) {
            const int st = (s0 + k) % STAGES;
            tma_load_2d(smem + st * kStageBytes + kABytes, tx, &full[st], (kb0 + k) * kBK, 0);
          }
          for (int k = pre; k < nkb; ++k) {
            mk_wait(&empty[stage], ph ^ 1);
            mbar_arrive_expect_tx(&full[stage], kStageBytes);
            uint8_t* a = smem + stage * kStageBytes;
            tma_load_2d_hint(a, tw, &full[stage], (kb0 + k) * kBK, n0, pol);
            tma_load_2d(a + kABytes, tx, &full[stage], (kb0 + k) * kBK, 0);
            if (++stage == STAGES) { stage = 0; ph ^= 1; }
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------ MMA issuer
    if (elect_one()) {
      constexpr uint32_t idesc = idesc_bf16_f32(128, kTok);
      int stage = 0, acc = 0;
      uint32_t ph = 0, aph = 0;
      for (int p = 0; p < P.n_phases; ++p) {
        const MkPhase& F = P.phases[p];
        if (F.kind == MK_EMBED || F.kind == MK_ATTN || F.kind == MK_SAMPLE) continue;
        const int kb_total = F.K / kBK;
        for (int i = first_item(c, F.rot, GR); i < F.n_items; i += GR) {
          const int split = i % F.cs;
          const int nkb = ((split + 1) * kb_total) / F.cs - (split * kb_total) / F.cs;
          mk_wait(&tempty[acc], aph ^ 1);
          tc_fence_after();
          const uint32_t d = tmem + acc * kTok;
          for (int k = 0; k < nkb; ++k) {
            mk_wait(&full[stage], ph);
            tc_fence_after();
            const uint32_t a = smem_u32(smem + stage * kStageBytes);
            const uint32_t b = a + kABytes;
#pragma unroll
            for (int kk = 0; kk < kBK / 16; ++kk)
              mma_bf16_ss(d, umma_desc_k_sw128(a, kk * 32), umma_desc_k_sw128(b, kk * 32), idesc,
                          (k | kk) != 0);
            mma_commit(&empty[stage]);
            if (++stage == STAGES) { stage = 0; ph ^= 1; }
          }
          mma_commit(&tfull[acc]);
          if (++acc == 2) { acc = 0; aph ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ------------------------------------------------------ compute
    const int ct = threadIdx.x - 128, cw = ct >> 5;
    const bool stamp = P.stamps != nullptr && c == 0 && ct == 0;
    int acc = 0;
    uint32_t aph = 0;
    if (stamp) P.stamps[0] = globaltimer();
    for (int p = 0; p < P.n_phases; ++p) {
      const MkPhase& F = P.phases[p];
      if (p > 0) {  // results of the previous phase, grid-wide
        if (ct == 0) {
          wait_count(&P.phase_done[p - 1], target);
          if (stamp) P.stamps[p] = globaltimer();
        }
        csync();
      }
      if (F.kind == MK_EMBED) {
        if (c == 0 && ct == 0) *P.round_ctr += 1;
        for (int m = first_item(c, F.rot, GR); m < F.n_items; m += GR) mk_embed(P, m, ct, s_red);
      } else if (F.kind == MK_ATTN) {
        for (int i = first_item(c, F.rot, GR); i < F.n_items; i += GR) {
          const int split = i % P.attn_splits;
          const int rest = i / P.attn_splits;
          mk_attention<HD, G>(P, F.layer, rest / P.nkv, rest % P.nkv, split, scratch,
                              P.tile_ctr + F.ctr_base, ep1, P.ws, ct, s_flag);
        }
      } else if (F.kind == MK_SAMPLE) {
        for (int s = first_item(c, F.rot, GR); s < F.n_items; s += GR) mk_sample(P, s, ct, scratch);
      } else {
        mk_rows(P, F.kind, s_rstd, s_row, ct);
        for (int i = first_item(c, F.rot, GR); i < F.n_items; i += GR) {
          const int tile_n = i / F.cs, split = i % F.cs;
          mk_wait(&tfull[acc], aph);
          tc_fence_after();
          const uint32_t lane_addr = tmem + acc * kTok + ((uint32_t)(cw * 32) << 16);
          uint32_t ra[32], rb[32];
          tmem_ld_32x32b_x32(lane_addr, ra);
          tmem_ld_32x32b_x32(lane_addr + 32, rb);
          tmem_ld_wait();
          tc_fence_before();
          mbar_arrive(&tempty[acc]);  // accumulator free for the MMA warp
          if (++acc == 2) { acc = 0; aph ^= 1; }
          int r0 = 0, r1 = P.S;
          if (F.cs == 1) {
#pragma unroll
            for (int j = 0; j < 32; ++j) tile[j * kPitch + ct] = __uint_as_float(ra[j]);
#pragma unroll
            for (int j = 0; j < 32; ++j) tile[(32 + j) * kPitch + ct] = __uint_as_float(rb[j]);
          } else {
            // publish this split's partial (rows < S), wait for the tile's other
            // splits, then reduce this split's row slice in split order
            float* part = P.ws + (size_t)i * kTileFloats;
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (j < P.S) __stcg(&part[j * kBN + ct], __uint_as_float(ra[j]));
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (32 + j < P.S) __stcg(&part[(32 + j) * kBN + ct], __uint_as_float(rb[j]));
            csync();
            if (ct == 0) {
              unsigned* tc = &P.tile_ctr[F.ctr_base + tile_n];
              __threadfence();
              atomicAdd(tc, 1u);
              wait_count(tc, ep1 * (unsigned)F.cs);
            }
            csync();
            r0 = (split * P.S) / F.cs;
            r1 = ((split + 1) * P.S) / F.cs;
            const float4* b4 = reinterpret_cast<const float4*>(P.ws + (size_t)tile_n * F.cs * kTileFloats);
            for (int e = r0 * (kBN / 4) + ct; e < r1 * (kBN / 4); e += kCT) {
              float4 a = __ldcg(b4 + e);
              for (int q = 1; q < F.cs; ++q) {
                const float4 v = __ldcg(b4 + (size_t)q * (kTileFloats / 4) + e);
                a.x += v.x; a.y += v.y; a.z += v.z; a.w += v.w;
              }
              const int j = e / (kBN / 4), cc = (e % (kBN / 4)) * 4;
              *reinterpret_cast<float4*>(&tile[j * kPitch + cc]) = a;
            }
          }
          csync();
          if (r1 > r0) mk_epilogue(P, F, tile_n, tile, s_rstd, s_row, ct, r0, r1);
          csync();
        }
      }
      fence_proxy_async_global();  // later phases read these results with TMA
      csync();
      if (ct == 0) {
        __threadfence();
        atomicAdd(&P.phase_done[p], 1u);
      }
    }
    if (stamp) {
      wait_count(&P.phase_done[P.n_phases - 1], target);
      P.stamps[P.n_phases] = globaltimer();
    }
  }
  // ---- teardown
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_free<128>(tmem);
  if (c == 0 && threadIdx.x == 0) *P.epoch += 1u;
}

template <int HD, int G>
bool set_smem_attr() {
  static const bool ok = cudaFuncSetAttribute(decode_megakernel<HD, G>,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)MkLayout<HD, G>::alloc) == cudaSuccess;
  return ok;
}

template <int HD, int G>
int occupancy_t() {
  if (!set_smem_attr<HD, G>()) return 0;
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, decode_megakernel<HD, G>, kThreads,
                                                    MkLayout<HD, G>::alloc) != cudaSuccess)
    return 0;
  return n;
}

template <int HD, int G>
cudaError_t launch_t(const MkParams& p, int grid, cudaStream_t st) {
  using Lo = MkLayout<HD, G>;
  if (!set_smem_attr<HD, G>()) return cudaErrorInvalidValue;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = Lo::alloc;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;  // co-residency for the phase counters
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, decode_megakernel<HD, G>, p);
}

}  // namespace

int megakernel_splits(int N, int K, int grid) {
  // cost ~ bytes one CTA streams (24 KB per k-block) + a flat charge for the
  // partial exchange; split-K only while the phase still fits one wave
  const int tiles = (N + kBN - 1) / kBN, kb = K / kBK;
  int best = 1;
  long best_cost = (long)((tiles + grid - 1) / grid) * kb * 24;
  for (int cs = 2; cs <= kb && tiles * cs <= grid; ++cs) {
    const long cost = (long)((kb + cs - 1) / cs) * 24 + 40;
    if (cost < best_cost) {
      best_cost = cost;
      best = cs;
    }
  }
  return best;
}

size_t megakernel_ws_floats(int n_items, int cs, int rows) {
  (void)rows;
  return cs > 1 ? (size_t)n_items * kTileFloats : 0;
}

bool megakernel_supported(const DecoderDims& d, int slots) {
  if (slots > kTok || d.nq % d.nkv) return false;
  const int G = d.nq / d.nkv;
  if (d.hd == 64) return G == 2 || G == 7;
  if (d.hd == 128) return G == 6 || G == 7;
  return false;
}

size_t megakernel_smem_bytes(const DecoderDims& d) {
  const int G = d.nq / d.nkv;
  if (d.hd == 64) return G == 2 ? MkLayout<64, 2>::alloc : MkLayout<64, 7>::alloc;
  return G == 6 ? MkLayout<128, 6>::alloc : MkLayout<128, 7>::alloc;
}

int megakernel_occupancy(const DecoderDims& d) {
  const int G = d.nq / d.nkv;
  if (d.hd == 64 && G == 2) return occupancy_t<64, 2>();
  if (d.hd == 64 && G == 7) return occupancy_t<64, 7>();
  if (d.hd == 128 && G == 6) return occupancy_t<128, 6>();
  if (d.hd == 128 && G == 7) return occupancy_t<128, 7>();
  return 0;
}

cudaError_t launch_megakernel(const MkParams& p, const DecoderDims& d, int grid, cudaStream_t st) {
  const int G = d.nq / d.nkv;
  if (d.hd == 64 && G == 2) return launch_t<64, 2>(p, grid, st);
  if (d.hd == 64 && G == 7) return launch_t<64, 7>(p, grid, st);
  if (d.hd == 128 && G == 6) return launch_t<128, 6>(p, grid, st);
  if (d.hd == 128 && G == 7) return launch_t<128, 7>(p, grid, st);
  return cudaErrorInvalidValue;
}

}  // namespace srl
