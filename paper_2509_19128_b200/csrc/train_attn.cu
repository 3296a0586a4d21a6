#include <cstdlib>
// train_attn.cu -- causal GQA attention backward of the trainer on the tensor
// cores (mma.sync m16n8k16 bf16 -> fp32), tiled FlashAttention-2 style.
//
// The trainer's forward keeps q (post-RoPE, bf16), the attention output o,
// the per-(row, head) log-sum-exp and writes K/V into a paged cache (one
// 64-token page per block of a sequence).  With D = rowsum(dO * O):
//   P  = exp(scale * Q K^T - lse)          (causal)
//   dV = P^T dO,   dP = dO V^T,   dS = P * (dP - D)
//   dQ = scale * dS K,   dK = scale * dS^T Q
// Two deterministic kernels (no atomics):
//   attn_bwd_dkv_mma : CTA = (64-key block, sequence, KV head); loops over the
//                      G query heads of the group and the causal query blocks;
//   attn_bwd_dq_mma  : CTA = (64-query block, sequence, query head); loops
//                      over the causal key blocks.
// Four warps per CTA, each owning 16 rows (keys resp. queries) of the block.
// P and dS enter the second GEMM of each pair as bf16, as in the forward.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "decoder.cuh"
#include "train.cuh"

namespace srl {
namespace {

constexpr int kBlk = 64;      // keys / queries per block (= one KV page)
constexpr int kWarps = 4;
constexpr int kPadT = kBlk + 8;  // transposed tiles [HD][64 + 8]

__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&v);
}
// (x, y) -> bf16x2 hi = RN(x, y) and lo = RN(x - hi, y - hi)
__device__ __forceinline__ void split2(float x, float y, uint32_t& hi, uint32_t& lo) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(x, y);
  const float2 hf = __bfloat1622float2(h);
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = pack_bf16(x - hf.x, y - hf.y);
}
// B fragment (16 x 8, B[k][n]) from a row-major tile X[k][n] (n contiguous), pitch P
// elements: ldmatrix .trans -- the transposed copy of the tile is not needed.
__device__ __forceinline__ void frag_b_trans(uint32_t& b0, uint32_t& b1, const __nv_bfloat16* X, int P, int k0,
                                             int n0, int lane) {
  const __nv_bfloat16* p = X + (size_t)(k0 + (lane & 15)) * P + n0;
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0, %1}, [%2];"
               : "=r"(b0), "=r"(b1)
               : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(p))));
}
__device__ __forceinline__ uint32_t ld32(const __nv_bfloat16* p) {
  return *reinterpret_cast<const uint32_t*>(p);
}
// A fragment (16 x 16) of a row-major bf16 tile X[row][col] with pitch P.
__device__ __forceinline__ void frag_a(uint32_t (&a)[4], const __nv_bfloat16* X, int P, int r0, int c0,
                                       int lane) {
  const int r = r0 + (lane >> 2), c = c0 + (lane & 3) * 2;
  a[0] = ld32(X + r * P + c);
  a[1] = ld32(X + (r + 8) * P + c);
  a[2] = ld32(X + r * P + c + 8);
  a[3] = ld32(X + (r + 8) * P + c + 8);
}
// B fragment (16 x 8, B[k][n]) read from Y[n][k] (k contiguous), pitch P.
__device__ __forceinline__ void frag_b(uint32_t& b0, uint32_t& b1, const __nv_bfloat16* Y, int P, int n0,
                                       int k0, int lane) {
  const __nv_bfloat16* p = Y + (n0 + (lane >> 2)) * P + k0 + (lane & 3) * 2;
  b0 = ld32(p);
  b1 = ld32(p + 8);
}

__device__ __forceinline__ const __nv_bfloat16* page_row(const __nv_bfloat16* c, const int32_t* bt, int pps,
                                                         int slot, int pos, int nkv, int kh, int hd) {
  const int page = bt[(size_t)slot * pps + pos / kPageTokens];
  return c + (((size_t)page * nkv + kh) * kPageTokens + (pos % kPageTokens)) * hd;
}

// Stage 64 rows x HD of a bf16 source (row r -> src(r) or zeros past L) into
// X[64][HD + 8] and, if XT, its transpose XT[HD][64 + 8].
template <int HD>
constexpr int kNvB = kBlk * (HD / 8) / (kWarps * 32);  // uint4 per thread of a bf16 tile
template <int HD>
constexpr int kNvF = kBlk * (HD / 4) / (kWarps * 32);  // float4 per thread of an fp32 tile

// Load a 64 x HD bf16 tile (row r -> src(r), zeros past `valid`) into registers
// -- every load in flight together -- and store it into X[64][HD + 8] and,
// if XT, its transpose XT[HD][64 + 8].
template <int HD, class Src>
__device__ __forceinline__ void load_bf16(uint4 (&v)[kNvB<HD>], int valid, Src src) {
  constexpr int V8 = HD / 8;
#pragma unroll
  for (int k = 0; k < kNvB<HD>; ++k) {
    const int e = threadIdx.x + k * kWarps * 32, r = e / V8, c = (e % V8) * 8;
    v[k] = r < valid ? *reinterpret_cast<const uint4*>(src(r) + c) : make_uint4(0, 0, 0, 0);
  }
}
template <int HD>
__device__ __forceinline__ void store_bf16(__nv_bfloat16* X, __nv_bfloat16* XT, const uint4 (&v)[kNvB<HD>]) {
  constexpr int P = HD + 8, V8 = HD / 8;
#pragma unroll
  for (int k = 0; k < kNvB<HD>; ++k) {
    const int e = threadIdx.x + k * kWarps * 32, r = e / V8, c = (e % V8) * 8;
    *reinterpret_cast<uint4*>(X + r * P + c) = v[k];
    if (XT) {
      const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&v[k]);
#pragma unroll
      for (int i = 0; i < 8; ++i) XT[(c + i) * kPadT + r] = h[i];
    }
  }
}
template <int HD, class Src>
__device__ __forceinline__ void stage_bf16(__nv_bfloat16* X, __nv_bfloat16* XT, int valid, Src src) {
  uint4 v[kNvB<HD>];
  load_bf16<HD>(v, valid, src);
  store_bf16<HD>(X, XT, v);
}
// Same for an fp32 source (dO), rounded to bf16.
template <int HD, class Src>
__device__ __forceinline__ void load_f32(float4 (&v)[kNvF<HD>], int valid, Src src) {
  constexpr int V4 = HD / 4;
#pragma unroll
  for (int k = 0; k < kNvF<HD>; ++k) {
    const int e = threadIdx.x + k * kWarps * 32, r = e / V4, c = (e % V4) * 4;
    v[k] = r < valid ? *reinterpret_cast<const float4*>(src(r) + c) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
}
template <int HD>
__device__ __forceinline__ void store_f32(__nv_bfloat16* X, __nv_bfloat16* XT, const float4 (&v)[kNvF<HD>]) {
  constexpr int P = HD + 8, V4 = HD / 4;
#pragma unroll
  for (int k = 0; k < kNvF<HD>; ++k) {
    const int e = threadIdx.x + k * kWarps * 32, r = e / V4, c = (e % V4) * 4;
    const __nv_bfloat16 h[4] = {__float2bfloat16(v[k].x), __float2bfloat16(v[k].y), __float2bfloat16(v[k].z),
                                __float2bfloat16(v[k].w)};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      X[r * P + c + i] = h[i];
      if (XT) XT[(c + i) * kPadT + r] = h[i];
    }
  }
}
// Split: hi = bf16(v) into X / XT, lo = bf16(v - hi) into Xl / XlT.
template <int HD>
__device__ __forceinline__ void store_f32_split(__nv_bfloat16* X, __nv_bfloat16* XT, __nv_bfloat16* Xl,
                                                __nv_bfloat16* XlT, const float4 (&v)[kNvF<HD>]) {
  constexpr int P = HD + 8, V4 = HD / 4;
#pragma unroll
  for (int k = 0; k < kNvF<HD>; ++k) {
    const int e = threadIdx.x + k * kWarps * 32, r = e / V4, c = (e % V4) * 4;
    const float f[4] = {v[k].x, v[k].y, v[k].z, v[k].w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const __nv_bfloat16 h = __float2bfloat16(f[i]);
      const __nv_bfloat16 l = __float2bfloat16(f[i] - __bfloat162float(h));
      X[r * P + c + i] = h;
      Xl[r * P + c + i] = l;
      if (XT) {
        XT[(c + i) * kPadT + r] = h;
        XlT[(c + i) * kPadT + r] = l;
      }
    }
  }
}
template <int HD, class Src>
__device__ __forceinline__ void stage_f32(__nv_bfloat16* X, __nv_bfloat16* XT, int valid, Src src) {
  float4 v[kNvF<HD>];
  load_f32<HD>(v, valid, src);
  store_f32<HD>(X, XT, v);
}

template <int HD>
struct BwdSmem {
  static constexpr int P = HD + 8;
  static constexpr size_t tile = sizeof(__nv_bfloat16) * kBlk * P;
  static constexpr size_t tileT = sizeof(__nv_bfloat16) * HD * kPadT;
  static constexpr size_t vec = sizeof(float) * kBlk;
  // dkv: K, V, Q, dO, lse, D ; dq: Q, dO, K, V, lse, D (+ split: the lo half of dO).
  // The products that need a transposed operand read it with ldmatrix .trans,
  // so no transposed tiles: two CTAs per SM at hd 128 even in split mode.
  static constexpr size_t dkv = 4 * tile + 2 * vec;
  static constexpr size_t dq = 4 * tile + 2 * vec;
  static constexpr size_t dkv_split = dkv + tile;
  static constexpr size_t dq_split = dq + tile;
};

// SPLIT (the trainer's precise mode): dO, P and dS enter the MMAs as bf16
// hi + lo halves (P dO ~ Ph dOh + Ph dOl + Pl dOh), fp32-class products.
template <int HD, bool SPLIT>
__global__ void __launch_bounds__(kWarps * 32)
    attn_bwd_dkv_mma(const __nv_bfloat16* __restrict__ q, const float* __restrict__ d_o,
                     const float* __restrict__ lse, const float* __restrict__ D,
                     const __nv_bfloat16* __restrict__ kc, const __nv_bfloat16* __restrict__ vc,
                     const int32_t* __restrict__ seq_start, const int32_t* __restrict__ seq_len,
                     const int32_t* __restrict__ bt, int pps, int nq, int nkv, float scale,
                     float* __restrict__ dqkv) {
  using S = BwdSmem<HD>;
  constexpr int P = S::P, NT = HD / 8;
  extern __shared__ __align__(16) uint8_t smem[];
  __nv_bfloat16* Ks = reinterpret_cast<__nv_bfloat16*>(smem);
  __nv_bfloat16* Vs = reinterpret_cast<__nv_bfloat16*>(smem + S::tile);
  __nv_bfloat16* Qs = reinterpret_cast<__nv_bfloat16*>(smem + 2 * S::tile);
  __nv_bfloat16* dOs = reinterpret_cast<__nv_bfloat16*>(smem + 3 * S::tile);
  float* s_lse = reinterpret_cast<float*>(smem + 4 * S::tile);
  float* s_D = s_lse + kBlk;
  __nv_bfloat16* dOl = reinterpret_cast<__nv_bfloat16*>(smem + S::dkv);

  const int slot = blockIdx.y, kh = blockIdx.z;
  const int L = seq_len[slot], s0 = seq_start[slot];
  const int k0 = blockIdx.x * kBlk;
  if (k0 >= L) return;
  const int G = nq / nkv;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kvalid = min(kBlk, L - k0);
  stage_bf16<HD>(Ks, nullptr, kvalid, [&](int r) { return page_row(kc, bt, pps, slot, k0 + r, nkv, kh, HD); });
  stage_bf16<HD>(Vs, nullptr, kvalid, [&](int r) { return page_row(vc, bt, pps, slot, k0 + r, nkv, kh, HD); });

  float dk[NT][4], dv[NT][4];
#pragma unroll
  for (int n = 0; n < NT; ++n)
#pragma unroll
    for (int i = 0; i < 4; ++i) dk[n][i] = dv[n][i] = 0.f;
  const int kr = warp * 16;  // this warp's 16 keys (block-local)
  const int key_lo = k0 + kr + (lane >> 2), key_hi = key_lo + 8;

  // (query head g, query block q0) tiles in order; with HD = 64 the next
  // tile's loads are issued before this tile's MMAs (registers: Q 16, dO 32)
  constexpr bool kPipe = HD == 64;
  uint4 pq[kPipe ? kNvB<HD> : 1];
  float4 pd[kPipe ? kNvF<HD> : 1];
  float pl = 0.f, pD = 0.f;
  static_assert(kWarps * 32 >= kBlk, "one lse / D row per thread");
  auto fetch = [&](int g, int q0) {
    if constexpr (kPipe) {
      const int h = kh * G + g, qvalid = min(kBlk, L - q0);
      load_bf16<HD>(pq, qvalid, [&](int r) { return q + ((size_t)(s0 + q0 + r) * nq + h) * HD; });
      load_f32<HD>(pd, qvalid, [&](int r) { return d_o + ((size_t)(s0 + q0 + r) * nq + h) * HD; });
      const int r = threadIdx.x;
      pl = r < qvalid ? lse[(size_t)(s0 + q0 + r) * nq + h] : 0.f;
      pD = r < qvalid ? D[(size_t)(s0 + q0 + r) * nq + h] : 0.f;
    }
  };
  fetch(0, k0);
  for (int g = 0; g < G; ++g) {
    const int h = kh * G + g;
    for (int q0 = k0; q0 < L; q0 += kBlk) {
      const int qvalid = min(kBlk, L - q0);
      __syncthreads();  // previous tiles consumed
      if constexpr (kPipe) {
        store_bf16<HD>(Qs, nullptr, pq);
        if constexpr (SPLIT) store_f32_split<HD>(dOs, nullptr, dOl, nullptr, pd);
        else store_f32<HD>(dOs, nullptr, pd);
        if (threadIdx.x < kBlk) {
          s_lse[threadIdx.x] = pl;
          s_D[threadIdx.x] = pD;
        }
      } else {
        stage_bf16<HD>(Qs, nullptr, qvalid, [&](int r) { return q + ((size_t)(s0 + q0 + r) * nq + h) * HD; });
        if constexpr (SPLIT) {
          float4 v[kNvF<HD>];
          load_f32<HD>(v, qvalid, [&](int r) { return d_o + ((size_t)(s0 + q0 + r) * nq + h) * HD; });
          store_f32_split<HD>(dOs, nullptr, dOl, nullptr, v);
        } else {
          stage_f32<HD>(dOs, nullptr, qvalid, [&](int r) { return d_o + ((size_t)(s0 + q0 + r) * nq + h) * HD; });
        }
        for (int r = threadIdx.x; r < kBlk; r += kWarps * 32) {
          s_lse[r] = r < qvalid ? lse[(size_t)(s0 + q0 + r) * nq + h] : 0.f;
          s_D[r] = r < qvalid ? D[(size_t)(s0 + q0 + r) * nq + h] : 0.f;
        }
      }
      __syncthreads();
      if constexpr (kPipe) {  // the next tile's loads fly during this tile's MMAs
        int g2 = g, q2 = q0 + kBlk;
        if (q2 >= L) { ++g2; q2 = k0; }
        if (g2 < G) fetch(g2, q2);
      }
      // S^T = K_w Q^T and dP^T = V_w dO^T: [16 keys x 64 queries]
      float st[8][4], dpt[8][4];
#pragma unroll
      for (int n = 0; n < 8; ++n)
#pragma unroll
        for (int i = 0; i < 4; ++i) st[n][i] = dpt[n][i] = 0.f;
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk) {
        uint32_t ak[4], av[4];
        frag_a(ak, Ks, P, kr, kk * 16, lane);
        frag_a(av, Vs, P, kr, kk * 16, lane);
#pragma unroll
        for (int n = 0; n < 8; ++n) {
          uint32_t b0, b1;
          frag_b(b0, b1, Qs, P, n * 8, kk * 16, lane);
          mma16816(st[n], ak, b0, b1);
          frag_b(b0, b1, dOs, P, n * 8, kk * 16, lane);
          mma16816(dpt[n], av, b0, b1);
          if constexpr (SPLIT) {
            frag_b(b0, b1, dOl, P, n * 8, kk * 16, lane);
            mma16816(dpt[n], av, b0, b1);
          }
        }
      }
      // P^T and dS^T (scaled), causal: query position >= key position
#pragma unroll
      for (int n = 0; n < 8; ++n) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int ql = n * 8 + (lane & 3) * 2 + (i & 1);
          const int qpos = q0 + ql, kpos = i < 2 ? key_lo : key_hi;
          const bool ok = ql < qvalid && qpos >= kpos && kpos < L;
          const float p = ok ? __expf(st[n][i] * scale - s_lse[ql]) : 0.f;
          st[n][i] = p;
          dpt[n][i] = p * (dpt[n][i] - s_D[ql]) * scale;
        }
      }
      // dV += P^T dO, dK += dS^T Q   (k = 64 queries in 4 steps of 16)
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        uint32_t ap[4], ad[4], apl[4], adl[4];
        if constexpr (SPLIT) {
          split2(st[2 * ks][0], st[2 * ks][1], ap[0], apl[0]);
          split2(st[2 * ks][2], st[2 * ks][3], ap[1], apl[1]);
          split2(st[2 * ks + 1][0], st[2 * ks + 1][1], ap[2], apl[2]);
          split2(st[2 * ks + 1][2], st[2 * ks + 1][3], ap[3], apl[3]);
          split2(dpt[2 * ks][0], dpt[2 * ks][1], ad[0], adl[0]);
          split2(dpt[2 * ks][2], dpt[2 * ks][3], ad[1], adl[1]);
          split2(dpt[2 * ks + 1][0], dpt[2 * ks + 1][1], ad[2], adl[2]);
          split2(dpt[2 * ks + 1][2], dpt[2 * ks + 1][3], ad[3], adl[3]);
        } else {
          ap[0] = pack_bf16(st[2 * ks][0], st[2 * ks][1]);
          ap[1] = pack_bf16(st[2 * ks][2], st[2 * ks][3]);
          ap[2] = pack_bf16(st[2 * ks + 1][0], st[2 * ks + 1][1]);
          ap[3] = pack_bf16(st[2 * ks + 1][2], st[2 * ks + 1][3]);
          ad[0] = pack_bf16(dpt[2 * ks][0], dpt[2 * ks][1]);
          ad[1] = pack_bf16(dpt[2 * ks][2], dpt[2 * ks][3]);
          ad[2] = pack_bf16(dpt[2 * ks + 1][0], dpt[2 * ks + 1][1]);
          ad[3] = pack_bf16(dpt[2 * ks + 1][2], dpt[2 * ks + 1][3]);
        }
#pragma unroll
        for (int n = 0; n < NT; ++n) {
          uint32_t b0, b1;
          frag_b_trans(b0, b1, dOs, P, ks * 16, n * 8, lane);
          mma16816(dv[n], ap, b0, b1);
          if constexpr (SPLIT) {
            mma16816(dv[n], apl, b0, b1);
            frag_b_trans(b0, b1, dOl, P, ks * 16, n * 8, lane);
            mma16816(dv[n], ap, b0, b1);
          }
          frag_b_trans(b0, b1, Qs, P, ks * 16, n * 8, lane);
          mma16816(dk[n], ad, b0, b1);
          if constexpr (SPLIT) mma16816(dk[n], adl, b0, b1);
        }
      }
    }
  }
  // write dk / dv rows (fp32, pre-RoPE rotation applied by the caller)
  const int qkv = (nq + 2 * nkv) * HD;
#pragma unroll
  for (int n = 0; n < NT; ++n) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int kpos = i < 2 ? key_lo : key_hi;
      if (kpos >= L) continue;
      const int d = n * 8 + (lane & 3) * 2 + (i & 1);
      float* row = dqkv + (size_t)(s0 + kpos) * qkv;
      row[nq * HD + kh * HD + d] = dk[n][i];
      row[(nq + nkv) * HD + kh * HD + d] = dv[n][i];
    }
  }
}

template <int HD, bool SPLIT>
__global__ void __launch_bounds__(kWarps * 32)
    attn_bwd_dq_mma(const __nv_bfloat16* __restrict__ q, const float* __restrict__ d_o,
                    const float* __restrict__ lse, const float* __restrict__ D,
                    const __nv_bfloat16* __restrict__ kc, const __nv_bfloat16* __restrict__ vc,
                    const int32_t* __restrict__ seq_start, const int32_t* __restrict__ seq_len,
                    const int32_t* __restrict__ bt, int pps, int nq, int nkv, float scale,
                    float* __restrict__ dqkv) {
  using S = BwdSmem<HD>;
  constexpr int P = S::P, NT = HD / 8;
  extern __shared__ __align__(16) uint8_t smem[];
  __nv_bfloat16* Qs = reinterpret_cast<__nv_bfloat16*>(smem);
  __nv_bfloat16* dOs = reinterpret_cast<__nv_bfloat16*>(smem + S::tile);
  __nv_bfloat16* Ks = reinterpret_cast<__nv_bfloat16*>(smem + 2 * S::tile);
  __nv_bfloat16* Vs = reinterpret_cast<__nv_bfloat16*>(smem + 3 * S::tile);
  float* s_lse = reinterpret_cast<float*>(smem + 4 * S::tile);
  float* s_D = s_lse + kBlk;
  __nv_bfloat16* dOl = reinterpret_cast<__nv_bfloat16*>(smem + S::dq);

  const int slot = blockIdx.y, h = blockIdx.z;
  const int L = seq_len[slot], s0 = seq_start[slot];
  const int q0 = blockIdx.x * kBlk;
  if (q0 >= L) return;
  const int kh = h / (nq / nkv);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qvalid = min(kBlk, L - q0);
  stage_bf16<HD>(Qs, nullptr, qvalid, [&](int r) { return q + ((size_t)(s0 + q0 + r) * nq + h) * HD; });
  if constexpr (SPLIT) {
    float4 v[kNvF<HD>];
    load_f32<HD>(v, qvalid, [&](int r) { return d_o + ((size_t)(s0 + q0 + r) * nq + h) * HD; });
    store_f32_split<HD>(dOs, nullptr, dOl, nullptr, v);
  } else {
    stage_f32<HD>(dOs, nullptr, qvalid, [&](int r) { return d_o + ((size_t)(s0 + q0 + r) * nq + h) * HD; });
  }
  for (int r = threadIdx.x; r < kBlk; r += kWarps * 32) {
    s_lse[r] = r < qvalid ? lse[(size_t)(s0 + q0 + r) * nq + h] : 0.f;
    s_D[r] = r < qvalid ? D[(size_t)(s0 + q0 + r) * nq + h] : 0.f;
  }
  const int qr = warp * 16;
  const int ql_lo = qr + (lane >> 2), ql_hi = ql_lo + 8;
  float dq[NT][4];
#pragma unroll
  for (int n = 0; n < NT; ++n)
#pragma unroll
    for (int i = 0; i < 4; ++i) dq[n][i] = 0.f;

  // with HD = 64 the next key block's K / V loads fly during this block's MMAs
  constexpr bool kPipe = HD == 64;
  uint4 pk[kPipe ? kNvB<HD> : 1], pv[kPipe ? kNvB<HD> : 1];
  auto fetch = [&](int k0) {
    if constexpr (kPipe) {
      const int kvalid = min(kBlk, L - k0);
      load_bf16<HD>(pk, kvalid, [&](int r) { return page_row(kc, bt, pps, slot, k0 + r, nkv, kh, HD); });
      load_bf16<HD>(pv, kvalid, [&](int r) { return page_row(vc, bt, pps, slot, k0 + r, nkv, kh, HD); });
    }
  };
  fetch(0);
  for (int k0 = 0; k0 <= q0; k0 += kBlk) {
    const int kvalid = min(kBlk, L - k0);
    __syncthreads();
    if constexpr (kPipe) {
      store_bf16<HD>(Ks, nullptr, pk);
      store_bf16<HD>(Vs, nullptr, pv);
    } else {
      stage_bf16<HD>(Ks, nullptr, kvalid, [&](int r) { return page_row(kc, bt, pps, slot, k0 + r, nkv, kh, HD); });
      stage_bf16<HD>(Vs, nullptr, kvalid, [&](int r) { return page_row(vc, bt, pps, slot, k0 + r, nkv, kh, HD); });
    }
    __syncthreads();
    if constexpr (kPipe) {
      if (k0 + kBlk <= q0) fetch(k0 + kBlk);
    }
    float s[8][4], dp[8][4];
#pragma unroll
    for (int n = 0; n < 8; ++n)
#pragma unroll
      for (int i = 0; i < 4; ++i) s[n][i] = dp[n][i] = 0.f;
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk) {
      uint32_t aq[4], ad[4], adl[4];
      frag_a(aq, Qs, P, qr, kk * 16, lane);
      frag_a(ad, dOs, P, qr, kk * 16, lane);
      if constexpr (SPLIT) frag_a(adl, dOl, P, qr, kk * 16, lane);
#pragma unroll
      for (int n = 0; n < 8; ++n) {
        uint32_t b0, b1;
        frag_b(b0, b1, Ks, P, n * 8, kk * 16, lane);
        mma16816(s[n], aq, b0, b1);
        frag_b(b0, b1, Vs, P, n * 8, kk * 16, lane);
        mma16816(dp[n], ad, b0, b1);
        if constexpr (SPLIT) mma16816(dp[n], adl, b0, b1);
      }
    }
#pragma unroll
    for (int n = 0; n < 8; ++n) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int kl = n * 8 + (lane & 3) * 2 + (i & 1);
        const int ql = i < 2 ? ql_lo : ql_hi;
        const int kpos = k0 + kl, qpos = q0 + ql;
        const bool ok = kl < kvalid && kpos <= qpos && ql < qvalid;
        const float p = ok ? __expf(s[n][i] * scale - s_lse[ql]) : 0.f;
        dp[n][i] = p * (dp[n][i] - s_D[ql]) * scale;
      }
    }
    // dQ += dS K  (k = 64 keys in 4 steps of 16)
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      uint32_t a[4], al[4];
      if constexpr (SPLIT) {
        split2(dp[2 * ks][0], dp[2 * ks][1], a[0], al[0]);
        split2(dp[2 * ks][2], dp[2 * ks][3], a[1], al[1]);
        split2(dp[2 * ks + 1][0], dp[2 * ks + 1][1], a[2], al[2]);
        split2(dp[2 * ks + 1][2], dp[2 * ks + 1][3], a[3], al[3]);
      } else {
        a[0] = pack_bf16(dp[2 * ks][0], dp[2 * ks][1]);
        a[1] = pack_bf16(dp[2 * ks][2], dp[2 * ks][3]);
        a[2] = pack_bf16(dp[2 * ks + 1][0], dp[2 * ks + 1][1]);
        a[3] = pack_bf16(dp[2 * ks + 1][2], dp[2 * ks + 1][3]);
      }
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        uint32_t b0, b1;
        frag_b_trans(b0, b1, Ks, P, ks * 16, n * 8, lane);
        mma16816(dq[n], a, b0, b1);
        if constexpr (SPLIT) mma16816(dq[n], al, b0, b1);
      }
    }
  }
  const int qkv = (nq + 2 * nkv) * HD;
#pragma unroll
  for (int n = 0; n < NT; ++n) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int ql = i < 2 ? ql_lo : ql_hi;
      if (ql >= qvalid) continue;
      const int d = n * 8 + (lane & 3) * 2 + (i & 1);
      dqkv[(size_t)(s0 + q0 + ql) * qkv + h * HD + d] = dq[n][i];
    }
  }
}

// Forward over packed sequences: CTA = (64-query block, sequence, query head),
// online softmax over the causal key blocks; O (bf16) and lse (natural log of
// the scaled scores' partition sum) per (row, head), as the backward expects.
// A key block is one 64-token page: K and V arrive row-major by cp.async into
// a double buffer (block j + 1 streams in while block j is computed), Q lives
// in registers as ldmatrix fragments, K^T and V are read with ldmatrix
// (.trans for V) -- no transposed staging.  Only blocks that reach past the
// block's first query position (or past the context) are masked.
template <int HD>
struct FwdSmem {
  static constexpr int P = HD + 8;  // row pitch (elements): conflict-free ldmatrix
  static constexpr size_t tile = sizeof(__nv_bfloat16) * kBlk * P;
  static constexpr size_t total = 4 * tile;  // K0 V0 K1 V1 (Q is staged in K1 first)
};

__device__ __forceinline__ void cp16_zfill(void* dst, const void* src, bool ok) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(static_cast<uint32_t>(
                   __cvta_generic_to_shared(dst))),
               "l"(src), "r"(ok ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const __nv_bfloat16* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(p))));
}
__device__ __forceinline__ void ldsm_x4_trans(uint32_t (&r)[4], const __nv_bfloat16* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(p))));
}

// Segment y: query rows seq_start[y] .. + seq_len[y] at positions pos0[y] ..
// (0 when pos0 is null) of slot seg_slot[y] (y when null); keys 0 .. the last
// query's position from the slot's pages.  The trainer passes whole packed
// sequences; a prefill round passes each new prompt (and recompute chunks).
template <int HD>
__global__ void __launch_bounds__(kWarps * 32)
    attn_fwd_mma(const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ kc,
                 const __nv_bfloat16* __restrict__ vc, const int32_t* __restrict__ seq_start,
                 const int32_t* __restrict__ seq_len, const int32_t* __restrict__ seg_pos0,
                 const int32_t* __restrict__ seg_slot, const int32_t* __restrict__ bt, int pps, int nq,
                 int nkv, float scale, __nv_bfloat16* __restrict__ out, float* __restrict__ lse_out,
                 int split_p, int out_lo) {
  using S = FwdSmem<HD>;
  constexpr int P = S::P, NT = HD / 8, C8 = HD / 8;
  static_assert(kBlk == kPageTokens, "a key block is one page");
  extern __shared__ __align__(16) uint8_t smem[];
  __nv_bfloat16* const sb = reinterpret_cast<__nv_bfloat16*>(smem);
  constexpr int TE = kBlk * P;  // elements per tile
  const int y = blockIdx.y, h = blockIdx.z;
  const int nrows = seq_len[y], s0 = seq_start[y];
  const int slot = seg_slot ? seg_slot[y] : y, p0 = seg_pos0 ? seg_pos0[y] : 0;
  const int q0 = blockIdx.x * kBlk;  // first query of the block (segment-local)
  if (q0 >= nrows) return;
  const int kh = h / (nq / nkv);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qvalid = min(kBlk, nrows - q0);
  const int kend = p0 + q0 + qvalid;  // keys [0, kend): up to the block's last query position
  const int nblk = (kend + kBlk - 1) / kBlk;
  // key block j (page j of the slot) -> K / V buffers (j & 1); rows past the
  // context are zero-filled (P is 0 there, but 0 x stale NaN bits is NaN)
  auto load_block = [&](int j) {
    const int valid = min(kBlk, kend - j * kBlk);
    const size_t page = (size_t)bt[(size_t)slot * pps + j];
    const __nv_bfloat16* kg = kc + (page * nkv + kh) * kPageTokens * HD;
    const __nv_bfloat16* vg = vc + (page * nkv + kh) * kPageTokens * HD;
    __nv_bfloat16* kd = sb + (size_t)(2 * (j & 1)) * TE;
    __nv_bfloat16* vd = kd + TE;
#pragma unroll
    for (int it = 0; it < kBlk * C8 / (kWarps * 32); ++it) {
      const int e = threadIdx.x + it * kWarps * 32, r = e / C8, c = (e % C8) * 8;
      const bool ok = r < valid;
      cp16_zfill(kd + r * P + c, ok ? kg + r * HD + c : kg, ok);
      cp16_zfill(vd + r * P + c, ok ? vg + r * HD + c : vg, ok);
    }
  };
  {  // Q -> the K1 buffer, with block 0
    __nv_bfloat16* qd = sb + 2 * TE;
    const __nv_bfloat16* qg = q + ((size_t)(s0 + q0) * nq + h) * HD;
#pragma unroll
    for (int it = 0; it < kBlk * C8 / (kWarps * 32); ++it) {
      const int e = threadIdx.x + it * kWarps * 32, r = e / C8, c = (e % C8) * 8;
      const bool ok = r < qvalid;
      cp16_zfill(qd + r * P + c, ok ? qg + (size_t)r * nq * HD + c : qg, ok);
    }
  }
  load_block(0);
  asm volatile("cp.async.commit_group;" ::: "memory");
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  const int qr = warp * 16;
  uint32_t qf[HD / 16][4];
#pragma unroll
  for (int kk = 0; kk < HD / 16; ++kk)
    ldsm_x4(qf[kk], sb + 2 * TE + (qr + (lane & 15)) * P + kk * 16 + (lane >> 4) * 8);
  __syncthreads();  // the Q staging (buffer 1) is refilled below
  const int ql_lo = qr + (lane >> 2), ql_hi = ql_lo + 8;
  float o[NT][4];
#pragma unroll
  for (int n = 0; n < NT; ++n)
#pragma unroll
    for (int i = 0; i < 4; ++i) o[n][i] = 0.f;
  float m_lo = -INFINITY, m_hi = -INFINITY, l_lo = 0.f, l_hi = 0.f;

  for (int j = 0; j < nblk; ++j) {
    if (j + 1 < nblk) {
      load_block(j + 1);
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const __nv_bfloat16* Ks = sb + (size_t)(2 * (j & 1)) * TE;
    const __nv_bfloat16* Vs = Ks + TE;
    const int k0 = j * kBlk;
    const int kvalid = min(kBlk, kend - k0);
    float s[8][4];
#pragma unroll
    for (int n = 0; n < 8; ++n)
#pragma unroll
      for (int i = 0; i < 4; ++i) s[n][i] = 0.f;
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk) {
#pragma unroll
      for (int n = 0; n < 8; n += 2) {  // two 8-key column blocks per ldmatrix.x4
        uint32_t b[4];
        ldsm_x4(b, Ks + (n * 8 + (lane & 7) + ((lane >> 4) << 3)) * P + kk * 16 + ((lane >> 3) & 1) * 8);
        mma16816(s[n], qf[kk], b[0], b[1]);
        mma16816(s[n + 1], qf[kk], b[2], b[3]);
      }
    }
    // scale (+ causal / context mask where the block reaches past the first
    // query's position), new running max per row (a row's 64 columns live on
    // the 4 lanes of a quad)
    const bool masked = k0 + kBlk - 1 > p0 + q0 || kvalid < kBlk;
    float mx_lo = m_lo, mx_hi = m_hi;
#pragma unroll
    for (int n = 0; n < 8; ++n) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int kl = n * 8 + (lane & 3) * 2 + (i & 1);
        const int ql = i < 2 ? ql_lo : ql_hi;
        const bool ok = !masked || (kl < kvalid && k0 + kl <= p0 + q0 + ql);
        s[n][i] = ok ? s[n][i] * scale : -INFINITY;
        if (i < 2) mx_lo = fmaxf(mx_lo, s[n][i]);
        else mx_hi = fmaxf(mx_hi, s[n][i]);
      }
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
    for (int n = 0; n < 8; ++n) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float mm = i < 2 ? m_lo : m_hi;
        const float p = s[n][i] == -INFINITY ? 0.f : __expf(s[n][i] - mm);
        s[n][i] = p;
        if (i < 2) sum_lo += p;
        else sum_hi += p;
      }
    }
    l_lo = l_lo * c_lo + sum_lo;  // per-lane partial sums; combined across the quad at the end
    l_hi = l_hi * c_hi + sum_hi;
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      o[n][0] *= c_lo; o[n][1] *= c_lo;
      o[n][2] *= c_hi; o[n][3] *= c_hi;
    }
    // O += P V: P enters as bf16 (optionally + its lo residual, split_p); V[key][d]
    // is the row-major B operand, read transposed by ldmatrix .trans
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      uint32_t ah[4], al[4];
      split2(s[2 * ks][0], s[2 * ks][1], ah[0], al[0]);
      split2(s[2 * ks][2], s[2 * ks][3], ah[1], al[1]);
      split2(s[2 * ks + 1][0], s[2 * ks + 1][1], ah[2], al[2]);
      split2(s[2 * ks + 1][2], s[2 * ks + 1][3], ah[3], al[3]);
#pragma unroll
      for (int n = 0; n < NT; n += 2) {  // two 8-dim column blocks per ldmatrix.x4.trans
        uint32_t b[4];
        ldsm_x4_trans(b, Vs + (ks * 16 + (lane & 7) + ((lane >> 3) & 1) * 8) * P + n * 8 + (lane >> 4) * 8);
        mma16816(o[n], ah, b[0], b[1]);
        mma16816(o[n + 1], ah, b[2], b[3]);
        if (split_p) {
          mma16816(o[n], al, b[0], b[1]);
          mma16816(o[n + 1], al, b[2], b[3]);
        }
      }
    }
    __syncthreads();  // buffer (j & 1) is refilled with block j + 2 next iteration
  }
#pragma unroll
  for (int off = 1; off <= 2; off <<= 1) {
    l_lo += __shfl_xor_sync(0xffffffffu, l_lo, off);
    l_hi += __shfl_xor_sync(0xffffffffu, l_hi, off);
  }
  const float inv_lo = l_lo > 0.f ? 1.f / l_lo : 0.f, inv_hi = l_hi > 0.f ? 1.f / l_hi : 0.f;
  // out row stride nq HD + out_lo; split (out_lo > 0): lo = bf16(o - hi) at + out_lo
  const int ldo = nq * HD + out_lo;
#pragma unroll
  for (int n = 0; n < NT; ++n) {
    const int d = n * 8 + (lane & 3) * 2;
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const int ql = hh ? ql_hi : ql_lo;
      if (ql >= qvalid) continue;
      const float inv = hh ? inv_hi : inv_lo;
      const float v0 = o[n][2 * hh] * inv, v1 = o[n][2 * hh + 1] * inv;
      __nv_bfloat16* dst = out + (size_t)(s0 + q0 + ql) * ldo + h * HD + d;
      const __nv_bfloat162 hi = __floats2bfloat162_rn(v0, v1);
      *reinterpret_cast<__nv_bfloat162*>(dst) = hi;
      if (out_lo) {
        const float2 hf = __bfloat1622float2(hi);
        *reinterpret_cast<__nv_bfloat162*>(dst + out_lo) = __floats2bfloat162_rn(v0 - hf.x, v1 - hf.y);
      }
    }
  }
  if (lse_out && (lane & 3) == 0) {
    if (ql_lo < qvalid) lse_out[(size_t)(s0 + q0 + ql_lo) * nq + h] = m_lo + logf(l_lo);
    if (ql_hi < qvalid) lse_out[(size_t)(s0 + q0 + ql_hi) * nq + h] = m_hi + logf(l_hi);
  }
}

template <int HD>
cudaError_t launch_fwd_t(const __nv_bfloat16* q, const __nv_bfloat16* kc, const __nv_bfloat16* vc,
                         const int32_t* seq_start, const int32_t* seq_len, const int32_t* pos0,
                         const int32_t* slot, const int32_t* bt, int pps, int n_seq, int max_rows, int nq,
                         int nkv, float scale, __nv_bfloat16* out, float* lse, int out_lo, cudaStream_t st) {
  static const bool attr = cudaFuncSetAttribute(attn_fwd_mma<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                (int)FwdSmem<HD>::total) == cudaSuccess;
  // P as hi + lo bf16 halves (default; vs the fp64 oracle at 0.5B the
  // log-prob error drops from 1.65e-2 to 1.04e-2 max, as with the CUDA-core
  // kernel); SRL_ATTN_SPLIT=0: a single bf16 P (A/B)
  static const int split = [] {
    const char* e = std::getenv("SRL_ATTN_SPLIT");
    return e && e[0] == '0' ? 0 : 1;
  }();
  if (!attr) return cudaErrorInvalidValue;
  attn_fwd_mma<HD><<<dim3((max_rows + kBlk - 1) / kBlk, n_seq, nq), kWarps * 32, FwdSmem<HD>::total, st>>>(
      q, kc, vc, seq_start, seq_len, pos0, slot, bt, pps, nq, nkv, scale, out, lse, split, out_lo);
  return cudaGetLastError();
}

template <int HD, bool SPLIT>
cudaError_t launch_t(const __nv_bfloat16* q, const float* d_o, const float* lse, const float* D,
                     const __nv_bfloat16* kc, const __nv_bfloat16* vc, const int32_t* seq_start,
                     const int32_t* seq_len, const int32_t* bt, int pps, int n_seq, int nq, int nkv,
                     float scale, float* dqkv, cudaStream_t st) {
  using S = BwdSmem<HD>;
  constexpr size_t sk = SPLIT ? S::dkv_split : S::dkv, sq = SPLIT ? S::dq_split : S::dq;
  static const bool attr =
      cudaFuncSetAttribute(attn_bwd_dkv_mma<HD, SPLIT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sk) ==
          cudaSuccess &&
      cudaFuncSetAttribute(attn_bwd_dq_mma<HD, SPLIT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sq) ==
          cudaSuccess;
  if (!attr) return cudaErrorInvalidValue;
  // pages per sequence = 64-token blocks per sequence
  attn_bwd_dkv_mma<HD, SPLIT><<<dim3(pps, n_seq, nkv), kWarps * 32, sk, st>>>(
      q, d_o, lse, D, kc, vc, seq_start, seq_len, bt, pps, nq, nkv, scale, dqkv);
  attn_bwd_dq_mma<HD, SPLIT><<<dim3(pps, n_seq, nq), kWarps * 32, sq, st>>>(
      q, d_o, lse, D, kc, vc, seq_start, seq_len, bt, pps, nq, nkv, scale, dqkv);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_attention_bwd_mma(const __nv_bfloat16* q, const float* d_o, const float* lse,
                                     const float* D, const __nv_bfloat16* kc, const __nv_bfloat16* vc,
                                     const int32_t* seq_start, const int32_t* seq_len,
                                     const int32_t* block_table, int pages_per_seq, int n_seq, int nq,
                                     int nkv, int hd, float* dqkv, cudaStream_t st, bool split) {
  const float scale = 1.0f / sqrtf((float)hd);
#define SRL_BWD_ARGS q, d_o, lse, D, kc, vc, seq_start, seq_len, block_table, pages_per_seq, n_seq, nq, nkv, scale, dqkv, st
  if (hd == 64) return split ? launch_t<64, true>(SRL_BWD_ARGS) : launch_t<64, false>(SRL_BWD_ARGS);
  if (hd == 128) return split ? launch_t<128, true>(SRL_BWD_ARGS) : launch_t<128, false>(SRL_BWD_ARGS);
#undef SRL_BWD_ARGS
  return cudaErrorInvalidValue;
}

}  // namespace srl

namespace srl {
cudaError_t launch_attention_fwd_mma(const __nv_bfloat16* q, const __nv_bfloat16* kc, const __nv_bfloat16* vc,
                                     const int32_t* seq_start, const int32_t* seq_len,
                                     const int32_t* block_table, int pages_per_seq, int n_seq, int nq,
                                     int nkv, int hd, __nv_bfloat16* out, float* lse, cudaStream_t st,
                                     const int32_t* seg_pos0, const int32_t* seg_slot, int max_rows,
                                     int out_lo) {
  const float scale = 1.0f / sqrtf((float)hd);
  if (max_rows <= 0) max_rows = pages_per_seq * kBlk;
  if (hd == 64)
    return launch_fwd_t<64>(q, kc, vc, seq_start, seq_len, seg_pos0, seg_slot, block_table, pages_per_seq,
                            n_seq, max_rows, nq, nkv, scale, out, lse, out_lo, st);
  if (hd == 128)
    return launch_fwd_t<128>(q, kc, vc, seq_start, seq_len, seg_pos0, seg_slot, block_table, pages_per_seq,
                             n_seq, max_rows, nq, nkv, scale, out, lse, out_lo, st);
  return cudaErrorInvalidValue;
}
}  // namespace srl
