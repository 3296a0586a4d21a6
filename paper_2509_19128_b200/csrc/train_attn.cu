#include <cstdlib>
// train_attn.cu -- causal GQA attention of the trainer (forward and
// backward) and of a prefill round's prompt rows, on the tensor cores
// (mma.sync m16n8k16 bf16 -> fp32), FlashAttention-2 tiling, deterministic.
//
// The trainer's forward keeps q (post-RoPE, bf16), the attention output o,
// the per-(row, head) log-sum-exp and writes K/V into a paged cache (one
// 64-token page per block of a sequence); every tile moves by cp.async into
// a double buffer and every fragment comes from ldmatrix (see the forward and
// the backward sections below).  Four warps per CTA, each owning 16 rows.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "decoder.cuh"
#include "train.cuh"

namespace srl {
namespace {

constexpr int kBlk = 64;      // keys / queries per block (= one KV page)
constexpr int kWarps = 4;

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

// ---------------------------------------------------------------- backward
// With D = rowsum(dO * O) (the dot pass, which also rounds dO to bf16 hi + lo):
//   P  = exp(scale * Q K^T - lse)          (causal)
//   dV = P^T dO,   dP = dO V^T,   dS = P * (dP - D)
//   dQ = scale * dS K,   dK = scale * dS^T Q
// Two deterministic kernels (no atomics), every operand tile streamed by
// cp.async into a double buffer (the next tile lands under this tile's MMAs),
// fragments by ldmatrix (.trans where the product needs the transpose):
//   attn_bwd_dkv_mma : CTA = (64-key block, sequence, KV head), 4 warps x 16
//                      keys; loops over the G query heads x the causal query
//                      tiles (QB rows: 64, 32 in split mode);
//   attn_bwd_dq_mma  : CTA = (64-query block, sequence, query head), 4 warps x
//                      16 queries; loops over the causal key pages.
// SPLIT (the trainer's precise mode): dO, P and dS enter as bf16 hi + lo
// (P dO ~ Ph dOh + Pl dOh + Ph dOl; dS Q ~ (dSh + dSl) Q; Q, K, V are bf16).
template <int HD, bool SPLIT>
struct DkvSmem {
  static constexpr int P = HD + 8;
  static constexpr int QB = SPLIT ? 32 : 64;                 // query rows per tile
  static constexpr size_t kv = sizeof(__nv_bfloat16) * kBlk * P;  // K or V
  static constexpr size_t qt = sizeof(__nv_bfloat16) * QB * P;    // Q, dO or dOl tile
  static constexpr size_t stage = (SPLIT ? 3 : 2) * qt + 2 * sizeof(float) * QB;  // + lse, D
  static constexpr size_t total = 2 * kv + 2 * stage;
};
template <int HD, bool SPLIT>
struct DqSmem {
  static constexpr int P = HD + 8;
  static constexpr size_t tile = sizeof(__nv_bfloat16) * kBlk * P;
  static constexpr size_t total = (SPLIT ? 2 : 1) * tile + 4 * tile;  // dO [dOl] K0 V0 K1 V1
};

// A fragment (16 x 16) of the C-layout fp32 values c[2 ks], c[2 ks + 1]
// (8-column blocks of a 16-row accumulator) as bf16 (+ the lo residual)
template <bool SPLIT>
__device__ __forceinline__ void c_to_a(const float (&c0)[4], const float (&c1)[4], uint32_t (&a)[4],
                                       uint32_t (&al)[4]) {
  if constexpr (SPLIT) {
    split2(c0[0], c0[1], a[0], al[0]);
    split2(c0[2], c0[3], a[1], al[1]);
    split2(c1[0], c1[1], a[2], al[2]);
    split2(c1[2], c1[3], a[3], al[3]);
  } else {
    a[0] = pack_bf16(c0[0], c0[1]);
    a[1] = pack_bf16(c0[2], c0[3]);
    a[2] = pack_bf16(c1[0], c1[1]);
    a[3] = pack_bf16(c1[2], c1[3]);
  }
}

template <int HD, bool SPLIT>
__global__ void __launch_bounds__(kWarps * 32)
    attn_bwd_dkv_mma(const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ dob,
                     const __nv_bfloat16* __restrict__ dol, const float* __restrict__ lse,
                     const float* __restrict__ D, const __nv_bfloat16* __restrict__ kc,
                     const __nv_bfloat16* __restrict__ vc, const int32_t* __restrict__ seq_start,
                     const int32_t* __restrict__ seq_len, const int32_t* __restrict__ bt, int pps, int nq,
                     int nkv, float scale, float* __restrict__ dqkv) {
  using S = DkvSmem<HD, SPLIT>;
  constexpr int P = S::P, NT = HD / 8, QB = S::QB, C8 = HD / 8, QN = QB / 8;
  extern __shared__ __align__(16) uint8_t smem[];
  __nv_bfloat16* Ks = reinterpret_cast<__nv_bfloat16*>(smem);
  __nv_bfloat16* Vs = reinterpret_cast<__nv_bfloat16*>(smem + S::kv);
  auto stage_base = [&](int b) { return smem + 2 * S::kv + (size_t)b * S::stage; };
  const int slot = blockIdx.y, kh = blockIdx.z;
  const int L = seq_len[slot], s0 = seq_start[slot];
  const int k0 = blockIdx.x * kBlk;
  if (k0 >= L) return;
  const int G = nq / nkv;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kvalid = min(kBlk, L - k0);
  {  // K, V: this block's page (rows past L zero)
    const size_t page = (size_t)bt[(size_t)slot * pps + blockIdx.x];
    const __nv_bfloat16* kg = kc + (page * nkv + kh) * kPageTokens * HD;
    const __nv_bfloat16* vg = vc + (page * nkv + kh) * kPageTokens * HD;
#pragma unroll
    for (int it = 0; it < kBlk * C8 / (kWarps * 32); ++it) {
      const int e = threadIdx.x + it * kWarps * 32, r = e / C8, c = (e % C8) * 8;
      const bool ok = r < kvalid;
      cp16_zfill(Ks + r * P + c, ok ? kg + r * HD + c : kg, ok);
      cp16_zfill(Vs + r * P + c, ok ? vg + r * HD + c : vg, ok);
    }
  }
  // tile it = (query head g, query rows q0 ..): g = it / nqb, q0 = k0 + (it % nqb) QB
  const int nqb = (L - k0 + QB - 1) / QB, n_it = G * nqb;
  auto tile_rows = [&](int it, int& h, int& q0) {
    h = kh * G + it / nqb;
    q0 = k0 + (it % nqb) * QB;
  };
  auto load_tile = [&](int it) {  // Q, dO [, dOl] rows of tile it -> stage it & 1 (cp.async)
    int h, q0;
    tile_rows(it, h, q0);
    const int qv = min(QB, L - q0);
    uint8_t* sb = stage_base(it & 1);
    __nv_bfloat16* Qd = reinterpret_cast<__nv_bfloat16*>(sb);
    __nv_bfloat16* Dd = reinterpret_cast<__nv_bfloat16*>(sb + S::qt);
#pragma unroll
    for (int i = 0; i < QB * C8 / (kWarps * 32); ++i) {
      const int e = threadIdx.x + i * kWarps * 32, r = e / C8, c = (e % C8) * 8;
      const bool ok = r < qv;
      const size_t row = ((size_t)(s0 + q0 + (ok ? r : 0)) * nq + h) * HD + c;
      cp16_zfill(Qd + r * P + c, q + row, ok);
      cp16_zfill(Dd + r * P + c, dob + row, ok);
      if constexpr (SPLIT) cp16_zfill(reinterpret_cast<__nv_bfloat16*>(sb + 2 * S::qt) + r * P + c, dol + row, ok);
    }
  };
  auto load_stats = [&](int it, float& pl, float& pd) {  // lse, D of row threadIdx.x of tile it
    int h, q0;
    tile_rows(it, h, q0);
    const int r = threadIdx.x, qv = min(QB, L - q0);
    pl = r < qv ? lse[(size_t)(s0 + q0 + r) * nq + h] : 0.f;
    pd = r < qv ? D[(size_t)(s0 + q0 + r) * nq + h] : 0.f;
  };
  auto put_stats = [&](int it, float pl, float pd) {
    float* st = reinterpret_cast<float*>(stage_base(it & 1) + (SPLIT ? 3 : 2) * S::qt);
    if (threadIdx.x < QB) {
      st[threadIdx.x] = pl;
      st[QB + threadIdx.x] = pd;
    }
  };
  static_assert(kWarps * 32 >= QB, "one lse / D row per thread");
  load_tile(0);
  asm volatile("cp.async.commit_group;" ::: "memory");
  {
    float pl, pd;
    load_stats(0, pl, pd);
    put_stats(0, pl, pd);
  }

  float dk[NT][4], dv[NT][4];
#pragma unroll
  for (int n = 0; n < NT; ++n)
#pragma unroll
    for (int i = 0; i < 4; ++i) dk[n][i] = dv[n][i] = 0.f;
  const int kr = warp * 16;  // this warp's 16 keys (block-local)
  const int key_lo = k0 + kr + (lane >> 2), key_hi = key_lo + 8;

  for (int it = 0; it < n_it; ++it) {
    float npl = 0.f, npd = 0.f;
    if (it + 1 < n_it) {
      load_tile(it + 1);
      asm volatile("cp.async.commit_group;" ::: "memory");
      load_stats(it + 1, npl, npd);  // registers: latency under this tile
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    int h, q0;
    tile_rows(it, h, q0);
    (void)h;
    const int qvalid = min(QB, L - q0);
    const uint8_t* sb = stage_base(it & 1);
    const __nv_bfloat16* Qs = reinterpret_cast<const __nv_bfloat16*>(sb);
    const __nv_bfloat16* dOs = reinterpret_cast<const __nv_bfloat16*>(sb + S::qt);
    const __nv_bfloat16* dOl = reinterpret_cast<const __nv_bfloat16*>(sb + 2 * S::qt);
    const float* s_lse = reinterpret_cast<const float*>(sb + (SPLIT ? 3 : 2) * S::qt);
    const float* s_D = s_lse + QB;
    // S^T = K_w Q^T and dP^T = V_w dO^T: [16 keys x QB queries]
    float st[QN][4], dpt[QN][4];
#pragma unroll
    for (int n = 0; n < QN; ++n)
#pragma unroll
      for (int i = 0; i < 4; ++i) st[n][i] = dpt[n][i] = 0.f;
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk) {
      uint32_t ak[4], av[4];
      ldsm_x4(ak, Ks + (kr + (lane & 15)) * P + kk * 16 + (lane >> 4) * 8);
      ldsm_x4(av, Vs + (kr + (lane & 15)) * P + kk * 16 + (lane >> 4) * 8);
#pragma unroll
      for (int n = 0; n < QN; n += 2) {  // two 8-query column blocks per ldmatrix.x4
        const int roff = (n * 8 + (lane & 7) + ((lane >> 4) << 3)) * P + kk * 16 + ((lane >> 3) & 1) * 8;
        uint32_t b[4];
        ldsm_x4(b, Qs + roff);
        mma16816(st[n], ak, b[0], b[1]);
        mma16816(st[n + 1], ak, b[2], b[3]);
        ldsm_x4(b, dOs + roff);
        mma16816(dpt[n], av, b[0], b[1]);
        mma16816(dpt[n + 1], av, b[2], b[3]);
        if constexpr (SPLIT) {
          ldsm_x4(b, dOl + roff);
          mma16816(dpt[n], av, b[0], b[1]);
          mma16816(dpt[n + 1], av, b[2], b[3]);
        }
      }
    }
    // P^T and dS^T (scaled), causal: query position >= key position
#pragma unroll
    for (int n = 0; n < QN; ++n) {
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
    // dV += P^T dO, dK += dS^T Q   (k = QB queries in steps of 16)
#pragma unroll
    for (int ks = 0; ks < QB / 16; ++ks) {
      uint32_t ap[4], apl[4], ad[4], adl[4];
      c_to_a<SPLIT>(st[2 * ks], st[2 * ks + 1], ap, apl);
      c_to_a<SPLIT>(dpt[2 * ks], dpt[2 * ks + 1], ad, adl);
#pragma unroll
      for (int n = 0; n < NT; n += 2) {  // two 8-dim blocks per ldmatrix.x4.trans
        const int roff = (ks * 16 + (lane & 7) + ((lane >> 3) & 1) * 8) * P + n * 8 + (lane >> 4) * 8;
        uint32_t b[4];
        ldsm_x4_trans(b, dOs + roff);
        mma16816(dv[n], ap, b[0], b[1]);
        mma16816(dv[n + 1], ap, b[2], b[3]);
        if constexpr (SPLIT) {
          mma16816(dv[n], apl, b[0], b[1]);
          mma16816(dv[n + 1], apl, b[2], b[3]);
          ldsm_x4_trans(b, dOl + roff);
          mma16816(dv[n], ap, b[0], b[1]);
          mma16816(dv[n + 1], ap, b[2], b[3]);
        }
        ldsm_x4_trans(b, Qs + roff);
        mma16816(dk[n], ad, b[0], b[1]);
        mma16816(dk[n + 1], ad, b[2], b[3]);
        if constexpr (SPLIT) {
          mma16816(dk[n], adl, b[0], b[1]);
          mma16816(dk[n + 1], adl, b[2], b[3]);
        }
      }
    }
    if (it + 1 < n_it) put_stats(it + 1, npl, npd);  // its slot's previous tile (it - 1) is done
    __syncthreads();  // stage it & 1 is refilled with tile it + 2 next iteration
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
    attn_bwd_dq_mma(const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ dob,
                    const __nv_bfloat16* __restrict__ dol, const float* __restrict__ lse,
                    const float* __restrict__ D, const __nv_bfloat16* __restrict__ kc,
                    const __nv_bfloat16* __restrict__ vc, const int32_t* __restrict__ seq_start,
                    const int32_t* __restrict__ seq_len, const int32_t* __restrict__ bt, int pps, int nq,
                    int nkv, float scale, float* __restrict__ dqkv) {
  using S = DqSmem<HD, SPLIT>;
  constexpr int P = S::P, NT = HD / 8, C8 = HD / 8;
  constexpr int TE = kBlk * P;
  extern __shared__ __align__(16) uint8_t smem[];
  __nv_bfloat16* const sb = reinterpret_cast<__nv_bfloat16*>(smem);
  __nv_bfloat16* const dOs = sb;
  __nv_bfloat16* const dOl = sb + TE;                        // (SPLIT)
  __nv_bfloat16* const kv0 = sb + (SPLIT ? 2 : 1) * TE;      // K0 V0 K1 V1
  const int slot = blockIdx.y, h = blockIdx.z;
  const int L = seq_len[slot], s0 = seq_start[slot];
  const int q0 = blockIdx.x * kBlk;
  if (q0 >= L) return;
  const int kh = h / (nq / nkv);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qvalid = min(kBlk, L - q0);
  auto load_block = [&](int j) {  // key page j -> K / V buffers (j & 1)
    const int valid = min(kBlk, L - j * kBlk);
    const size_t page = (size_t)bt[(size_t)slot * pps + j];
    const __nv_bfloat16* kg = kc + (page * nkv + kh) * kPageTokens * HD;
    const __nv_bfloat16* vg = vc + (page * nkv + kh) * kPageTokens * HD;
    __nv_bfloat16* kd = kv0 + (size_t)(2 * (j & 1)) * TE;
    __nv_bfloat16* vd = kd + TE;
#pragma unroll
    for (int it = 0; it < kBlk * C8 / (kWarps * 32); ++it) {
      const int e = threadIdx.x + it * kWarps * 32, r = e / C8, c = (e % C8) * 8;
      const bool ok = r < valid;
      cp16_zfill(kd + r * P + c, ok ? kg + r * HD + c : kg, ok);
      cp16_zfill(vd + r * P + c, ok ? vg + r * HD + c : vg, ok);
    }
  };
  {  // Q -> the K1 buffer (fragments to registers below), dO [, dOl], with page 0
    __nv_bfloat16* qd = kv0 + 2 * TE;
#pragma unroll
    for (int it = 0; it < kBlk * C8 / (kWarps * 32); ++it) {
      const int e = threadIdx.x + it * kWarps * 32, r = e / C8, c = (e % C8) * 8;
      const bool ok = r < qvalid;
      const size_t row = ((size_t)(s0 + q0 + (ok ? r : 0)) * nq + h) * HD + c;
      cp16_zfill(qd + r * P + c, q + row, ok);
      cp16_zfill(dOs + r * P + c, dob + row, ok);
      if constexpr (SPLIT) cp16_zfill(dOl + r * P + c, dol + row, ok);
    }
  }
  load_block(0);
  asm volatile("cp.async.commit_group;" ::: "memory");
  const int qr = warp * 16;
  const int ql_lo = qr + (lane >> 2), ql_hi = ql_lo + 8;
  const float lse_lo = ql_lo < qvalid ? lse[(size_t)(s0 + q0 + ql_lo) * nq + h] : 0.f;
  const float lse_hi = ql_hi < qvalid ? lse[(size_t)(s0 + q0 + ql_hi) * nq + h] : 0.f;
  const float D_lo = ql_lo < qvalid ? D[(size_t)(s0 + q0 + ql_lo) * nq + h] : 0.f;
  const float D_hi = ql_hi < qvalid ? D[(size_t)(s0 + q0 + ql_hi) * nq + h] : 0.f;
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  uint32_t qf[HD / 16][4];
#pragma unroll
  for (int kk = 0; kk < HD / 16; ++kk)
    ldsm_x4(qf[kk], kv0 + 2 * TE + (qr + (lane & 15)) * P + kk * 16 + (lane >> 4) * 8);
  __syncthreads();  // the Q staging (buffer 1) is refilled below

  float dq[NT][4];
#pragma unroll
  for (int n = 0; n < NT; ++n)
#pragma unroll
    for (int i = 0; i < 4; ++i) dq[n][i] = 0.f;
  const int nblk = (q0 + qvalid - 1) / kBlk + 1;  // causal: keys up to the block's last query
  for (int j = 0; j < nblk; ++j) {
    if (j + 1 < nblk) {
      load_block(j + 1);
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const __nv_bfloat16* Ks = kv0 + (size_t)(2 * (j & 1)) * TE;
    const __nv_bfloat16* Vs = Ks + TE;
    const int k0 = j * kBlk;
    const int kvalid = min(kBlk, L - k0);
    float s[8][4], dp[8][4];
#pragma unroll
    for (int n = 0; n < 8; ++n)
#pragma unroll
      for (int i = 0; i < 4; ++i) s[n][i] = dp[n][i] = 0.f;
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk) {
      uint32_t ad[4], adl[4];
      ldsm_x4(ad, dOs + (qr + (lane & 15)) * P + kk * 16 + (lane >> 4) * 8);
      if constexpr (SPLIT) ldsm_x4(adl, dOl + (qr + (lane & 15)) * P + kk * 16 + (lane >> 4) * 8);
#pragma unroll
      for (int n = 0; n < 8; n += 2) {
        const int roff = (n * 8 + (lane & 7) + ((lane >> 4) << 3)) * P + kk * 16 + ((lane >> 3) & 1) * 8;
        uint32_t b[4];
        ldsm_x4(b, Ks + roff);
        mma16816(s[n], qf[kk], b[0], b[1]);
        mma16816(s[n + 1], qf[kk], b[2], b[3]);
        ldsm_x4(b, Vs + roff);
        mma16816(dp[n], ad, b[0], b[1]);
        mma16816(dp[n + 1], ad, b[2], b[3]);
        if constexpr (SPLIT) {
          mma16816(dp[n], adl, b[0], b[1]);
          mma16816(dp[n + 1], adl, b[2], b[3]);
        }
      }
    }
    const bool masked = k0 + kBlk - 1 > q0 || kvalid < kBlk;  // the diagonal page, or past L
#pragma unroll
    for (int n = 0; n < 8; ++n) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int kl = n * 8 + (lane & 3) * 2 + (i & 1);
        const int ql = i < 2 ? ql_lo : ql_hi;
        const bool ok = ql < qvalid && (!masked || (kl < kvalid && k0 + kl <= q0 + ql));
        const float p = ok ? __expf(s[n][i] * scale - (i < 2 ? lse_lo : lse_hi)) : 0.f;
        dp[n][i] = p * (dp[n][i] - (i < 2 ? D_lo : D_hi)) * scale;
      }
    }
    // dQ += dS K  (k = 64 keys in 4 steps of 16; K[key][d] read transposed)
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      uint32_t a[4], al[4];
      c_to_a<SPLIT>(dp[2 * ks], dp[2 * ks + 1], a, al);
#pragma unroll
      for (int n = 0; n < NT; n += 2) {
        uint32_t b[4];
        ldsm_x4_trans(b, Ks + (ks * 16 + (lane & 7) + ((lane >> 3) & 1) * 8) * P + n * 8 + (lane >> 4) * 8);
        mma16816(dq[n], a, b[0], b[1]);
        mma16816(dq[n + 1], a, b[2], b[3]);
        if constexpr (SPLIT) {
          mma16816(dq[n], al, b[0], b[1]);
          mma16816(dq[n + 1], al, b[2], b[3]);
        }
      }
    }
    __syncthreads();  // buffer (j & 1) is refilled with page j + 2 next iteration
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
cudaError_t launch_t(const __nv_bfloat16* q, const __nv_bfloat16* dob, const __nv_bfloat16* dol, const float* lse,
                     const float* D, const __nv_bfloat16* kc, const __nv_bfloat16* vc, const int32_t* seq_start,
                     const int32_t* seq_len, const int32_t* bt, int pps, int n_seq, int nq, int nkv,
                     float scale, float* dqkv, cudaStream_t st) {
  constexpr size_t sk = DkvSmem<HD, SPLIT>::total, sq = DqSmem<HD, SPLIT>::total;
  static const bool attr =
      cudaFuncSetAttribute(attn_bwd_dkv_mma<HD, SPLIT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sk) ==
          cudaSuccess &&
      cudaFuncSetAttribute(attn_bwd_dq_mma<HD, SPLIT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sq) ==
          cudaSuccess;
  if (!attr) return cudaErrorInvalidValue;
  // pages per sequence = 64-token blocks per sequence
  attn_bwd_dkv_mma<HD, SPLIT><<<dim3(pps, n_seq, nkv), kWarps * 32, sk, st>>>(
      q, dob, dol, lse, D, kc, vc, seq_start, seq_len, bt, pps, nq, nkv, scale, dqkv);
  attn_bwd_dq_mma<HD, SPLIT><<<dim3(pps, n_seq, nq), kWarps * 32, sq, st>>>(
      q, dob, dol, lse, D, kc, vc, seq_start, seq_len, bt, pps, nq, nkv, scale, dqkv);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_attention_bwd_mma(const __nv_bfloat16* q, const __nv_bfloat16* dob, const __nv_bfloat16* dol,
                                     const float* lse, const float* D, const __nv_bfloat16* kc,
                                     const __nv_bfloat16* vc, const int32_t* seq_start, const int32_t* seq_len,
                                     const int32_t* block_table, int pages_per_seq, int n_seq, int nq,
                                     int nkv, int hd, float* dqkv, cudaStream_t st, bool split) {
  const float scale = 1.0f / sqrtf((float)hd);
  if (split && dol == nullptr) return cudaErrorInvalidValue;
#define SRL_BWD_ARGS q, dob, dol, lse, D, kc, vc, seq_start, seq_len, block_table, pages_per_seq, n_seq, nq, nkv, scale, dqkv, st
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
