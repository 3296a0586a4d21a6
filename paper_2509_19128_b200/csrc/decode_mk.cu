// decode_mk.cu -- persistent decode-round megakernel (see decode_mk.cuh).
//
// One CTA per SM, 12 warps: warp 0 TMA producer, warp 1 tcgen05.mma issuer,
// warps 4-11 compute (256 threads, named barrier 1).  Warps 2-3 only hold the
// TMEM quadrant mapping in place (a warp may only tcgen05.ld the 32 TMEM lanes
// of quadrant warp_id % 4: compute warps w and w + 4 share a quadrant and
// drain the two 32-token halves of the 64-column accumulator).
#include <cmath>
#include <cstdio>

#include "decode_mk.cuh"
#include "fastexp.cuh"
#include "gemm_epi.cuh"
#include "sm100.cuh"

namespace srl {
using namespace sm100;

namespace {

constexpr int kTok = 64;   // rows (UMMA N): decode batch <= 64
constexpr int kBN = 128;   // weight rows per tile (UMMA M)
constexpr int kBK = 64;    // k-block (128-B swizzle row)
constexpr int kThreads = 384;
constexpr int kCW = 8;     // compute warps (4..11)
constexpr int kCT = 32 * kCW;
constexpr int kABytes = kBN * kBK * 2;
constexpr int kBBytes = kTok * kBK * 2;
constexpr int kStageBytes = kABytes + kBBytes;
constexpr int kPitch = kBN + 4;
constexpr int kTileFloats = kTok * kBN;
constexpr int kLmTile = 128;
constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ULL;
constexpr int kMaxSplitPages = 128;  // attention split <= 8192 keys
constexpr int kMaxCs = 16;          // split-K factor cap (reduce staging)
#ifndef SRL_MK_KT128
#define SRL_MK_KT128 16
#endif
#ifndef SRL_MK_STAGES128
#define SRL_MK_STAGES128 5
#endif

__device__ __forceinline__ void csync() { asm volatile("bar.sync 1, 256;" ::: "memory"); }
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int ld_acquire_cta(const int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared.b32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_cta(int* p, int v) {
  asm volatile("st.release.cta.shared.b32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Bounded spins: a broken schedule traps after ~4 s (the launch fails loudly)
// instead of hanging the device.
struct SpinGuard {
  unsigned n = 0;
  unsigned long long t0 = 0;
  __device__ __forceinline__ void tick() {
    if ((++n & 255u) == 0) {
      const unsigned long long t = globaltimer();
      if (t0 == 0) t0 = t;
      else if (t - t0 > 4000000000ull) __trap();
    }
  }
};
// Acquire-load polling (measured faster than relaxed polling + one fence).
__device__ __forceinline__ void wait_count(const unsigned* p, unsigned target) {
  SpinGuard g;
  while ((int)(ld_acquire(p) - target) < 0) {
    __nanosleep(32);
    g.tick();
  }
}
// Phase barrier: kBarLanes sub-counters per phase (CTA c arrives on c %
// kBarLanes), a waiter sums them.  One lane measured fastest (several acquire
// loads per poll cost more than the arrival serialisation they avoid).
#ifndef SRL_BAR_LANES
#define SRL_BAR_LANES 1
#endif
constexpr int kBarLanes = SRL_BAR_LANES;
// Arrival = one release reduction (no return value to wait for; .release
// orders this CTA's prior writes -- made CTA-visible by the preceding bar.sync
// -- before the count, like __threadfence + atomicAdd, without the round trip).
__device__ __forceinline__ void phase_arrive(unsigned* pd, int p, int c) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(&pd[p * kBarLanes + (c % kBarLanes)]), "r"(1u)
               : "memory");
}
__device__ __forceinline__ void phase_wait(const unsigned* pd, int p, unsigned target) {
  SpinGuard g;
  const unsigned* b = pd + p * kBarLanes;
  while (true) {
    unsigned v[kBarLanes];
#pragma unroll
    for (int k = 0; k < kBarLanes; ++k) v[k] = ld_acquire(b + k);
    unsigned s = 0;
#pragma unroll
    for (int k = 0; k < kBarLanes; ++k) s += v[k];
    if ((int)(s - target) >= 0) return;
    __nanosleep(32);
    g.tick();
  }
}
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, 20000;\n\t"
      "selp.u32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mk_wait(uint64_t* bar, uint32_t parity) {
  SpinGuard g;
  while (!mbar_try(bar, parity)) g.tick();
}
// first item of CTA c in a phase whose items are dealt round-robin from `rot`
__device__ __forceinline__ int first_item(int c, int rot, int G) { return c >= rot ? c - rot : c - rot + G; }

// DSMEM (cluster of two CTAs): address of the same shared location in the
// partner CTA, remote store, remote release-arrive, cluster-scope acquire wait.
__device__ __forceinline__ uint32_t partner_addr(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
// mma.sync m16n8k16 (bf16 -> fp32) for the attention items: fragments of a
// row-major bf16 tile X[row][col] (pitch in elements) and of B from Y[n][k].
__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t ld_b32(const __nv_bfloat16* p) { return *reinterpret_cast<const uint32_t*>(p); }
__device__ __forceinline__ uint32_t pack2_bf16(float lo, float hi) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&v);
}
// (x, y) -> bf16x2 hi = RN(x, y) and lo = RN(x - hi, y - hi): hi + lo carries
// ~16 significant bits.
__device__ __forceinline__ void split_bf16(float x, float y, uint32_t& hi, uint32_t& lo) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(x, y);
  const float2 hf = __bfloat1622float2(h);
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = pack2_bf16(x - hf.x, y - hf.y);
}
// B fragment (k = 16 rows of a row-major [k][n] tile, n = 8 columns at col0)
// through ldmatrix.trans: lanes 0-15 address rows k0 .. k0 + 15.
__device__ __forceinline__ void ldsm_x2_trans(uint32_t& b0, uint32_t& b1, const uint8_t* tile, int pitch_bytes,
                                              int k0, int col0, int lane) {
  const uint8_t* p = tile + (size_t)(k0 + (lane & 15)) * pitch_bytes + col0 * 2;
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0, %1}, [%2];"
               : "=r"(b0), "=r"(b1)
               : "r"(smem_u32(p)));
}

__device__ __forceinline__ void fence_proxy_async_shared() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
// Bulk (non-tensor) async copy global -> shared, completion on an mbarrier.
__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

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
__device__ __forceinline__ double uniform_draw(uint64_t seed, uint64_t n) {
  uint64_t z = seed + (n + 1) * kGolden;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  z ^= z >> 31;
  return (double)(z >> 11) * 0x1.0p-53;
}


// Attention item scratch: q, per-warp K/V tiles (cp.async), probabilities,
// per-warp softmax state, the row's reduced q|k|v; the QKV split partials are
// staged in the tile area first and the warp accumulators alias it last.
template <int HD, int G>
struct AttnSmem {
  // keys per warp tile.  hd 128: 16-key tiles beside a 5-stage weight ring; 32-key
  // tiles need a 3-stage ring (SRL_MK_KT128=32 SRL_MK_STAGES128=3) -- measured at
  // 1.5B / 8k contexts: attention unchanged (4.05 vs 3.99 ms per round), the GEMM
  // phases 0.1 ms slower
  static constexpr int KT = HD == 64 ? 32 : SRL_MK_KT128;
  static constexpr int ROW = HD * 2 + 16;        // padded K row (conflict-free fragment loads)
  static constexpr int VROW = HD * 2 + 16;       // padded V row (conflict-free ldmatrix.trans)
  static constexpr int QP = HD + 8;              // bf16 q tile [16 (heads, zero-padded)][QP]
  static constexpr size_t sq = sizeof(__nv_bfloat16) * 16 * QP > sizeof(float) * G * HD
                                   ? sizeof(__nv_bfloat16) * 16 * QP : sizeof(float) * G * HD;
  static constexpr size_t kbuf = (size_t)KT * ROW, vbuf = (size_t)KT * VROW;
  static constexpr size_t warp_bytes = kbuf + vbuf;
  static constexpr size_t tiles = kCW * warp_bytes;
  static constexpr size_t sp = 0;  // (probabilities stay in registers: mma.sync P.V)
  static constexpr size_t sml = sizeof(float) * 2 * kCW * G;
  static constexpr size_t spage = sizeof(int) * kMaxSplitPages;
  static constexpr size_t sraw = sizeof(float) * (G + 2) * HD;  // reduced q | k | v of the row
  static constexpr size_t snew = sizeof(__nv_bfloat16) * 2 * HD;  // the new token's k, v
  static constexpr size_t total = sq + tiles + sp + sml + spage + sraw + snew;
  static_assert(sizeof(float) * kCW * G * HD <= tiles, "accumulators alias the tiles");
};

template <int HD, int G>
struct MkLayout {
  static constexpr int STAGES = HD == 64 ? 6 : SRL_MK_STAGES128;
  static constexpr size_t ring = (size_t)STAGES * kStageBytes;
  static constexpr size_t epi = sizeof(float) * kTok * kPitch;
  static constexpr size_t stage_red = (size_t)(kTok + kMaxCs) * kBN * 4;  // split-K row slices
  static constexpr size_t att = AttnSmem<HD, G>::total;
  static constexpr size_t smp = sizeof(double) * (kCT + 40) + 256;
  static constexpr size_t gemm_scr = epi + stage_red;
  static constexpr size_t scratch =
      gemm_scr > att ? (gemm_scr > smp ? gemm_scr : smp) : (att > smp ? att : smp);
  static constexpr size_t bar = ring + scratch;
  static constexpr size_t misc = bar + (2 * STAGES + 6) * 8;
  static constexpr size_t rstd = misc + 32;
  static constexpr size_t rows = rstd + kTok * 4;  // round-constant (slot, pos) of every row
  static constexpr size_t anx = rows + kTok * 8;     // attention lookahead mailbox (MkAnx, 64 B)
  // the next attention item's QKV partials, bulk-copied by the lookahead warp
  // while the current item finishes (hd 128; hd 64 has no room beside its
  // 6-stage ring: its items stage the partials in the K/V buffers)
  static constexpr size_t qpre = (anx + 64 + 127) & ~size_t(127);
  static constexpr size_t qpre_want = HD == 128 ? 24576 : 0;
  static constexpr size_t qpre_bytes = qpre + qpre_want + 1024 <= 232448 ? qpre_want : 0;  // (if it fits)
  static constexpr size_t total = qpre + qpre_bytes;
  static constexpr size_t alloc = total + 1024;
  static_assert(alloc <= 232448, "shared memory budget");
  static_assert(scratch >= 8192 + (2 * (size_t)kMkMaxAttnItems + 2) * 4, "mk_attn_order scratch");
};

// ----------------------------------------------------------- compute ---
// Deferred RMSNorm: rstd of every row for the GEMMs that consume xg.
__device__ void mk_rows(const MkParams& P, int kind, float* s_rstd, int ct) {
  for (int j = ct; j < kTok; j += kCT) {
    float r = 1.f;
    if ((kind == MK_GU || kind == MK_LM) && j < P.S) {
      float s = 0.f;
      s = gemm_detail::ssq_row_sum(P.ssq + (size_t)j * P.parts, P.parts);
      r = rsqrtf(s * P.inv_h + P.eps);
    }
    s_rstd[j] = r;
  }
}

// LM-head tile statistics: max and fp64 sum of exp(x - max) per row over the
// tile's 128 columns (the sampler's per-tile partition sums).  Four threads
// per row, 32 independent exponentials each; the four partial sums combine
// by a symmetric butterfly, so every lane holds the same, order-fixed value.
__device__ __noinline__ void mk_lm_stats(const MkParams& P, const float* tile, int n_tile, int N,
                                         int ct, int r0, int r1) {
  const int T = (N + kLmTile - 1) / kLmTile;
  const int j = r0 + (ct >> 2), part = ct & 3;
  const bool valid = j < r1;  // converged shuffles: invalid quads recompute row r0
  const float* row = &tile[(valid ? j : r0) * kPitch + part * 32];
  float mx = -INFINITY;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const float4 v = *reinterpret_cast<const float4*>(row + 4 * q);
    mx = fmaxf(mx, fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)));
  }
  mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
  mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
  double a[4] = {0.0, 0.0, 0.0, 0.0};
  if (mx != -INFINITY) {
    const double md = (double)mx;
#pragma unroll 2
    for (int q = 0; q < 8; ++q) {
      const float4 v = *reinterpret_cast<const float4*>(row + 4 * q);
      a[0] += exp_nonpos((double)v.x - md);
      a[1] += exp_nonpos((double)v.y - md);
      a[2] += exp_nonpos((double)v.z - md);
      a[3] += exp_nonpos((double)v.w - md);
    }
  }
  double sm = (a[0] + a[1]) + (a[2] + a[3]);
  sm += __shfl_xor_sync(0xffffffffu, sm, 1);
  sm += __shfl_xor_sync(0xffffffffu, sm, 2);
  if (part == 0 && valid) {
    P.lse_max[(size_t)j * T + n_tile] = mx;
    P.lse_sum[(size_t)j * T + n_tile] = sm;
  }
}

// Fused epilogues on the reduced [64 x 128] tile (rows = tokens, cols = n0..).
// Rows [r0, r1) of the tile belong to this CTA (split-K row slices).
// colv: this thread's column constant (next RMSNorm gain), loaded before the
// accumulator wait.  QKV has no epilogue here: its split partials are
// reduced by the attention items that consume them.
__device__ __forceinline__ void mk_epilogue(const MkParams& P, const MkPhase& ph, int n_tile,
                                            float* tile, const float* s_rstd, int ct, int r0,
                                            int r1, float colv, const float* xs) {
  const int n0 = n_tile * kBN, N = ph.N, M = r1;
  const int nr = r1 - r0;
  const int cw = ct >> 5, lane = ct & 31;
  if (ph.kind == MK_O || ph.kind == MK_DOWN) {
    // residual add; column c = ct & 127, the two thread halves take
    // alternating rows, 8 residual loads in flight per chunk
    const int c = ct & (kBN - 1), hf = ct >> 7, n = n0 + c;
    for (int j0 = r0 + hf; j0 < r1; j0 += 16) {
      float xr[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int j = j0 + 2 * u;
        xr[u] = (j < r1 && n < N) ? (xs ? xs[(j - r0) * kBN + c] : P.x[(size_t)j * N + n]) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int j = j0 + 2 * u;
        if (j >= r1) break;
        float x = 0.f;
        if (n < N) {
          const size_t o = (size_t)j * N + n;
          x = xr[u] + tile[j * kPitch + c];
          P.x[o] = x;
          P.xg[o] = __float2bfloat16(x * colv);
        }
        tile[j * kPitch + c] = x;
      }
    }
    csync();
    for (int j = r0 + cw; j < M; j += kCW) {
      float s = 0.f;
      for (int c2 = lane; c2 < kBN; c2 += 32) {
        const float xv = tile[j * kPitch + c2];
        s += xv * xv;
      }
      s = wsum(s);
      if (lane == 0) P.ssq[(size_t)j * P.parts + n_tile] = s;
    }
  } else if (ph.kind == MK_GU) {
#pragma unroll 2
    for (int idx = ct; idx < nr * (kBN / 4); idx += kCT) {  // two columns per thread
      const int j = r0 + (idx >> 5), c = (idx & 31) * 2;
      const float r = s_rstd[j];
      const float2 g2 = *reinterpret_cast<const float2*>(&tile[j * kPitch + c]);
      const float2 u2 = *reinterpret_cast<const float2*>(&tile[j * kPitch + 64 + c]);
      const float g0 = g2.x * r, g1 = g2.y * r, u0 = u2.x * r, u1 = u2.y * r;
      *reinterpret_cast<__nv_bfloat162*>(&P.act[(size_t)j * P.I + (n0 >> 1) + c]) =
          __floats2bfloat162_rn(__fdividef(g0, 1.f + __expf(-g0)) * u0,
                                __fdividef(g1, 1.f + __expf(-g1)) * u1);
    }
  } else if (ph.kind == MK_LM) {
    // scale by rstd and store the logits (one float4 per thread per row), keep
    // the scaled tile for the statistics
    const int c4 = lane * 4, n = n0 + c4;
    for (int j = r0 + cw; j < r1; j += kCW) {
      float4 v = *reinterpret_cast<const float4*>(&tile[j * kPitch + c4]);
      const float r = s_rstd[j];
      v.x = n + 0 < N ? v.x * r : -INFINITY;
      v.y = n + 1 < N ? v.y * r : -INFINITY;
      v.z = n + 2 < N ? v.z * r : -INFINITY;
      v.w = n + 3 < N ? v.w * r : -INFINITY;
      float* dst = P.logits + (size_t)j * N + n;
      if (n + 3 < N && (N & 3) == 0) {
        *reinterpret_cast<float4*>(dst) = v;
      } else {
        if (n + 0 < N) dst[0] = v.x;
        if (n + 1 < N) dst[1] = v.y;
        if (n + 2 < N) dst[2] = v.z;
        if (n + 3 < N) dst[3] = v.w;
      }
      *reinterpret_cast<float4*>(&tile[j * kPitch + c4]) = v;
    }
    csync();
    mk_lm_stats(P, tile, n_tile, N, ct, r0, r1);
  }
}

// Causal paged GQA attention for (row m, kv head kh, key split) on the 8
// compute warps, with the QKV GEMM's epilogue fused in front:
//  1. the row's q|k|v columns of every QKV split partial arrive by bulk copy;
//     their sum (split order) x rstd + bias, RoPE on q and k, bf16 rounding;
//     the new token's k/v go to the paged cache (and to the tile that holds
//     its position, so no global round trip is waited on);
//  2. keys [k0, k1) in KT-key tiles dealt round-robin to the warps (cp.async),
//     online softmax (lane = key for scores, lane = dims for P.V);
//  3. warps merged in shared memory; several splits (long contexts) merged by
//     the last-arriving split in split order (deterministic).
// Work queue of an attention phase: the next item (attn_order index) or -1
// once the queue is drained.  next_item: ct 0 only.
struct MkQueue {
  unsigned* ctr;
  unsigned base;
  int n_items;
  const int32_t* order;
  __device__ __forceinline__ unsigned grab() const { return atomicAdd(ctr, 1u) - base; }
  __device__ __forceinline__ int resolve(unsigned iq) const {
    return iq < (unsigned)n_items ? __ldcg(order + iq) : -1;
  }
};
// Every CTA makes exactly one failing grab per attention phase, so a launch
// adds n_items + grid to the phase's counter: (epoch x that) is its base.
__device__ __forceinline__ MkQueue mk_queue(const MkParams& P, const MkPhase& F, unsigned ep1, int grid) {
  return MkQueue{P.tile_ctr + F.ctr_base + P.S * P.nkv, (ep1 - 1u) * (unsigned)(F.n_items + grid), F.n_items,
                 P.attn_order};
}

// Attention lookahead mailbox (shared memory) between the compute warps and
// the otherwise idle warp 3: when compute warp 0 starts its last key tile of
// an item it posts a request; warp 3 takes the next queue item, resolves it,
// loads the block-table pages of its first kCW x KT keys and the new key's
// page, and (hd 128) bulk-copies its QKV partials into the qpre buffer on
// cbar -- so the next item starts with its first K/V tiles issued at once and
// its q operand one reduction away, instead of ~4 us of dependent round trips.
struct MkAnx {
  int req, done;    // request sequence (compute warp 0) / completed request (warp 3)
  int item, bulk;   // resolved item (attn_order value, -1: queue drained); on cbar: 1 the QKV
                    // partials, 2 also the extras (bias slice, cos / sin row, x^2 partials)
  int cpage, phase; // the new key's page; the request's phase (-1: exit)
  int pad[2];
  int pages[8];     // pages of the item's first kCW x KT keys
};
static_assert(sizeof(MkAnx) == 64, "mailbox");

// Returns true when the lookahead warp has taken the next queue item (in
// *s_next); false on the early exits (the caller grabs).  pre: this item
// was resolved by the lookahead warp (pages in the mailbox; partials already
// in flight on cbar when anx->bulk).
template <int HD, int G>
__device__ bool mk_attention(const MkParams& P, int layer, long long bias_off, int qkv_cs, int m, int kh, int split,
                             uint8_t* scr, const int2* s_rows, unsigned* ctr, unsigned ep1,
                             float* ws, int ct, int* s_flag, uint64_t* cbar, uint32_t& cph,
                             unsigned long long* tr, MkAnx* anx, bool pre, float* qpre, int p, int& seq,
                             int* s_next, bool lookahead) {
  using A = AttnSmem<HD, G>;
  const long long c_start = clock64();
  constexpr int KT = A::KT, V4 = HD / 8, PER = KT * V4 / 32;
  constexpr int W = (G + 2) * HD;            // q heads | k | v of this kv head
  constexpr int WPT = (W + kCT - 1) / kCT;   // of them per thread
  uint8_t* tiles = scr + A::sq;
  float(*sp)[G][32] = reinterpret_cast<float(*)[G][32]>(scr + A::sq + A::tiles);
  float(*sm_m)[G] = reinterpret_cast<float(*)[G]>(scr + A::sq + A::tiles + A::sp);
  float(*sm_l)[G] = reinterpret_cast<float(*)[G]>(scr + A::sq + A::tiles + A::sp + sizeof(float) * kCW * G);
  float* sraw = reinterpret_cast<float*>(scr + A::sq + A::tiles + A::sp + A::sml + A::spage);
  __nv_bfloat16* snew = reinterpret_cast<__nv_bfloat16*>(scr + A::sq + A::tiles + A::sp + A::sml +
                                                         A::spage + A::sraw);
  float(*sm_acc)[G][HD] = reinterpret_cast<float(*)[G][HD]>(tiles);  // after the tiles are consumed
  __nv_bfloat16* sqb = reinterpret_cast<__nv_bfloat16*>(scr);          // [16][QP] bf16 q (rows >= G zero)
  const int warp = ct >> 5, lane = ct & 31;
  const int splits = P.attn_splits, nq = P.nq, nkv = P.nkv;
  const int slot = s_rows[m].x;
  if (slot < 0) {  // a free slot: split 0 arrives for all of its splits (monotonic counters)
    if (splits > 1 && split == 0 && ct == 0) atomicAdd(&ctr[m * nkv + kh], (unsigned)splits);
    return false;
  }
  const int pos = s_rows[m].y;  // position of the new token; ctx = pos + 1 keys
  const int ctx = pos + 1;
  const int k0 = split * P.attn_chunk;
  const int k1 = min(ctx, k0 + P.attn_chunk);
  const int nkeys = max(0, k1 - k0);
  const int ntiles = (nkeys + KT - 1) / KT;
  const bool owner = pos >= k0 && pos < k0 + P.attn_chunk;  // this split holds the new key
  const int qend = nq * HD, kend = qend + nkv * HD;
  constexpr size_t rec = (size_t)G * (HD + 2);
  // Split merge (deterministic, split order): the last split to arrive
  // merges the used ones.  The split holding the new key (the row's last
  // non-empty one) arrives for itself and for every empty split after it,
  // which then do nothing at all; a row whose only split is split 0 writes
  // its output directly.  Every round adds exactly `splits` per (row, kv
  // head) counter (monotonic over epochs).  An owner-merges variant (the
  // others leave without the atomic's round trip) measured far slower: with
  // the longest items first, the short owner split waits for full splits
  // still streaming (attention 64 -> 94 us per layer at 1.5B).
  unsigned* my_ctr = &ctr[m * nkv + kh];
  const unsigned weight = owner ? (unsigned)(splits - split) : 1u;
  if (nkeys == 0) return false;  // a split past the context: the owner split arrived for it

  // K/V tiles: warp w streams tiles w, w + 8, ... into buffer slot 7 - w, so the
  // first tiles land in the slots the QKV partial staging does not alias and
  // their loads are issued now, under the partials' L2 round trip
  const __nv_bfloat16* kc = P.kc + P.kv_layer_elems * layer;
  const __nv_bfloat16* vc = P.vc + P.kv_layer_elems * layer;
  uint8_t* kb = tiles + (kCW - 1 - warp) * A::warp_bytes;
  uint8_t* vb = kb + A::kbuf;
  // K and V of a tile travel as two cp.async groups, so the next tile's K
  // streams in while this tile's softmax and P.V run, and its V while the
  // next S = Q K^T runs (the same two buffers per warp, no extra smem)
  auto tile_base = [&](int t, int page) {
    const int key0 = k0 + t * KT;
    return (((size_t)page * nkv + kh) * kPageTokens + (key0 % kPageTokens)) * HD;
  };
  auto load_k = [&](int t, int page) {
    const int nv = min(KT, k1 - (k0 + t * KT));
    const uint4* kg = reinterpret_cast<const uint4*>(kc + tile_base(t, page));
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int e = lane + 32 * i, r = e / V4, c = e % V4;
      if (r < nv) cp_async16(kb + r * A::ROW + c * 16, kg + e);
    }
    cp_async_commit();
  };
  auto load_v = [&](int t, int page) {
    const int nv = min(KT, k1 - (k0 + t * KT));
    const uint4* vg = reinterpret_cast<const uint4*>(vc + tile_base(t, page));
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int e = lane + 32 * i, r = e / V4, c = e % V4;
      if (r < nv) cp_async16(vb + r * A::VROW + c * 16, vg + e);
      else  // P is 0 there, but 0 x a stale NaN pattern is NaN in the MMA
        *reinterpret_cast<uint4*>(vb + r * A::VROW + c * 16) = make_uint4(0u, 0u, 0u, 0u);
    }
    cp_async_commit();
  };
  auto load_tile = [&](int t, int page) {
    load_k(t, page);
    load_v(t, page);
  };
  auto tile_page = [&](int t) { return P.block_table[(size_t)slot * P.pps + (k0 + t * KT) / kPageTokens]; };
  const bool use_qpre = qpre != nullptr;  // partials in their own buffer: every warp's first tile loads early
  const bool pre_bulk = pre && anx->bulk;
  const int free_slot0 =
      (P.pairs || use_qpre) ? 0 : (qkv_cs * W * 4 + (int)A::warp_bytes - 1) / (int)A::warp_bytes;
  const bool early = warp < ntiles && kCW - 1 - warp >= free_slot0;
  if (P.pairs) {
    if (early) load_tile(warp, P.block_table[(size_t)slot * P.pps + (k0 + warp * KT) / kPageTokens]);
    // pair mode: the QKV phase already wrote q (bf16, post-RoPE) and the new
    // token's K/V into the paged cache
    const __nv_bfloat16* qrow = P.q + (size_t)m * nq * HD + (size_t)kh * G * HD;
    for (int i = ct; i < 16 * HD; i += kCT)
      sqb[(i / HD) * A::QP + i % HD] = i < G * HD ? qrow[i] : __float2bfloat16(0.f);
    csync();
  } else {
  // ---- (1) operands: split partials (bulk), pages, bias, rope, rstd -- all in flight
  float* stage = use_qpre ? qpre : reinterpret_cast<float*>(tiles);  // [qkv_cs][W]
  if (ct == 0 && !pre_bulk) {  // the row's partials are contiguous: [m][kh][split][W]
    // (the writers fenced generic -> async proxy before their phase arrival)
    mbar_arrive_expect_tx(cbar, (uint32_t)(qkv_cs * W * 4));
    bulk_g2s(stage, P.qkv_part + ((size_t)m * nkv + kh) * qkv_cs * W, qkv_cs * W * 4, cbar);
    if (tr && tr[4] == 0) tr[4] = clock64() - c_start;
  }
  // every independent load first (one L2 round trip for all of them), the
  // consumers after: the early tile's page, the new token's page, the bias
  // (raw bf16 bits), RoPE cos / sin, the row's x^2 partials
  const int page_early = !early ? 0
                         : pre ? anx->pages[(warp * KT) / kPageTokens]
                               : P.block_table[(size_t)slot * P.pps + (k0 + warp * KT) / kPageTokens];
  const int cpage = pre ? anx->cpage : P.block_table[(size_t)slot * P.pps + pos / kPageTokens];
  constexpr int half = HD / 2;
  unsigned short bbits[WPT];
  float co[WPT], si[WPT];
  float ss = 0.f;
  if (pre && anx->bulk == 2) {
    // the lookahead warp copied the partials AND the bias slice, the cos / sin
    // row and the x^2 partials (mk_attn_extras): tiles first, then one wait
    if (early) load_tile(warp, page_early);
    for (int i = ct; i < (16 - G) * HD; i += kCT)
      sqb[(G + i / HD) * A::QP + i % HD] = __float2bfloat16(0.f);
    if (tr && ct == 0 && tr[1] == 0) tr[1] = clock64() - c_start;
    mk_wait(cbar, cph);
    cph ^= 1;
    const uint8_t* ext = reinterpret_cast<const uint8_t*>(stage) + (size_t)qkv_cs * W * 4;
    const unsigned short* sbias = reinterpret_cast<const unsigned short*>(ext);
    const float* scs = reinterpret_cast<const float*>(ext + W * 2);
    const float* sss = scs + HD;
    for (int q = 0; q < P.parts; ++q) ss += sss[q];  // the order of gemm_detail::ssq_row_sum
#pragma unroll
    for (int u = 0; u < WPT; ++u) {
      const int idx = ct + u * kCT;
      bbits[u] = 0;
      co[u] = 1.f;
      si[u] = 0.f;
      if (idx < W) {
        bbits[u] = sbias[idx];
        if (idx < (G + 1) * HD) {
          const int jj = idx % HD, i = jj < half ? jj : jj - half;
          co[u] = scs[i];
          si[u] = scs[half + i];
        }
      }
    }
  } else {
    const unsigned short* bias = reinterpret_cast<const unsigned short*>(P.w + bias_off);
#pragma unroll
    for (int u = 0; u < WPT; ++u) {
      const int idx = ct + u * kCT;
      bbits[u] = 0;
      co[u] = 1.f;
      si[u] = 0.f;
      if (idx < W) {
        const int col = idx < G * HD ? kh * G * HD + idx
                        : idx < (G + 1) * HD ? qend + kh * HD + (idx - G * HD)
                                             : kend + kh * HD + (idx - (G + 1) * HD);
        bbits[u] = bias[col];
        if (idx < (G + 1) * HD) {
          const int jj = idx % HD, i = jj < half ? jj : jj - half;
          co[u] = P.cos_sin[(size_t)pos * HD + i];
          si[u] = P.cos_sin[(size_t)pos * HD + half + i];
        }
      }
    }
    ss = gemm_detail::ssq_row_sum(P.ssq + (size_t)m * P.parts, P.parts);
    if (tr && ct == 0 && tr[6] == 0) tr[6] = clock64() - c_start;
    if (early) load_tile(warp, page_early);
    for (int i = ct; i < (16 - G) * HD; i += kCT)
      sqb[(G + i / HD) * A::QP + i % HD] = __float2bfloat16(0.f);
    if (tr && ct == 0 && tr[1] == 0) tr[1] = clock64() - c_start;
    mk_wait(cbar, cph);
    cph ^= 1;
  }
  float bia[WPT];
#pragma unroll
  for (int u = 0; u < WPT; ++u) bia[u] = __uint_as_float((unsigned)bbits[u] << 16);
  const float rstd = rsqrtf(ss * P.inv_h + P.eps);
  if (tr && ct == 0 && tr[2] == 0) tr[2] = clock64() - c_start;
#pragma unroll
  for (int u = 0; u < WPT; ++u) {
    const int idx = ct + u * kCT;
    if (idx < W) {
      float v = 0.f;
#pragma unroll 1
      for (int q = 0; q < qkv_cs; ++q) v += stage[q * W + idx];
      sraw[idx] = v * rstd + bia[u];
    }
  }
  csync();
  if (tr && ct == 0 && tr[5] == 0) tr[5] = clock64() - c_start;
  {
    const size_t at = (((size_t)cpage * nkv + kh) * kPageTokens + (pos % kPageTokens)) * HD;
    __nv_bfloat16* kcw = P.kc + P.kv_layer_elems * layer;
    __nv_bfloat16* vcw = P.vc + P.kv_layer_elems * layer;
#pragma unroll
    for (int u = 0; u < WPT; ++u) {
      const int idx = ct + u * kCT;
      if (idx >= W) continue;
      const int jj = idx % HD, base = idx - jj;
      float y;
      if (idx < (G + 1) * HD) {  // RoPE (rotate pairs (i, i + hd/2)) on q heads and k
        const int i = jj < half ? jj : jj - half;
        const float x1 = sraw[base + i], x2 = sraw[base + i + half];
        y = jj < half ? x1 * co[u] - x2 * si[u] : x2 * co[u] + x1 * si[u];
      } else {
        y = sraw[idx];
      }
      const __nv_bfloat16 b = __float2bfloat16(y);
      if (idx < G * HD) {
        sqb[(idx / HD) * A::QP + jj] = b;
      } else if (idx < (G + 1) * HD) {
        snew[jj] = b;
        if (owner) kcw[at + jj] = b;
      } else {
        snew[HD + jj] = b;
        if (owner) vcw[at + jj] = b;
      }
    }
  }
  csync();
  }

  if (tr && ct == 0 && tr[11] == 0) tr[11] = clock64() - c_start;
  // ---- (2) keys: each warp streams its tiles; S = Q K^T and O += P V on the
  // tensor cores (mma.sync m16n8k16: rows = the G query heads padded to 16)
  constexpr int NKT = KT / 8, NDT = HD / 8;
  float o[NDT][4];
#pragma unroll
  for (int n = 0; n < NDT; ++n)
#pragma unroll
    for (int i = 0; i < 4; ++i) o[n][i] = 0.f;
  float m_lo = -INFINITY, m_hi = -INFINITY, l_lo = 0.f, l_hi = 0.f;  // heads lane/4, lane/4 + 8
  if (warp < ntiles && !early) load_tile(warp, tile_page(warp));
  for (int t = warp; t < ntiles; t += kCW) {
    const int key0 = k0 + t * KT;
    const int nv = min(KT, k1 - key0);
    const bool has_next = t + kCW < ntiles;
    const int next_page = has_next ? tile_page(t + kCW) : 0;  // lookup latency under this tile
    const bool new_key = !P.pairs && owner && pos >= key0 && pos < key0 + nv;
    if (ct == 0 && !has_next && lookahead) {  // last tiles: the lookahead warp resolves the next item
      anx->phase = p;
      st_release_cta(&anx->req, ++seq);
    }
    cp_async_wait_1();  // pending: K(t), V(t) -> K(t) landed
    __syncwarp();
    if (new_key) {  // the new key from shared memory
      const int r = pos - key0;
      for (int d = lane; d < HD; d += 32) reinterpret_cast<__nv_bfloat16*>(kb + r * A::ROW)[d] = snew[d];
      __syncwarp();
    }
    float sc[NKT][4];
#pragma unroll
    for (int n = 0; n < NKT; ++n)
#pragma unroll
      for (int i = 0; i < 4; ++i) sc[n][i] = 0.f;
    const __nv_bfloat16* kt = reinterpret_cast<const __nv_bfloat16*>(kb);
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk) {
      uint32_t a[4];
      const __nv_bfloat16* qa = sqb + (lane >> 2) * A::QP + kk * 16 + (lane & 3) * 2;
      a[0] = ld_b32(qa);
      a[1] = ld_b32(qa + 8 * A::QP);
      a[2] = ld_b32(qa + 8);
      a[3] = ld_b32(qa + 8 * A::QP + 8);
#pragma unroll
      for (int n = 0; n < NKT; ++n) {
        const __nv_bfloat16* kp = kt + (n * 8 + (lane >> 2)) * (A::ROW / 2) + kk * 16 + (lane & 3) * 2;
        mma16816(sc[n], a, ld_b32(kp), ld_b32(kp + 8));
      }
    }
    __syncwarp();  // every lane is done with K(t)
    if (has_next) load_k(t + kCW, next_page);
    float mx_lo = m_lo, mx_hi = m_hi;
#pragma unroll
    for (int n = 0; n < NKT; ++n)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int key = n * 8 + (lane & 3) * 2 + (i & 1);
        sc[n][i] = key < nv ? sc[n][i] * P.scale : -INFINITY;
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
    for (int n = 0; n < NKT; ++n)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float mm = i < 2 ? m_lo : m_hi;
        const float pv = sc[n][i] == -INFINITY ? 0.f : __expf(sc[n][i] - mm);
        sc[n][i] = pv;
        if (i < 2) sum_lo += pv;
        else sum_hi += pv;
      }
    l_lo = l_lo * c_lo + sum_lo;  // per-lane partial sums (quad-reduced at the end)
    l_hi = l_hi * c_hi + sum_hi;
#pragma unroll
    for (int n = 0; n < NDT; ++n) {
      o[n][0] *= c_lo; o[n][1] *= c_lo;
      o[n][2] *= c_hi; o[n][3] *= c_hi;
    }
    // pending: V(t) [, K(t + 8)] -> V(t) landed
    if (has_next) cp_async_wait_1();
    else cp_async_wait_all();
    __syncwarp();
    if (new_key) {
      const int r = pos - key0;
      for (int d = lane; d < HD; d += 32) reinterpret_cast<__nv_bfloat16*>(vb + r * A::VROW)[d] = snew[HD + d];
      __syncwarp();
    }
    // P enters as hi + lo bf16 halves (two MMAs on the same V fragment): ~16
    // mantissa bits, so P.V keeps fp32-class accuracy (the oracle's P is fp64)
#pragma unroll
    for (int ks = 0; ks < KT / 16; ++ks) {
      uint32_t ah[4], al[4];
      split_bf16(sc[2 * ks][0], sc[2 * ks][1], ah[0], al[0]);
      split_bf16(sc[2 * ks][2], sc[2 * ks][3], ah[1], al[1]);
      split_bf16(sc[2 * ks + 1][0], sc[2 * ks + 1][1], ah[2], al[2]);
      split_bf16(sc[2 * ks + 1][2], sc[2 * ks + 1][3], ah[3], al[3]);
#pragma unroll
      for (int n = 0; n < NDT; ++n) {
        uint32_t b0, b1;
        ldsm_x2_trans(b0, b1, vb, A::VROW, ks * 16, n * 8, lane);
        mma16816(o[n], ah, b0, b1);
        if (!(P.dbg & 1)) mma16816(o[n], al, b0, b1);  // SRL_MK_DBG=1: single bf16 P (A/B)
      }
    }
    __syncwarp();  // every lane is done with V(t)
    if (has_next) load_v(t + kCW, next_page);
  }
#pragma unroll
  for (int off = 1; off <= 2; off <<= 1) {
    l_lo += __shfl_xor_sync(0xffffffffu, l_lo, off);
    l_hi += __shfl_xor_sync(0xffffffffu, l_hi, off);
  }

  // ---- (3) merge the warps, then the splits
  if (tr && ct == 0 && tr[12] == 0) tr[12] = clock64() - c_start;
  csync();  // sm_acc aliases the tiles
  if (tr && ct == 0 && tr[13] == 0) tr[13] = clock64() - c_start;
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
  csync();
  float* my_ws = ws + (((size_t)m * nkv + kh) * splits + split) * rec;
  // single-split rows (split 0 holds the new key) need no partials at all
  const bool direct = splits == 1 || (owner && split == 0);
  for (int i = ct; i < G * HD; i += kCT) {
    const int g = i / HD, d = i % HD;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < kCW; ++w) M = fmaxf(M, sm_m[w][g]);
    float L = 0.f, Acc = 0.f;
#pragma unroll
    for (int w = 0; w < kCW; ++w) {
      const float a = (sm_m[w][g] == -INFINITY) ? 0.f : __expf(sm_m[w][g] - M);
      L += sm_l[w][g] * a;
      Acc += sm_acc[w][g][d] * a;
    }
    if (direct) {
      P.attn[(size_t)m * nq * HD + (kh * G + g) * HD + d] = __float2bfloat16(L > 0.f ? Acc / L : 0.f);
    } else {
      __stcg(&my_ws[g * (HD + 2) + 2 + d], Acc);
      if (d == 0) {
        __stcg(&my_ws[g * (HD + 2)], M);
        __stcg(&my_ws[g * (HD + 2) + 1], L);
      }
    }
  }
  if (!direct) {
    csync();
    if (ct == 0) {
      __threadfence();
      *s_flag = (atomicAdd(my_ctr, weight) + weight == ep1 * (unsigned)splits);
    }
    csync();
    if (*s_flag) {  // last to arrive: merge the used splits in split order
      __threadfence();
      const float* base = ws + ((size_t)m * nkv + kh) * splits * rec;
      const int used = min(splits, (ctx + P.attn_chunk - 1) / P.attn_chunk);
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
  } else if (splits > 1 && ct == 0) {  // nobody waits on this arrival
    asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(my_ctr), "r"(weight) : "memory");
  }
  if (!lookahead) {  // the caller grabs (or the phase is a static deal)
    csync();
    return false;
  }
  if (ct == 0) {  // the lookahead warp's answer (normally long ready)
    SpinGuard g;
    while (ld_acquire_cta(&anx->done) != seq) g.tick();
    *s_next = anx->item;
  }
  csync();  // (the tiles / sm_acc and s_flag are reused by the next item; *s_next is published)
  if (tr && ct == 0 && tr[14] == 0) tr[14] = clock64() - c_start;
  return true;
}

// plan copy + embedding + first RMSNorm statistics for row m.  red: one
// partial per (128-column part, warp-quarter of the part).
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
  const int cols = P.parts * 128;
#pragma unroll 4
  for (int c = ct; c < cols; c += kCT) {  // a warp's 32 columns lie in one part
    float v = 0.f;
    if (c < P.H) {
      v = ok ? bf2f(E[(size_t)tok * P.H + c]) : 0.f;
      P.x[(size_t)m * P.H + c] = v;
      P.xg[(size_t)m * P.H + c] = __float2bfloat16(v * bf2f(g[c]));
    }
    const float s = wsum(v * v);
    if ((ct & 31) == 0) red[c >> 5] = s;
  }
  csync();
  for (int p = ct; p < P.parts; p += kCT)
    P.ssq[(size_t)m * P.parts + p] = red[p * 4] + red[p * 4 + 1] + red[p * 4 + 2] + red[p * 4 + 3];
  csync();
}

// This round's attention items, longest first (one CTA, in the embed phase;
// the plan of the round is P.next until the embed items copy it): the full
// attn_chunk-key splits in split-major order, then the partial splits by key
// count (descending), then the empty ones -- the work queue of every attention
// phase hands them out in this order, so the phase ends on short items
// instead of a full split started late.  sm: >= 2 n + 2 ints of scratch
// (n <= kMkMaxAttnItems: 32 KB at 8 KB into the scratch area).
__device__ void mk_attn_order(const MkParams& P, int ct, int* sm) {
  const int rowheads = P.S * P.nkv, n = rowheads * P.attn_splits, chunk = P.attn_chunk;
  int* cnt = sm;       // [n] keys of each item (-1: free slot)
  int* part = sm + n;  // the partial items, index order
  for (int i = ct; i < n; i += kCT) {
    const int split = i / rowheads, m = (i % rowheads) / P.nkv;
    int c = -1;
    if (P.next.row_slot[m] >= 0) c = min(chunk, max(0, P.next.row_pos[m] + 1 - split * chunk));
    cnt[i] = c;
  }
  csync();
  if (ct < 32) {  // ballot compaction: full items into the order, partial ones into part[]
    int nf = 0, np = 0;
    const unsigned lower = (1u << ct) - 1u;
    for (int b = 0; b < n; b += 32) {
      const int i = b + ct;
      const int c = i < n ? cnt[i] : -1;
      const bool full = c == chunk, partial = c > 0 && c < chunk;
      const unsigned mf = __ballot_sync(0xffffffffu, full), mp = __ballot_sync(0xffffffffu, partial);
      if (full) P.attn_order[nf + __popc(mf & lower)] = i;
      if (partial) part[np + __popc(mp & lower)] = i;
      nf += __popc(mf);
      np += __popc(mp);
    }
    if (ct == 0) {
      sm[2 * n] = nf;
      sm[2 * n + 1] = np;
    }
  }
  csync();
  const int nf = sm[2 * n], np = sm[2 * n + 1];
  for (int j = ct; j < np; j += kCT) {  // rank of a partial item by key count, ties by index
    const int c = cnt[part[j]];
    int r = 0;
    for (int k = 0; k < np; ++k) {
      const int ck = cnt[part[k]];
      r += (ck > c) || (ck == c && k < j);
    }
    P.attn_order[nf + r] = part[j];
  }
  if (ct < 32) {  // empty splits and free slots last
    int ne = 0;
    const unsigned lower = (1u << ct) - 1u;
    for (int b = 0; b < n; b += 32) {
      const int i = b + ct;
      const bool rest = i < n && cnt[i] <= 0;
      const unsigned mr = __ballot_sync(0xffffffffu, rest);
      if (rest) P.attn_order[nf + np + ne + __popc(mr & lower)] = i;
      ne += __popc(mr);
    }
  }
  csync();
}

// Sampling of slot s from the LM-head tile partials (256 threads): the tile
// (max, sum) pairs of the row are loaded once into registers; lse; then the
// inverse CDF: tile masses, block exclusive scan (warp shuffles), first tile
// whose range may hold u (1e-12 margin), and warp 0 walks that tile element
// by element in fp64 (the sampler of decoder.cu, same numerics class).
constexpr int kSampleC = 8;  // tiles per thread held in registers (V <= 262144)
__device__ void mk_sample(const MkParams& P, int s, int ct, uint8_t* scr, unsigned long long* tr) {
  const long long c0 = clock64();
  auto stampc = [&](int k) { if (tr && ct == 0 && tr[k] == 0) tr[k] = clock64() - c0; };
  double* wtot = reinterpret_cast<double*>(scr);  // [kCW]
  double* red = wtot + kCW;                       // [kCW]
  int* iv = reinterpret_cast<int*>(red + kCW);    // [kCW + 1]
  float* fv = reinterpret_cast<float*>(iv + kCW + 2);
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
  const int C = (T + kCT - 1) / kCT;  // <= kSampleC
  const int t0 = ct * C, t1 = min(T, t0 + C);
  float pm[kSampleC];
  double ps[kSampleC];
#pragma unroll
  for (int q = 0; q < kSampleC; ++q) {
    const bool ok = q < C && t0 + q < t1;
    pm[q] = ok ? P.lse_max[(size_t)s * T + t0 + q] : -INFINITY;
    ps[q] = ok ? P.lse_sum[(size_t)s * T + t0 + q] : 0.0;
  }
  const uint64_t seed = P.ss.seed[s];
  const int gen0 = P.ss.gen_count[s];
  // the event's scalars, loaded now (off the critical path)
  const int pos_row = P.plan.row_pos[r];
  const int term = P.ss.terminator[s], maxtok = P.ss.max_tokens[s], ver = *P.version;
  stampc(10);
  float mx = -INFINITY;
  int mt = 0x7fffffff;
#pragma unroll
  for (int q = 0; q < kSampleC; ++q)
    if (pm[q] > mx) { mx = pm[q]; mt = t0 + q; }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float om = __shfl_xor_sync(0xffffffffu, mx, o);
    const int oi = __shfl_xor_sync(0xffffffffu, mt, o);
    if (om > mx || (om == mx && oi < mt)) { mx = om; mt = oi; }
  }
  if (lane == 0) { fv[warp] = mx; iv[warp] = mt; }
  csync();
  float Mf = fv[0];
  int mtile = iv[0];
  for (int w = 1; w < kCW; ++w)
    if (fv[w] > Mf || (fv[w] == Mf && iv[w] < mtile)) { Mf = fv[w]; mtile = iv[w]; }
  const double M = (double)Mf;
  double part = 0.0;
  double em[kSampleC];  // s_t * exp(m_t - M): reused for the tile masses
#pragma unroll
  for (int q = 0; q < kSampleC; ++q) {
    em[q] = ps[q] * exp_nonpos_call((double)pm[q] - M);
    part += em[q];
  }
  part = wsum_d(part);
  if (lane == 0) red[warp] = part;
  csync();
  double tot = 0.0;
  for (int w = 0; w < kCW; ++w) tot += red[w];
  const double lse = M + log(tot);
  const double u = uniform_draw(seed, (uint64_t)gen0);
  stampc(11);
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
      if (lane == 0) iv[kCW] = best == 0x7fffffff ? mtile * kLmTile : best;
    }
    csync();
    tok = iv[kCW];
  } else {
    double mass[kSampleC];
    double mine = 0.0;
    const double scale = exp_nonpos_call(M - lse);  // tile mass = s_t exp(m_t - M) exp(M - lse)
#pragma unroll
    for (int q = 0; q < kSampleC; ++q) {
      mass[q] = em[q] * scale;
      mine += mass[q];
    }
    // exclusive scan of the threads' masses: warp shuffles, then warp totals
    double incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double n = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += n;
    }
    if (lane == 31) wtot[warp] = incl;
    csync();
    double off = 0.0;
    for (int w = 0; w < warp; ++w) off += wtot[w];
    const double excl = off + (incl - mine);
    int cand = 0x7fffffff;
    if (u < excl + mine + 1e-12) {
      double base = excl;
#pragma unroll
      for (int q = 0; q < kSampleC; ++q) {
        if (cand == 0x7fffffff && t0 + q < t1) {
          if (u < base + mass[q] + 1e-12) cand = t0 + q;
          base += mass[q];
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cand = min(cand, __shfl_xor_sync(0xffffffffu, cand, o));
    if (lane == 0) iv[warp] = cand;
    // the candidate's base: the owner thread's exclusive prefix + its earlier tiles
    csync();
    int t = 0x7fffffff;
    for (int w = 0; w < kCW; ++w) t = min(t, iv[w]);
    if (t != 0x7fffffff && ct == t / C) {
      double base = excl;
#pragma unroll
      for (int q = 0; q < kSampleC; ++q)
        if (t0 + q < t) base += mass[q];
      red[0] = base;
    }
    csync();
    stampc(12);
    if (warp == 0) {
      int tk = V - 1;
      if (t != 0x7fffffff) {
        double base = red[0];
        bool done = false;
        for (; t < T && !done; ++t) {
          double p[4];
          double ls = 0.0;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int k = t * kLmTile + lane * 4 + i;
            p[i] = k < V ? exp_nonpos_call((double)x[k] - lse) : 0.0;
            ls += p[i];
          }
          double in2 = ls;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const double n = __shfl_up_sync(0xffffffffu, in2, o);
            if (lane >= o) in2 += n;
          }
          double cum = base + (in2 - ls);
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
          base += __shfl_sync(0xffffffffu, in2, 31);
        }
      }
      if (lane == 0) iv[kCW] = tk;
    }
    csync();
    tok = iv[kCW];
  }
  stampc(13);
  if (ct == 0) {
    const int new_len = pos_row + 1;
    const int gen = gen0;
    int flag = 1;
    if (tok == term) flag = 3;
    else if (gen + 1 >= maxtok) flag = 2;
    else if (new_len + 1 > P.ss.max_seq) flag = 2;
    DevEvent e;
    e.flag = flag;
    e.token = tok;
    e.position = gen;
    e.version = ver;
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
  stampc(14);
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
  uint64_t* cbar = tempty + 2;  // compute warps' bulk-copy barrier
  uint64_t* xbar = cbar + 1;    // pair phases: the partner CTA's partial rows have landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + Lo::misc);
  int* s_flag = reinterpret_cast<int*>(smem + Lo::misc + 4);
  int* s_seen = reinterpret_cast<int*>(smem + Lo::misc + 8);  // last phase seen complete
  int* s_next = reinterpret_cast<int*>(smem + Lo::misc + 12);  // attention: the CTA's next queue item
  MkAnx* anx = reinterpret_cast<MkAnx*>(smem + Lo::anx);
  float* s_rstd = reinterpret_cast<float*>(smem + Lo::rstd);
  int2* s_rows = reinterpret_cast<int2*>(smem + Lo::rows);

  const int warp = threadIdx.x >> 5;
  const int GR = gridDim.x, c = blockIdx.x;
  const unsigned ep1 = *P.epoch + 1u;
  const unsigned target = ep1 * (unsigned)GR;

  if (threadIdx.x == 64) {
    *s_seen = 0;
    anx->req = 0;
    anx->done = 0;
  }
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
      mbar_init(cbar, 1);
      mbar_init(xbar, 1);
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
          // dataflow phases: k-block kb's activations are ready once the
          // producing tile's done counter reaches its per-round target
          const bool flow = F.flow_ctr >= 0;
          int flow_seen = -1;
          auto flow_wait = [&](int kb) {
            const int t = (kb * kBK) / F.flow_cols;
            if (t == flow_seen) return;
            wait_count(&P.tile_ctr[F.flow_ctr + t], ep1 * (unsigned)F.flow_target);
            fence_proxy_async_global();  // generic-proxy results -> TMA reads
            flow_seen = t;
          };
          // the rest of the first item's weight boxes go to L2 while the
          // previous phase finishes (its HBM time is mostly idle: split-K
          // exchanges, barriers), so this phase streams them from L2
          // (SRL_MK_L2PF=0: off, A/B)
          if (!dep_ok && P.l2_prefetch)
            for (int k = pre; k < nkb; ++k) tma_prefetch_2d_l2(tw, (kb0 + k) * kBK, n0);
          if (!dep_ok && !flow) {
            // the compute warps' poller publishes each completed phase here
            // (one global poller per CTA)
            {
              SpinGuard g;
              while (ld_acquire_cta(s_seen) < p) g.tick();
            }
            fence_proxy_async_global();  // generic-proxy results -> TMA reads
            dep_ok = true;
            if (P.trace) P.trace[((size_t)p * GR + c) * 16 + 4] = clock64();  // raw cycles
          }
          for (int k = 0; k < pre; ++k) {
            const int st = (s0 + k) % STAGES;
            if (flow) flow_wait(kb0 + k);
            tma_load_2d(smem + st * kStageBytes + kABytes, tx, &full[st], (kb0 + k) * kBK, 0);
          }
          for (int k = pre; k < nkb; ++k) {
            mk_wait(&empty[stage], ph ^ 1);
            mbar_arrive_expect_tx(&full[stage], kStageBytes);
            uint8_t* a = smem + stage * kStageBytes;
            tma_load_2d_hint(a, tw, &full[stage], (kb0 + k) * kBK, n0, pol);
            if (flow) flow_wait(kb0 + k);
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
          unsigned long long* trm = P.trace ? P.trace + ((size_t)p * GR + c) * 16 : nullptr;
          for (int k = 0; k < nkb; ++k) {
            mk_wait(&full[stage], ph);
            tc_fence_after();
            if (trm && k == 0 && trm[14] == 0) trm[14] = clock64();  // raw cycles
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
          if (trm && trm[15] == 0) trm[15] = clock64();  // raw cycles
          if (++acc == 2) { acc = 0; aph ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp == 3) {
    // ------------------------------------------- attention lookahead (MkAnx)
    if (elect_one()) {
      int seen = 0;
      constexpr int W = (G + 2) * HD, KT = AttnSmem<HD, G>::KT, NPG = kCW * KT / kPageTokens;
      static_assert(NPG <= 8, "mailbox pages");
      while (true) {
        int r;
        {
          SpinGuard g;
          while ((r = ld_acquire_cta(&anx->req)) == seen) {
            __nanosleep(32);
            g.tick();
          }
        }
        seen = r;
        const int p = anx->phase;
        if (p < 0) break;  // the compute warps are done
        const MkPhase& F = P.phases[p];
        const int i = mk_queue(P, F, ep1, GR).resolve(mk_queue(P, F, ep1, GR).grab());
        int bulk = 0;
        if (i >= 0) {
          const int rowheads = P.S * P.nkv, split = i / rowheads, rest = i % rowheads;
          const int m = rest / P.nkv, kh = rest % P.nkv;
          const int2 sr = s_rows[m];
          const int k0 = split * P.attn_chunk, k1 = min(sr.y + 1, k0 + P.attn_chunk);
          if (sr.x >= 0 && k1 > k0) {
            const int32_t* btr = P.block_table + (size_t)sr.x * P.pps;
            const int pg0 = k0 / kPageTokens;
            int pg[NPG];
#pragma unroll
            for (int w = 0; w < NPG; ++w) pg[w] = (pg0 + w) * kPageTokens < k1 ? btr[pg0 + w] : 0;
            const int cp = btr[sr.y / kPageTokens];
            const uint32_t bytes = (uint32_t)(F.cs * W * 4);
            // extras (mk_attention reads them when bulk == 2): the bias slice
            // [q heads | k | v] of this kv head, the cos / sin row of the new
            // position and the row's x^2 partials -- every operand of the item's
            // q / k / v in one wait.  (Tensors are 128-byte aligned; the x^2
            // row needs parts % 4 == 0.)
            const uint32_t xb = (uint32_t)(W * 2 + HD * 4 + P.parts * 4);
            const bool ext = (P.parts & 3) == 0 && Lo::qpre_bytes >= bytes + xb;
            if (Lo::qpre_bytes >= bytes) {
              fence_proxy_async_shared();  // the previous item's generic reads of qpre, then the bulk write
              mbar_arrive_expect_tx(cbar, bytes + (ext ? xb : 0u));
              uint8_t* dst = smem + Lo::qpre;
              bulk_g2s(dst, P.qkv_part + ((size_t)m * P.nkv + kh) * F.cs * W, bytes, cbar);
              if (ext) {
                const int qend = P.nq * HD, kend = qend + P.nkv * HD;
                const __nv_bfloat16* b = P.w + F.colv;
                uint8_t* x = dst + bytes;
                bulk_g2s(x, b + kh * G * HD, G * HD * 2, cbar);
                bulk_g2s(x + G * HD * 2, b + qend + kh * HD, HD * 2, cbar);
                bulk_g2s(x + (G + 1) * HD * 2, b + kend + kh * HD, HD * 2, cbar);
                bulk_g2s(x + W * 2, P.cos_sin + (size_t)sr.y * HD, HD * 4, cbar);
                bulk_g2s(x + W * 2 + HD * 4, P.ssq + (size_t)m * P.parts, P.parts * 4, cbar);
              }
              bulk = ext ? 2 : 1;
            }
#pragma unroll
            for (int w = 0; w < NPG; ++w) anx->pages[w] = pg[w];
            anx->cpage = cp;
          }
        }
        anx->item = i;
        anx->bulk = bulk;
        st_release_cta(&anx->done, r);
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ------------------------------------------------------ compute
    const int ct = threadIdx.x - 128, cw = ct >> 5, lane = ct & 31;
    const int col = ct & (kBN - 1);      // accumulator lane (= output column) drained
    const int hf = cw >> 2;              // token half [32 hf, 32 hf + 32) drained
    uint32_t cph = 0;                    // cbar phase
    uint32_t xph = 0;                    // xbar phase
    bool rows_ready = false;
    int seq = 0;  // lookahead requests posted (ct 0)
    const bool stamp = P.stamps != nullptr && c == 0 && ct == 0;
    int acc = 0;
    uint32_t aph = 0;
    if (stamp) P.stamps[0] = globaltimer();
    for (int p = 0; p < P.n_phases; ++p) {
      const MkPhase& F = P.phases[p];
      // the first item's epilogue column constant (a weight: independent of
      // the barrier below) -- its global load latency overlaps the wait
      unsigned short colv0 = 0;
      const long long colv_off = (F.kind == MK_O || F.kind == MK_DOWN) ? F.colv : -1;
      if (colv_off >= 0) {
        const int i0 = first_item(c, F.rot, GR);
        const int n = (i0 / F.cs) * kBN + col;
        if (i0 < F.n_items && n < F.N) colv0 = reinterpret_cast<const unsigned short*>(P.w)[colv_off + n];
      }
      const bool flow_phase = F.flow_ctr >= 0;
      if (p > 0 && !flow_phase) {  // results of the previous phase, grid-wide
        if (ct == 0) {
          phase_wait(P.phase_done, p - 1, target);
          st_release_cta(s_seen, p);
          if (stamp) P.stamps[p] = globaltimer();
        }
        csync();
      }
      unsigned long long* tr = P.trace ? P.trace + ((size_t)p * GR + c) * 16 : nullptr;
      if (tr && ct == 0) {
        tr[0] = globaltimer();
        tr[8] = clock64();
      }
      if (F.kind == MK_EMBED) {
        if (c == 0 && ct == 0) *P.round_ctr += 1;
        for (int m = first_item(c, F.rot, GR); m < F.n_items; m += GR)
          mk_embed(P, m, ct, reinterpret_cast<float*>(scratch));
        if (c == GR - 1 && P.S * P.nkv * P.attn_splits > GR)  // (a static deal needs no order)
          mk_attn_order(P, ct, reinterpret_cast<int*>(scratch + 8192));
      } else if (F.kind == MK_ATTN) {
        if (!rows_ready) {  // the round's plan, once per CTA
          for (int j = ct; j < P.S; j += kCT) s_rows[j] = make_int2(P.plan.row_slot[j], P.plan.row_pos[j]);
          csync();
          rows_ready = true;
        }
        // items are taken from a work queue (one counter per attention phase,
        // after its split counters): item cost follows the row's context, so a
        // static deal left CTAs idle at the phase barrier.  Every CTA makes
        // exactly one failing grab, so a launch adds n_items + grid to the
        // counter and (epoch x that) is this launch's base.  The queue position
        // maps through attn_order (longest items first, built in the embed phase).
        const MkQueue qu = mk_queue(P, F, ep1, GR);
        const int rowheads = P.S * P.nkv;
        float* qpre = (Lo::qpre_bytes >= (size_t)F.cs * (G + 2) * HD * 4)
                          ? reinterpret_cast<float*>(smem + Lo::qpre) : nullptr;
        // at most one item per CTA (short contexts, e.g. 0.5B / 256-token
        // rollouts): a static deal -- no queue atomic, no order lookup, no
        // lookahead (the queue counter of such a phase is never touched)
        const bool deal = F.n_items <= GR;
        if (deal) {
          if (ct == 0) *s_next = c < F.n_items ? c : -1;
        } else if (ct == 0) {
          *s_next = qu.resolve(qu.grab());  // the phase's first item
        }
        csync();
        bool pre = false;
        int ordinal = 0;  // items taken by this CTA in the phase (trace: stamps of item P.trace_item)
        while (true) {
          const int i = *s_next;  // longest first (mk_attn_order)
          csync();  // everyone has read it
          if (i < 0) break;
          unsigned long long* tri = (tr && ordinal == P.trace_item) ? tr : nullptr;
          ++ordinal;
          if (tr && ct == 0) tr[15] = (unsigned long long)ordinal;
          const int split = i / rowheads;
          const int rest = i % rowheads;
          const long long a_c0 = clock64();
          const bool took = mk_attention<HD, G>(P, F.layer, F.colv, F.cs, rest / P.nkv, rest % P.nkv, split,
                                                scratch, s_rows, P.tile_ctr + F.ctr_base, ep1, P.ws, ct, s_flag,
                                                cbar, cph, tri, anx, pre, qpre, p, seq, s_next,
                                                !deal && !(P.dbg & 2));  // SRL_MK_DBG=2: no lookahead (A/B)
          if (tri && ct == 0 && tri[10] == 0) tri[10] = clock64() - a_c0;
          if (deal) break;
          pre = took;
          if (!took) {
            if (ct == 0) *s_next = qu.resolve(qu.grab());
            csync();
          }
        }
      } else if (F.kind == MK_SAMPLE) {
        for (int s = first_item(c, F.rot, GR); s < F.n_items; s += GR) mk_sample(P, s, ct, scratch, tr);
      } else {
        mk_rows(P, F.kind, s_rstd, ct);
        for (int i = first_item(c, F.rot, GR); i < F.n_items; i += GR) {
          const int tile_n = i / F.cs, split = i % F.cs;
          unsigned short colv_bits = colv0;
          if (i != first_item(c, F.rot, GR) && colv_off >= 0 && tile_n * kBN + col < F.N)
            colv_bits = reinterpret_cast<const unsigned short*>(P.w)[colv_off + tile_n * kBN + col];
          // pair items: register the partner's incoming bytes, and gather what
          // the epilogue needs (it does not depend on this phase) under the MMA
          const bool pair = P.pairs && F.cs == 2;
          const int phalf = (P.S + 1) / 2;
          const int pr0 = split == 0 ? 0 : phalf, pr1 = split == 0 ? phalf : P.S;
          float* xbuf = tile + kTok * kPitch;                            // partner's rows (pitch kPitch)
          int4* s_row4 = reinterpret_cast<int4*>(xbuf + 32 * kPitch);   // QKV row metadata
          float* xs = reinterpret_cast<float*>(s_row4 + kTok);          // O: residual rows (pitch kBN)
          EpiParams qe;
          if (pair) {
            if (ct == 0) mbar_arrive_expect_tx(xbar, (uint32_t)((pr1 - pr0) * kPitch * 4));
            if (F.kind == MK_QKV) {
              qe.kind = EPI_QKV;
              qe.ssq_in = P.ssq; qe.ssq_in_parts = P.parts; qe.inv_dim = P.inv_h; qe.eps = P.eps;
              qe.bias = P.w + P.layers[F.layer].qkv_b;
              qe.nq = P.nq; qe.nkv = P.nkv; qe.hd = P.hd; qe.pages_per_seq = P.pps;
              qe.row_slot = P.plan.row_slot; qe.row_pos = P.plan.row_pos; qe.block_table = P.block_table;
              qe.cos_sin = P.cos_sin; qe.q_out = P.q;
              qe.kc = P.kc + P.kv_layer_elems * F.layer; qe.vc = P.vc + P.kv_layer_elems * F.layer;
              gemm_detail::epi_row_meta(qe, pr0, pr1, 0, P.S, s_rstd, s_row4, ct, kCT);
            } else {  // O: x[pr0, pr1) x 128 columns into xs by cp.async
              const int n0 = tile_n * kBN;
              for (int e = ct; e < (pr1 - pr0) * (kBN / 4); e += kCT) {
                const int j = pr0 + e / (kBN / 4), cc = (e % (kBN / 4)) * 4;
                cp_async16(xs + (j - pr0) * kBN + cc, P.x + (size_t)j * F.N + n0 + cc);
              }
              cp_async_commit();
            }
          }
          mk_wait(&tfull[acc], aph);
          tc_fence_after();
          if (tr && ct == 0 && tr[1] == 0) tr[1] = clock64() - tr[8];
          uint32_t ra[32];
          tmem_ld_32x32b_x32(tmem + acc * kTok + hf * 32 + ((uint32_t)((cw & 3) * 32) << 16), ra);
          tmem_ld_wait();
          tc_fence_before();
          mbar_arrive(&tempty[acc]);  // accumulator free for the MMA warp
          if (++acc == 2) { acc = 0; aph ^= 1; }
          const int j0 = hf * 32;  // tokens of ra
          int r0 = 0, r1 = P.S;
          if (pair) {
            // ---- split-K over the CTA pair (cluster of 2): split s owns rows
            // [pr0, pr1).  Both halves of the partial go to the local tile; the
            // partner's half is shipped in ONE bulk copy into its xbuf, landing
            // on its xbar.  Result = p0 + p1 on both sides (fp add commutes):
            // deterministic.
            const uint32_t other = (uint32_t)split ^ 1u;
            r0 = pr0;
            r1 = pr1;
            const int o0 = split == 0 ? phalf : 0, o1 = split == 0 ? P.S : phalf;
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (j0 + j < P.S) tile[(j0 + j) * kPitch + col] = __uint_as_float(ra[j]);
            fence_proxy_async_shared();
            csync();
            if (ct == 0 && o1 > o0) {
              const uint32_t dst = partner_addr(xbuf, other), bar = partner_addr(xbar, other);
              asm volatile(
                  "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                  ::"r"(dst), "r"(smem_u32(tile + o0 * kPitch)), "r"((uint32_t)((o1 - o0) * kPitch * 4)), "r"(bar)
                  : "memory");
            }
            mk_wait(xbar, xph);
            xph ^= 1;
            if (tr && ct == 0 && tr[2] == 0) tr[2] = clock64() - tr[8];
            for (int e = ct; e < (r1 - r0) * kBN; e += kCT) {
              const int j = r0 + e / kBN, cc = e % kBN;
              tile[j * kPitch + cc] += xbuf[(j - r0) * kPitch + cc];
            }
            if (F.kind == MK_O) cp_async_wait_all();
            csync();
            if (F.kind == MK_QKV) {
              // bias, rstd, RoPE, q -> bf16 rows, k / v -> the paged cache (gemm_epi.cuh)
              gemm_detail::epi_apply(qe, tile, kPitch, r0, r1, 0, tile_n * kBN, tile_n, (F.N + kBN - 1) / kBN,
                                     P.S, F.N, s_rstd, s_row4, ct, kCT, [] { csync(); });
              csync();
              continue;
            }
          } else if (F.kind == MK_QKV) {
            // raw split partial [split][row][col]; the attention items reduce it
            const int n = tile_n * kBN + col;
            if (n < F.N) {  // consumer layout [row][kv head][split][q heads | k | v]
              const int hd = P.hd, qend = P.nq * hd, kend = qend + P.nkv * hd;
              const int Wr = (P.nq / P.nkv + 2) * hd;
              int kh, idx;
              if (n < qend) { kh = n / hd / (P.nq / P.nkv); idx = n - kh * (P.nq / P.nkv) * hd; }
              else if (n < kend) { kh = (n - qend) / hd; idx = (P.nq / P.nkv) * hd + (n - qend) % hd; }
              else { kh = (n - kend) / hd; idx = (P.nq / P.nkv + 1) * hd + (n - kend) % hd; }
              const size_t rstride = (size_t)P.nkv * F.cs * Wr;
              float* ptr = P.qkv_part + ((size_t)kh * F.cs + split) * Wr + idx + (size_t)j0 * rstride;
              const int nj = min(32, P.S - j0);
#pragma unroll
              for (int j = 0; j < 32; ++j) {
                if (j < nj) __stcg(ptr, __uint_as_float(ra[j]));
                ptr += rstride;
              }
            }
            continue;
          } else if (F.cs == 1) {
#pragma unroll
            for (int j = 0; j < 32; ++j) tile[(j0 + j) * kPitch + col] = __uint_as_float(ra[j]);
          } else {
            // publish this split's partial (rows < S), wait for the tile's other
            // splits, then reduce this split's row slice in split order
            float* part = P.ws + (size_t)i * kTileFloats;
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (j0 + j < P.S) __stcg(&part[(j0 + j) * kBN + col], __uint_as_float(ra[j]));
            fence_proxy_async_global();
            if (tr && ct == 0 && tr[11] == 0) tr[11] = clock64() - tr[8];
            r0 = (split * P.S) / F.cs;
            r1 = ((split + 1) * P.S) / F.cs;
            const int nr = r1 - r0;
            float* stage = tile + kTok * kPitch;  // [cs][nr][128]
            csync();
            if (cw == 0) {  // warp 0: arrive, wait for the other splits, fetch the slices
              if (lane == 0) {
                unsigned* tc = &P.tile_ctr[F.ctr_base + tile_n];
                __threadfence();
                atomicAdd(tc, 1u);
                if (tr && tr[12] == 0) tr[12] = clock64() - tr[8];
                wait_count(tc, ep1 * (unsigned)F.cs);
                if (tr && tr[2] == 0) tr[2] = clock64() - tr[8];
                if (nr > 0) mbar_arrive_expect_tx(cbar, (uint32_t)(F.cs * nr * kBN * 4));
              }
              __syncwarp();
              if (nr > 0 && lane < F.cs) {  // one bulk copy per lane, issued in parallel
                // (each writer fenced its partial generic -> async proxy before arriving)
                const float* src = P.ws + (size_t)tile_n * F.cs * kTileFloats + (size_t)r0 * kBN;
                bulk_g2s(stage + (size_t)lane * nr * kBN, src + (size_t)lane * kTileFloats, nr * kBN * 4, cbar);
              }
            }
            if (nr > 0) {
              mk_wait(cbar, cph);
              cph ^= 1;
              const float4* s4 = reinterpret_cast<const float4*>(stage);
              for (int e = ct; e < nr * (kBN / 4); e += kCT) {
                float4 a = s4[e];
                for (int q = 1; q < F.cs; ++q) {
                  const float4 v = s4[(size_t)q * nr * (kBN / 4) + e];
                  a.x += v.x; a.y += v.y; a.z += v.z; a.w += v.w;
                }
                const int j = r0 + e / (kBN / 4), cc = (e % (kBN / 4)) * 4;
                *reinterpret_cast<float4*>(&tile[j * kPitch + cc]) = a;
              }
            }
          }
          if (tr && ct == 0 && tr[5] == 0) tr[5] = clock64() - tr[8];
          csync();
          const float colv = __uint_as_float((unsigned)colv_bits << 16);
          if (r1 > r0) mk_epilogue(P, F, tile_n, tile, s_rstd, ct, r0, r1, colv, pair ? xs : nullptr);
          if (F.done_ctr >= 0) fence_proxy_async_global();  // consumers read with TMA
          csync();
          if (F.done_ctr >= 0 && ct == 0)  // this tile (row slice) is final
            asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(&P.tile_ctr[F.done_ctr + tile_n]),
                         "r"(1u)
                         : "memory");
          if (tr && ct == 0 && tr[6] == 0) tr[6] = clock64() - tr[8];
        }
      }
      fence_proxy_async_global();  // later phases read these results with TMA
      csync();
      if (ct == 0) {
        if (flow_phase) {
          // arrival here must still imply the previous phase is complete
          // (later phases read its other results: ssq, x)
          phase_wait(P.phase_done, p - 1, target);
          st_release_cta(s_seen, p);
          if (stamp) P.stamps[p] = globaltimer();
        }
        if (tr) {
          tr[3] = globaltimer();
          tr[9] = clock64() - tr[8];
        }
        phase_arrive(P.phase_done, p, c);
        if (tr) tr[7] = globaltimer();
      }
    }
    if (ct == 0) {  // release the lookahead warp
      anx->phase = -1;
      st_release_cta(&anx->req, ++seq);
    }
    if (stamp) {
      phase_wait(P.phase_done, P.n_phases - 1, target);
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
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeCooperative;  // co-residency for the phase counters
  at[0].val.cooperative = 1;
  at[1].id = cudaLaunchAttributeClusterDimension;  // pair mode: CTAs 2i, 2i+1 share DSMEM
  at[1].val.clusterDim.x = p.pairs ? 2 : 1;
  at[1].val.clusterDim.y = 1;
  at[1].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = p.pairs ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, decode_megakernel<HD, G>, p);
}

template <int HD, int G>
int qkv_cap_t() {
  return (int)(AttnSmem<HD, G>::tiles / ((size_t)(G + 2) * HD * 4));
}

}  // namespace

int megakernel_splits(int N, int K, int grid) {
  // cost ~ bytes one CTA streams (24 KB per k-block) + a flat charge for the
  // partial exchange; split-K only while the phase still fits one wave
  const int tiles = (N + kBN - 1) / kBN, kb = K / kBK;
  int best = 1;
  long best_cost = (long)((tiles + grid - 1) / grid) * kb * 24;
  for (int cs = 2; cs <= kb && cs <= kMaxCs && tiles * cs <= grid; ++cs) {
    const long cost = (long)((kb + cs - 1) / cs) * 24 + 40;
    if (cost < best_cost) {
      best_cost = cost;
      best = cs;
    }
  }
  return best;
}

int megakernel_qkv_splits(const DecoderDims& d, int grid) {
  const int G = d.nq / d.nkv;
  int cap = 1;
  if (d.hd == 64) cap = G == 2 ? qkv_cap_t<64, 2>() : qkv_cap_t<64, 7>();
  else cap = G == 6 ? qkv_cap_t<128, 6>() : qkv_cap_t<128, 7>();
  cap = cap / 4 > 1 ? cap / 4 : 1;  // staging <= 2 of the 8 K/V warp buffers: 6 tiles load early
  const int cs = megakernel_splits(d.qkv(), d.H, grid);
  return cs < cap ? cs : cap;
}

size_t megakernel_ws_floats(int n_items, int cs, int rows) {
  (void)rows;
  return cs > 1 ? (size_t)n_items * kTileFloats : 0;
}

bool megakernel_supported(const DecoderDims& d, int slots) {
  if (slots > kTok || d.nq % d.nkv) return false;
  if ((d.V + kLmTile - 1) / kLmTile > kSampleC * kCT) return false;  // sampler registers
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

template <int HD, int G>
int pair_clusters_t() {
  if (!set_smem_attr<HD, G>()) return 0;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = MkLayout<HD, G>::alloc;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, decode_megakernel<HD, G>, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int megakernel_pair_clusters(const DecoderDims& d) {
  const int G = d.nq / d.nkv;
  if (d.hd == 64 && G == 2) return pair_clusters_t<64, 2>();
  if (d.hd == 64 && G == 7) return pair_clusters_t<64, 7>();
  if (d.hd == 128 && G == 6) return pair_clusters_t<128, 6>();
  if (d.hd == 128 && G == 7) return pair_clusters_t<128, 7>();
  return 0;
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
