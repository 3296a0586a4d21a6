// gemm_big_impl.cuh -- the persistent tcgen05 GEMM kernel template
// (gemm_big.cu describes it).  Specialised per epilogue kind EK so each
// instance carries only its own epilogue (a kernel holding every variant
// stalled on instruction-cache misses); instantiated in gemm_big_i*.cu.
#pragma once
#include <cstdio>

#include "gemm.cuh"
#include "gemm_epi.cuh"
#include "sm100.cuh"

namespace srl {
namespace bigk {
using namespace sm100;


constexpr int kBN = 128;  // weight rows per tile (UMMA M)
constexpr int kBK = 64;   // k-block (128-B swizzle row)
constexpr int kThreads = 384;
constexpr int kChunk = 32;  // tokens per epilogue chunk
constexpr int kPitch = kBN;  // drain writes are lane-contiguous: no padding needed

template <int TOK>
struct BigLayout {
  static constexpr int STAGES = TOK == 256 ? 4 : 6;
  static constexpr int kABytes = kBN * kBK * 2;
  static constexpr int kBBytes = TOK * kBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kRing = STAGES * kStageBytes;
  static constexpr int kEpi = kRing;                               // [2][kChunk][kPitch] fp32
  static constexpr int kRstd = kEpi + 2 * kChunk * kPitch * 4;     // [2][kChunk] fp32
  static constexpr int kRow = kRstd + 2 * kChunk * 4;              // [2][kChunk] int4
  static constexpr int kBar = kRow + 2 * kChunk * 16;
  static constexpr int kMisc = kBar + (2 * STAGES + 4) * 8;
  static constexpr int kTotal = kMisc + 16;
  static constexpr int kAlloc = kTotal + 1024;
  static_assert(kAlloc <= 232448, "shared memory budget");
};

// 32 values per lane -> lane l holds the reduction over the warp's lanes of
// value l (recursive halving: 16 + 8 + 4 + 2 + 1 shuffles).  Sum or max.
template <bool kSum>
__device__ __forceinline__ void butterfly_reduce(float (&v)[32], int lane) {
#pragma unroll
  for (int w = 16; w >= 1; w >>= 1) {
    const bool upper = (lane & w) != 0;
#pragma unroll
    for (int i = 0; i < w; ++i) {
      const float send = upper ? v[i] : v[i + w];
      const float keep = upper ? v[i + w] : v[i];
      const float got = __shfl_xor_sync(0xffffffffu, send, w);
      v[i] = kSum ? keep + got : fmaxf(keep, got);
    }
  }
}

// The direct SwiGLU epilogue stores 16-byte vectors: whole 128-column tiles,
// 16-byte aligned rows.
__device__ __forceinline__ bool direct_swiglu_ok(const EpiParams& epi, int N) {
  return N % 128 == 0 && (epi.ld_bf16 & 7) == 0 && (reinterpret_cast<uintptr_t>(epi.out_bf16) & 15) == 0 &&
         (reinterpret_cast<uintptr_t>(epi.out2_bf16) & 15) == 0;
}

// debug timeline (epi.stamps, [ctas x 8] %globaltimer): 0 start, 1 setup done,
// 2 first TMA issued, 3 first k-block landed, 4 last MMA committed,
// 5 first accumulator ready (epilogue), 6 epilogue done (group 0), 7 exit
__device__ __forceinline__ void big_stamp(const EpiParams& epi, int i) {
  if (epi.stamps != nullptr) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    epi.stamps[(size_t)blockIdx.x * 8 + i] = t;
  }
}

__device__ __forceinline__ uint32_t bf2_bits(float lo, float hi) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&h);
}

__device__ __forceinline__ void group_sync(int g) {
  asm volatile("bar.sync %0, 128;" ::"r"(1 + g) : "memory");
}

// AMN / BMN: the W / X operand is MN-major (given as [K x N] / [K x M]
// row-major, e.g. the trainer's dW = dY^T X with the token axis as K, or
// dX = dY W with W's rows as K): 64 x 64 TMA boxes, UMMA descriptors with
// the 64-element MN groups 8 KB apart.  `splits` > 1 cuts K into
// ordered slices whose EPI_ACCUM epilogues add into the output one after the
// other (per-tile counters in epi.tile_flags, self-resetting): deterministic
// split-K for the small-output, long-K weight gradients.
template <int TOK, bool AMN, bool BMN, int EK>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_big_kernel(const __grid_constant__ CUtensorMap tw, const __grid_constant__ CUtensorMap tx,
                    int M, int N, int K, int splits, const EpiParams epi) {
  using L = BigLayout<TOK>;
  const int kind = gemm_detail::epi_kind<EK>(epi);
  constexpr int STAGES = L::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kBar);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::kMisc);

  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) big_stamp(epi, 0);
  const int n_tiles = (N + kBN - 1) / kBN;
  const int tok_tiles = (M + TOK - 1) / TOK;
  const int tiles = n_tiles * tok_tiles;
  const int total = tiles * splits;
  const int kbt = K / kBK;

  if (warp == 0) {
    if (elect_one()) {
      tma_prefetch_desc(&tw);
      tma_prefetch_desc(&tx);
    }
    __syncwarp();
    tmem_alloc<2 * TOK>(tmem_slot);
  } else if (warp == 1) {
    if (elect_one()) {
      for (int s = 0; s < STAGES; ++s) {
        mbar_init(&full[s], 1);
        mbar_init(&empty[s], 1);
      }
      for (int a = 0; a < 2; ++a) {
        mbar_init(&tfull[a], 1);
        mbar_init(&tempty[a], 256);  // every epilogue thread, after its last TMEM load
      }
      fence_barrier_init();
    }
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  griddep_launch_dependents();
  if (threadIdx.x == 0) big_stamp(epi, 1);

  if (warp == 0) {
    if (elect_one()) {  // ---- TMA producer
      griddep_wait();   // the activations come from the previous kernel
      int stage = 0;
      uint32_t ph = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        const int tile = t % tiles, sp = t / tiles;
        const int n0 = (tile % n_tiles) * kBN, t0 = (tile / n_tiles) * TOK;
        for (int kb = sp * kbt / splits; kb < (sp + 1) * kbt / splits; ++kb) {
          mbar_wait(&empty[stage], ph ^ 1);
          uint8_t* a = smem + stage * L::kStageBytes;
          mbar_arrive_expect_tx(&full[stage], L::kStageBytes);
          if (kb == 0 && t == (int)blockIdx.x) big_stamp(epi, 2);
          // split operands: segment sg of the K concatenation (see EpiParams)
          int kl = kb, xo = 0, wo = 0;
          if (epi.seg_kb > 0) {
            const int sg = kb / epi.seg_kb;
            kl = kb - sg * epi.seg_kb;
            xo = sg == 0 ? epi.x_off0 : sg == 1 ? epi.x_off1 : epi.x_off2;
            wo = sg == 0 ? epi.w_off0 : sg == 1 ? epi.w_off1 : epi.w_off2;
          }
          if constexpr (AMN) {  // 64 x 64 boxes: [k rows][64 MN columns], 8 KB each
            tma_load_2d(a, &tw, &full[stage], n0 + wo, kl * kBK);
            tma_load_2d(a + 8192, &tw, &full[stage], n0 + 64 + wo, kl * kBK);
          } else {
            tma_load_2d(a, &tw, &full[stage], kl * kBK + wo, n0);
          }
          if constexpr (BMN) {
#pragma unroll
            for (int h = 0; h < TOK / 64; ++h)
              tma_load_2d(a + L::kABytes + h * 8192, &tx, &full[stage], t0 + h * 64 + xo, kl * kBK);
          } else {
#pragma unroll
            for (int h = 0; h < TOK / 128; ++h)  // the X map's box is 128 rows
              tma_load_2d(a + L::kABytes + h * 128 * 128, &tx, &full[stage], kl * kBK + xo, t0 + h * 128);
          }
          if (++stage == STAGES) { stage = 0; ph ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (elect_one()) {  // ---- MMA issuer
      constexpr uint32_t idesc = idesc_bf16_f32(128, TOK) | (AMN ? idesc_a_mn_major : 0u) |
                                 (BMN ? idesc_b_mn_major : 0u);
      int stage = 0, acc = 0;
      uint32_t ph = 0, aph = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        mbar_wait(&tempty[acc], aph ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * TOK;
        const int sp = t / tiles, kb0 = sp * kbt / splits;
        for (int kb = kb0; kb < (sp + 1) * kbt / splits; ++kb) {
          mbar_wait(&full[stage], ph);
          tc_fence_after();
          if (kb == kb0 && t == (int)blockIdx.x) big_stamp(epi, 3);
          const uint32_t a = smem_u32(smem + stage * L::kStageBytes);
          const uint32_t b = a + L::kABytes;
#pragma unroll
          for (int kk = 0; kk < kBK / 16; ++kk) {
            // MN-major: 16 k rows = two 1-KB swizzle atoms; K-major: 32 B inside the atom
            const uint64_t da = AMN ? umma_desc_mn_sw128(a + kk * 2048, 8192) : umma_desc_k_sw128(a, kk * 32);
            const uint64_t db = BMN ? umma_desc_mn_sw128(b + kk * 2048, 8192) : umma_desc_k_sw128(b, kk * 32);
            mma_bf16_ss(d, da, db, idesc, (kb != kb0) || kk != 0);
          }
          mma_commit(&empty[stage]);
          if (++stage == STAGES) { stage = 0; ph ^= 1; }
        }
        mma_commit(&tfull[acc]);
        big_stamp(epi, 4);
        if (++acc == 2) { acc = 0; aph ^= 1; }
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ---- epilogue: group g (warps 4-7 / 8-11), TMEM lane quadrant q
    const int g = (warp - 4) >> 2, q = warp & 3;
    const int tid = q * 32 + (threadIdx.x & 31);  // = the TMEM lane = the tile column drained
    float* tile = reinterpret_cast<float*>(smem + L::kEpi) + g * kChunk * kPitch;
    float* s_rstd = reinterpret_cast<float*>(smem + L::kRstd) + g * kChunk;
    int4* s_row = reinterpret_cast<int4*>(smem + L::kRow) + g * kChunk;
    auto sync = [g] { group_sync(g); };
    // statistics-only LM head (the trainer's pass 1: no logits stored)
    const bool stats_only = kind == EPI_LOGITS && epi.out_f32 == nullptr;
    const bool direct = kind == EPI_STORE_F32 || kind == EPI_STORE_BF16 ||
                        kind == EPI_ACCUM_F32 || kind == EPI_DLOGITS ||
                        kind == EPI_SWIGLU_BWD || kind == EPI_RESID ||
                        (kind == EPI_QKV && 128 % epi.hd == 0 && epi.hd % 8 == 0 && N % 8 == 0) ||
                        (kind == EPI_SWIGLU && direct_swiglu_ok(epi, N)) || stats_only;
    float* red = tile;  // stats_only: [4 warps][32 tokens] cross-warp partials (the unused staging tile)
    bool waited = false;
    int acc = 0;
    uint32_t aph = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x) {
      const int otile = t % tiles, sp = t / tiles;
      const int n_tile = otile % n_tiles, n0 = n_tile * kBN, t0 = (otile / n_tiles) * TOK;
      if (!waited) {  // epilogue inputs (residual, ssq) come from earlier kernels
        griddep_wait();
        waited = true;
      }
      // Row inputs of this group's chunks (independent of the accumulator),
      // loaded while the tile's MMAs run: lane l holds token (chunk row) l's
      // deferred-RMSNorm rstd and (EPI_QKV) slot / position / page / offset.
      constexpr int kCpg = TOK / (2 * kChunk);  // chunks per group
      float pre_rs[kCpg];
      int2 pre_rc[kCpg];  // (position or -1, page)
      if (direct) {
        const int lane = threadIdx.x & 31;
        float ssum[kCpg];
#pragma unroll
        for (int ci = 0; ci < kCpg; ++ci) {
          const int m = t0 + (g + 2 * ci) * kChunk + lane;
          ssum[ci] = -1.f;
          pre_rc[ci] = make_int2(-1, -1);  // .y = slot until the page is known
          if (m < M) {
            if (epi.ssq_in != nullptr)
              ssum[ci] = gemm_detail::ssq_row_sum(epi.ssq_in + (size_t)m * epi.ssq_in_parts, epi.ssq_in_parts);
            if (kind == EPI_QKV) {
              pre_rc[ci].y = epi.row_slot[m];
              pre_rc[ci].x = epi.row_pos[m];
            }
          }
        }
#pragma unroll
        for (int ci = 0; ci < kCpg; ++ci) {
          pre_rs[ci] = ssum[ci] >= 0.f ? rsqrtf(ssum[ci] * epi.inv_dim + epi.eps) : 1.f;
          if (pre_rc[ci].y >= 0)
            pre_rc[ci].y = epi.block_table[(size_t)pre_rc[ci].y * epi.pages_per_seq + pre_rc[ci].x / 64];
          else
            pre_rc[ci].x = -1;
        }
      }
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
      if (tid == 0 && g == 0 && t == (int)blockIdx.x) big_stamp(epi, 5);
      if (splits > 1 && sp > 0) {  // K slice sp adds after slices 0..sp-1 (both groups each)
        if (tid == 0) {
          while (ld_acquire_gpu(epi.tile_flags + otile) < 2 * sp) __nanosleep(64);
        }
        sync();
      }
      const int last = TOK / kChunk - 2 + g;  // this group's last chunk of the tile
      for (int c = g; c < TOK / kChunk; c += 2) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(tmem + acc * TOK + c * kChunk + ((uint32_t)(q * 32) << 16), r);
        tmem_ld_wait();
        if (c == last) {  // accumulator drained by this thread
          tc_fence_before();
          mbar_arrive(&tempty[acc]);
        }
        const int tc0 = t0 + c * kChunk;
        if (tc0 >= M) continue;  // rows past M: nothing to store (uniform per group)
        if (direct) {
          // plain stores straight from the accumulator registers: thread =
          // output column n, so each warp store covers 32 consecutive columns
          const int n = n0 + tid;
          const int lane = threadIdx.x & 31;
          // rstd of token tc0 + lane (prefetched), broadcast below
          const int ci = (c - g) >> 1;
          float rs = pre_rs[0];
          int2 rc = pre_rc[0];
#pragma unroll
          for (int k = 1; k < kCpg; ++k)
            if (ci == k) { rs = pre_rs[k]; rc = pre_rc[k]; }
          const float bias = (epi.bias != nullptr && n < N) ? gemm_detail::epi_bf2f(epi.bias[n]) : 0.f;
          const int jn = min(32, M - tc0);
          if (stats_only) {
            // per token: the target's logit, and over this tile's 128 columns
            // the max and the sum of exp(x - max) (fp32 exp, fp64 combine).
            // Each warp reduces its 32 columns for all 32 tokens at once with a
            // butterfly transpose (31 shuffles, lane l ends with token l), the
            // group's four warps combine through shared memory.
            int tg = -1;
            if (epi.tgt_row && tc0 + lane < M) tg = epi.tgt_row[tc0 + lane];
            float v[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const float rj = __shfl_sync(0xffffffffu, rs, j);
              const int tj = __shfl_sync(0xffffffffu, tg, j);
              v[j] = n < N && j < jn ? __uint_as_float(r[j]) * rj : -INFINITY;
              if (n == tj && j < jn) epi.tgt_out[tc0 + j] = v[j];
            }
            float mx[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) mx[j] = v[j];
            butterfly_reduce<false>(mx, lane);  // lane l: max of token l over this warp's columns
            const int q = tid >> 5;
            red[q * 32 + lane] = mx[0];
            sync();
            float M_l = red[lane];
#pragma unroll
            for (int w = 1; w < 4; ++w) M_l = fmaxf(M_l, red[w * 32 + lane]);
            float e[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const float Mj = __shfl_sync(0xffffffffu, M_l, j);
              e[j] = v[j] == -INFINITY ? 0.f : __expf(v[j] - Mj);
            }
            butterfly_reduce<true>(e, lane);  // lane l: this warp's sum for token l
            sync();  // everyone has read the maxima
            red[q * 32 + lane] = e[0];
            sync();
            if (q == 0 && lane < jn) {
              const double sum = (double)red[lane] + (double)red[32 + lane] + (double)red[64 + lane] +
                                 (double)red[96 + lane];
              epi.part_max[(size_t)(tc0 + lane) * n_tiles + n_tile] = M_l;
              epi.part_sum[(size_t)(tc0 + lane) * n_tiles + n_tile] = M_l == -INFINITY ? 0.0 : sum;
            }
            sync();  // red is reused by the next chunk
            continue;
          }
          if (kind == EPI_DLOGITS) {
            // d = coef * (onehot - softmax) of token tc0 + j at vocab column n; the
            // transposed copy [n][tokens] is 32 contiguous bf16 per thread
            float lse = 0.f, cf = 0.f;
            int tg = -1;
            if (tc0 + lane < M) {
              lse = (float)epi.lse_in[tc0 + lane];
              cf = epi.row_coef[tc0 + lane];
              tg = epi.tgt_row[tc0 + lane];
            }
            const bool vec = epi.outT_bf16 == nullptr && (epi.ld_bf16 & 7) == 0 && (N & 7) == 0 &&
                             (reinterpret_cast<uintptr_t>(epi.out_bf16) & 15) == 0 &&
                             (epi.lo_off & 7) == 0;
            // [32 tokens][128] bf16 staging, the lo halves (split output) after it
            uint16_t* st16 = reinterpret_cast<uint16_t*>(tile);
            uint32_t packed[16];
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const float rj = __shfl_sync(0xffffffffu, rs, j);
              const float lj = __shfl_sync(0xffffffffu, lse, j);
              const float cj = __shfl_sync(0xffffffffu, cf, j);
              const int tj = __shfl_sync(0xffffffffu, tg, j);
              const float x = __uint_as_float(r[j]) * rj;
              float d = j < jn ? cj * ((n == tj ? 1.f : 0.f) - __expf(x - lj)) : 0.f;
              if (epi.fold_rstd) d *= rj;
              const __nv_bfloat16 b = __float2bfloat16(d);
              const uint32_t bits = (uint32_t)__bfloat16_as_ushort(b);
              const __nv_bfloat16 bl = __float2bfloat16(d - __bfloat162float(b));
              if (vec) {
                st16[j * 128 + tid] = (uint16_t)bits;
                if (epi.lo_off) st16[4096 + j * 128 + tid] = __bfloat16_as_ushort(bl);
              } else {
                if (epi.lo_off && j < jn && n < N) epi.out_bf16[(size_t)(tc0 + j) * epi.ld_bf16 + n + epi.lo_off] = bl;
                if (j < jn && n < N) epi.out_bf16[(size_t)(tc0 + j) * epi.ld_bf16 + n] = b;
                if (j & 1) packed[j >> 1] |= bits << 16;
                else packed[j >> 1] = bits;
              }
            }
            if (vec) {  // 16-byte rows of 8 columns, 4 per thread
              sync();
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const int idx = tid + 128 * k, j = idx >> 4, c8 = (idx & 15) * 8;
                if (j < jn && n0 + c8 < N) {
                  __nv_bfloat16* dst = epi.out_bf16 + (size_t)(tc0 + j) * epi.ld_bf16 + n0 + c8;
                  *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(&st16[j * 128 + c8]);
                  if (epi.lo_off)
                    *reinterpret_cast<uint4*>(dst + epi.lo_off) =
                        *reinterpret_cast<const uint4*>(&st16[4096 + j * 128 + c8]);
                }
              }
              sync();  // the staging area is reused next
            } else if (epi.outT_bf16 && n < N) {  // columns past M are written as 0 (padding)
              uint4* dst = reinterpret_cast<uint4*>(epi.outT_bf16 + (size_t)n * epi.ldT + tc0);
#pragma unroll
              for (int v = 0; v < 4; ++v)
                dst[v] = make_uint4(packed[4 * v], packed[4 * v + 1], packed[4 * v + 2], packed[4 * v + 3]);
            }
            continue;
          }
          if (kind == EPI_RESID) {
            // resid += acc, xg = bf16(resid * gain); the 32 residual loads in
            // flight together, the per-token x^2 sum over the tile's 128 columns
            // by a butterfly transpose (lane l: token l) + the group's 4 warps
            const bool colok = n < N;
            const float gain = colok ? gemm_detail::epi_bf2f(epi.gain[n]) : 0.f;
            float xr[32];
#pragma unroll
            for (int j = 0; j < 32; ++j)
              xr[j] = (colok && j < jn) ? epi.resid[(size_t)(tc0 + j) * N + n] : 0.f;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              float x = 0.f;
              if (colok && j < jn) {
                const size_t o = (size_t)(tc0 + j) * N + n;
                x = xr[j] + __uint_as_float(r[j]);
                epi.resid[o] = x;
                const float xgv = x * gain;
                const __nv_bfloat16 hi = __float2bfloat16(xgv);
                if (epi.lo_off == 0) {
                  epi.xg[o] = hi;
                } else {  // split: row stride N + lo_off, lo = the rounding residual
                  const size_t os = (size_t)(tc0 + j) * (N + epi.lo_off) + n;
                  epi.xg[os] = hi;
                  epi.xg[os + epi.lo_off] = __float2bfloat16(xgv - __bfloat162float(hi));
                }
              }
              xr[j] = x * x;
            }
            butterfly_reduce<true>(xr, lane);
            const int q = tid >> 5;
            red[q * 32 + lane] = xr[0];
            sync();
            if (q == 0 && lane < jn)
              epi.ssq_out[(size_t)(tc0 + lane) * n_tiles + n_tile] =
                  ((red[lane] + red[32 + lane]) + red[64 + lane]) + red[96 + lane];
            sync();  // red is reused by the next chunk
            continue;
          }
          if (kind == EPI_QKV) {
            // v = rstd acc + bias staged (RoPE pairs live in other warps) with
            // each token's (position, page); then thread-steps of 8 consecutive
            // columns of one token: cos / sin as two float4 each, one 16-byte
            // store into q or the K / V page
            const bool colok = n < N;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const float rj = __shfl_sync(0xffffffffu, rs, j);
              tile[j * kPitch + tid] = (colok && j < jn) ? __uint_as_float(r[j]) * rj + bias : 0.f;
            }
            if (tid < 32) s_row[tid] = make_int4(rc.x, rc.y, 0, 0);
            sync();
            const int hd = epi.hd, half = hd >> 1;
            const int qend = epi.nq * hd, kend = (epi.nq + epi.nkv) * hd;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const int idx = tid + 128 * k, j = idx >> 4, c8 = (idx & 15) * 8, nn = n0 + c8;
              if (j >= jn || nn >= N) continue;
              const int4 rr = s_row[j];
              const int ps = rr.x;
              if (ps < 0) continue;  // free slot / padding row
              const int jj = nn % hd, hb = c8 - jj;
              const float* row = &tile[j * kPitch + hb];
              float y[8];
              if (nn < kend) {  // RoPE on q and k: pairs (i, i + hd/2)
                const int i0 = jj < half ? jj : jj - half;
                const float4* cs = reinterpret_cast<const float4*>(epi.cos_sin + (size_t)ps * hd);
                float co[8], si[8];
                *reinterpret_cast<float4*>(&co[0]) = cs[i0 / 4];
                *reinterpret_cast<float4*>(&co[4]) = cs[i0 / 4 + 1];
                *reinterpret_cast<float4*>(&si[0]) = cs[(half + i0) / 4];
                *reinterpret_cast<float4*>(&si[4]) = cs[(half + i0) / 4 + 1];
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                  const float x1 = row[i0 + e], x2 = row[i0 + e + half];
                  y[e] = jj < half ? x1 * co[e] - x2 * si[e] : x2 * co[e] + x1 * si[e];
                }
              } else {
#pragma unroll
                for (int e = 0; e < 8; ++e) y[e] = row[jj + e];
              }
              uint4 o;
              o.x = bf2_bits(y[0], y[1]); o.y = bf2_bits(y[2], y[3]);
              o.z = bf2_bits(y[4], y[5]); o.w = bf2_bits(y[6], y[7]);
              __nv_bfloat16* dst;
              if (nn < qend) {
                dst = epi.q_out + (size_t)(tc0 + j) * qend + nn;
              } else {
                const int kv = nn < kend ? nn - qend : nn - kend;
                const size_t at = (((size_t)rr.y * epi.nkv + kv / hd) * 64 + ps % 64) * hd + jj;
                dst = (nn < kend ? epi.kc : epi.vc) + at;
              }
              *reinterpret_cast<uint4*>(dst) = o;
            }
            sync();  // the staged chunk and s_row are reused next
            continue;
          }
          if (kind == EPI_SWIGLU) {
            // tile = 64 gate | 64 up columns: the rstd-scaled values go to the
            // gate|up copy straight from registers (this thread's column, 32
            // tokens: contiguous in the gu_index layout) and are staged for
            // act = silu(g) u (16-byte stores of 8 act columns x 1 token)
            float v[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const float rj = __shfl_sync(0xffffffffu, rs, j);
              v[j] = __uint_as_float(r[j]) * rj;
              tile[j * kPitch + tid] = v[j];
            }
            if (epi.out2_f32 && n < N) {  // fp32 gate | up copy (precise backward); token quad k is 128
              float* dst = epi.out2_f32 + gu_index_f32(tc0, n, N);  // floats after quad k - 1
#pragma unroll
              for (int k = 0; k < 8; ++k)
                *reinterpret_cast<float4*>(dst + 128 * k) = make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
            }
            if (epi.out2_bf16 && n < N) {  // token octet k is 256 bf16 after octet k - 1
              __nv_bfloat16* dst = epi.out2_bf16 + gu_index(tc0, n, N);
#pragma unroll
              for (int k = 0; k < 4; ++k)
                *reinterpret_cast<uint4*>(dst + 256 * k) =
                    make_uint4(bf2_bits(v[8 * k], v[8 * k + 1]), bf2_bits(v[8 * k + 2], v[8 * k + 3]),
                               bf2_bits(v[8 * k + 4], v[8 * k + 5]), bf2_bits(v[8 * k + 6], v[8 * k + 7]));
            }
            sync();
#pragma unroll
            for (int k = 0; k < 2; ++k) {
              const int idx = tid + 128 * k, j = idx >> 3, c8 = (idx & 7) * 8;
              if (j >= jn) continue;
              float g[8], u[8];
              *reinterpret_cast<float4*>(&g[0]) = *reinterpret_cast<const float4*>(&tile[j * kPitch + c8]);
              *reinterpret_cast<float4*>(&g[4]) = *reinterpret_cast<const float4*>(&tile[j * kPitch + c8 + 4]);
              *reinterpret_cast<float4*>(&u[0]) = *reinterpret_cast<const float4*>(&tile[j * kPitch + 64 + c8]);
              *reinterpret_cast<float4*>(&u[4]) = *reinterpret_cast<const float4*>(&tile[j * kPitch + 64 + c8 + 4]);
              float a[8];
              // split output (precise mode, ~2^-17): the SFU sigmoid (ex2 + rcp, ~2 ulp)
              // is far below the pair's resolution; a single bf16 act keeps the IEEE
              // sigmoid so its rounding decisions track the fp64 oracle's (the
              // trainer's fast-mode log-probs sit at that bf16 floor)
              if (epi.lo_off) {
#pragma unroll
                for (int e = 0; e < 8; ++e) a[e] = __fdividef(g[e], 1.f + __expf(-g[e])) * u[e];
              } else {
#pragma unroll
                for (int e = 0; e < 8; ++e) a[e] = g[e] / (1.f + expf(-g[e])) * u[e];
              }
              uint4 o;
              o.x = bf2_bits(a[0], a[1]); o.y = bf2_bits(a[2], a[3]);
              o.z = bf2_bits(a[4], a[5]); o.w = bf2_bits(a[6], a[7]);
              __nv_bfloat16* dst = epi.out_bf16 + (size_t)(tc0 + j) * epi.ld_bf16 + (n0 >> 1) + c8;
              *reinterpret_cast<uint4*>(dst) = o;
              if (epi.lo_off) {
                const uint32_t hw[4] = {o.x, o.y, o.z, o.w};
                float lo[8];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  lo[2 * e] = a[2 * e] - __uint_as_float(hw[e] << 16);
                  lo[2 * e + 1] = a[2 * e + 1] - __uint_as_float(hw[e] & 0xffff0000u);
                }
                uint4 ol;
                ol.x = bf2_bits(lo[0], lo[1]); ol.y = bf2_bits(lo[2], lo[3]);
                ol.z = bf2_bits(lo[4], lo[5]); ol.w = bf2_bits(lo[6], lo[7]);
                *reinterpret_cast<uint4*>(dst + epi.lo_off) = ol;
              }
            }
            sync();  // the staged chunk is reused next
            continue;
          }
          if (kind == EPI_SWIGLU_BWD) {
            // column n = act index of 64-block b: gate at 128 b + (n & 63), up 64
            // after; the tile's 256 dgu columns of a token are contiguous
            // (2 n0 ..), staged as bf16 and written as 16-byte rows
            const int lc = (tid >> 6) * 128 + (tid & 63);  // tile-local gate column
            uint16_t* st16 = reinterpret_cast<uint16_t*>(tile);  // [32][256]
            const size_t gcol = (size_t)2 * n0 + lc;
            // this thread's gate and up columns for the chunk's 32 tokens: 2 x 32
            // contiguous values (gu_index layout), all in flight together
            float gf[32], uf[32];
            if (epi.gu_in_f32) {  // precise: fp32 gate | up (token quad k: + 128 k floats)
              const float* g4 = epi.gu_in_f32 + gu_index_f32(tc0, gcol, 2 * (size_t)N);
              const float* u4 = epi.gu_in_f32 + gu_index_f32(tc0, gcol + 64, 2 * (size_t)N);
              float4 gv4[8], uv4[8];
#pragma unroll
              for (int k = 0; k < 8; ++k) {
                gv4[k] = n < N ? __ldg(reinterpret_cast<const float4*>(g4 + 128 * k)) : make_float4(0.f, 0.f, 0.f, 0.f);
                uv4[k] = n < N ? __ldg(reinterpret_cast<const float4*>(u4 + 128 * k)) : make_float4(0.f, 0.f, 0.f, 0.f);
              }
#pragma unroll
              for (int k = 0; k < 8; ++k) {
                gf[4 * k] = gv4[k].x; gf[4 * k + 1] = gv4[k].y; gf[4 * k + 2] = gv4[k].z; gf[4 * k + 3] = gv4[k].w;
                uf[4 * k] = uv4[k].x; uf[4 * k + 1] = uv4[k].y; uf[4 * k + 2] = uv4[k].z; uf[4 * k + 3] = uv4[k].w;
              }
            } else {  // token octet k: + 256 k bf16
              const __nv_bfloat16* g8 = epi.gu_in + gu_index(tc0, gcol, 2 * (size_t)N);
              const __nv_bfloat16* u8 = epi.gu_in + gu_index(tc0, gcol + 64, 2 * (size_t)N);
              uint4 gv8[4], uv8[4];
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                gv8[k] = n < N ? __ldg(reinterpret_cast<const uint4*>(g8 + 256 * k)) : make_uint4(0u, 0u, 0u, 0u);
                uv8[k] = n < N ? __ldg(reinterpret_cast<const uint4*>(u8 + 256 * k)) : make_uint4(0u, 0u, 0u, 0u);
              }
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const uint32_t gw[4] = {gv8[k].x, gv8[k].y, gv8[k].z, gv8[k].w};
                const uint32_t uw[4] = {uv8[k].x, uv8[k].y, uv8[k].z, uv8[k].w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  gf[8 * k + 2 * e] = __uint_as_float(gw[e] << 16);
                  gf[8 * k + 2 * e + 1] = __uint_as_float(gw[e] & 0xffff0000u);
                  uf[8 * k + 2 * e] = __uint_as_float(uw[e] << 16);
                  uf[8 * k + 2 * e + 1] = __uint_as_float(uw[e] & 0xffff0000u);
                }
              }
            }
            float rsc = 1.f;
            if (epi.row_scale != nullptr && tc0 + lane < M) rsc = epi.row_scale[tc0 + lane];
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const float gv = gf[j], uv = uf[j];
              const float da = __uint_as_float(r[j]) * __shfl_sync(0xffffffffu, rsc, j);
              // sigmoid by the SFU (ex2 + rcp, ~2 ulp): the IEEE expf / divide sequences
              // made this epilogue instruction-bound
              const float sg = __fdividef(1.f, 1.f + __expf(-gv));
              const float silu = gv * sg;
              gf[j] = da * uv * (sg * (1.f + gv * (1.f - sg)));  // d gate
              uf[j] = da * silu;                                  // d up
            }
            // hi halves, then (split output) the lo halves through the same staging
            for (int part = 0; part < (epi.lo_off ? 2 : 1); ++part) {
#pragma unroll
              for (int j = 0; j < 32; ++j) {
                __nv_bfloat16 hg = __float2bfloat16(gf[j]), hu = __float2bfloat16(uf[j]);
                if (part) {
                  hg = __float2bfloat16(gf[j] - __bfloat162float(hg));
                  hu = __float2bfloat16(uf[j] - __bfloat162float(hu));
                }
                st16[j * 256 + lc] = __bfloat16_as_ushort(hg);
                st16[j * 256 + lc + 64] = __bfloat16_as_ushort(hu);
              }
              sync();
              const int off = part ? epi.lo_off : 0;
#pragma unroll
              for (int k = 0; k < 8; ++k) {
                const int idx = tid + 128 * k, j = idx >> 5, c8 = (idx & 31) * 8;
                if (j < jn && n0 + (c8 >> 1) < N)
                  *reinterpret_cast<uint4*>(epi.out_bf16 + (size_t)(tc0 + j) * epi.ld_bf16 + 2 * n0 + c8 + off) =
                      *reinterpret_cast<const uint4*>(&st16[j * 256 + c8]);
              }
              sync();  // the staging area is reused next
            }
            continue;
          }
          {
            // store / accumulate through a staged fp32 chunk: 16-byte rows, the
            // accumulate's loads all in flight before its stores
            const bool bf = kind == EPI_STORE_BF16;
            const int ld = bf ? epi.ld_bf16 : epi.ld_out;
            const void* base = bf ? static_cast<const void*>(epi.out_bf16) : static_cast<const void*>(epi.out_f32);
            const bool vec = (N & 7) == 0 && (ld & 7) == 0 && (reinterpret_cast<uintptr_t>(base) & 15) == 0;
            if (vec) {
              const bool acc_kind = kind == EPI_ACCUM_F32;
#pragma unroll
              for (int j = 0; j < 32; ++j) {
                const float rj = __shfl_sync(0xffffffffu, rs, j);
                const float v = __uint_as_float(r[j]);
                tile[j * kPitch + tid] = acc_kind ? epi.scale * v : v * rj + bias;
              }
              sync();
              if (bf) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                  const int idx = tid + 128 * k, j = idx >> 4, c8 = (idx & 15) * 8;
                  if (j >= jn || n0 + c8 >= N) continue;
                  const float4 x0 = *reinterpret_cast<const float4*>(&tile[j * kPitch + c8]);
                  const float4 x1 = *reinterpret_cast<const float4*>(&tile[j * kPitch + c8 + 4]);
                  uint4 o;
                  o.x = bf2_bits(x0.x, x0.y); o.y = bf2_bits(x0.z, x0.w);
                  o.z = bf2_bits(x1.x, x1.y); o.w = bf2_bits(x1.z, x1.w);
                  *reinterpret_cast<uint4*>(epi.out_bf16 + (size_t)(tc0 + j) * ld + n0 + c8) = o;
                }
              } else {
                float4 cur[8];
                if (acc_kind) {
#pragma unroll
                  for (int k = 0; k < 8; ++k) {
                    const int idx = tid + 128 * k, j = idx >> 5, c4 = (idx & 31) * 4;
                    cur[k] = (j < jn && n0 + c4 < N)
                                 ? *reinterpret_cast<const float4*>(epi.out_f32 + (size_t)(tc0 + j) * ld + n0 + c4)
                                 : make_float4(0.f, 0.f, 0.f, 0.f);
                  }
                }
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                  const int idx = tid + 128 * k, j = idx >> 5, c4 = (idx & 31) * 4;
                  if (j >= jn || n0 + c4 >= N) continue;
                  float4 v = *reinterpret_cast<const float4*>(&tile[j * kPitch + c4]);
                  if (acc_kind) {
                    v.x += cur[k].x; v.y += cur[k].y; v.z += cur[k].z; v.w += cur[k].w;
                  }
                  *reinterpret_cast<float4*>(epi.out_f32 + (size_t)(tc0 + j) * ld + n0 + c4) = v;
                }
              }
              sync();  // the staged chunk is reused next
              continue;
            }
          }
          if (n < N) {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const float rj = __shfl_sync(0xffffffffu, rs, j);
              if (j >= jn) continue;
              const float v = __uint_as_float(r[j]);
              const size_t m = (size_t)(tc0 + j);
              if (kind == EPI_STORE_F32) epi.out_f32[m * epi.ld_out + n] = v * rj + bias;
              else if (kind == EPI_STORE_BF16) epi.out_bf16[m * epi.ld_bf16 + n] = __float2bfloat16(v * rj + bias);
              else epi.out_f32[m * epi.ld_out + n] += epi.scale * v;
            }
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) (void)__shfl_sync(0xffffffffu, rs, j);
          }
          continue;
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) tile[j * kPitch + tid] = __uint_as_float(r[j]);
        gemm_detail::epi_row_meta<EK>(epi, 0, kChunk, tc0, M, s_rstd, s_row, tid, 128);
        sync();
        gemm_detail::epi_apply<EK>(epi, tile, kPitch, 0, kChunk, tc0, n0, n_tile, n_tiles, M, N, s_rstd,
                               s_row, tid, 128, sync);
        sync();  // the staged chunk is reused next
      }
      if (splits > 1) {
        __threadfence();
        sync();
        if (tid == 0 && atomicAdd(epi.tile_flags + otile, 1) == 2 * splits - 1)
          atomicExch(epi.tile_flags + otile, 0);  // last slice: reset for the next launch
      }
      if (++acc == 2) { acc = 0; aph ^= 1; }
    }
  }
  if (warp == 4 && (threadIdx.x & 31) == 0) big_stamp(epi, 6);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_free<2 * TOK>(tmem);
  if (threadIdx.x == 0) big_stamp(epi, 7);
}

inline int num_sms_cached() {
  static int n = [] {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

template <int TOK, bool AMN, bool BMN, int EK>
cudaError_t launch_big(const CUtensorMap& tw, const CUtensorMap& tx, int M, int N, int K, int splits,
                       const EpiParams& epi, cudaStream_t stream) {
  using L = BigLayout<TOK>;
  static const cudaError_t attr = cudaFuncSetAttribute(
      gemm_big_kernel<TOK, AMN, BMN, EK>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kAlloc);
  if (attr != cudaSuccess) return attr;
  const int tiles = ((N + kBN - 1) / kBN) * ((M + TOK - 1) / TOK) * splits;
  const int grid = tiles < num_sms_cached() ? tiles : num_sms_cached();
  return launch_pdl(gemm_big_kernel<TOK, AMN, BMN, EK>, dim3(grid), dim3(kThreads), (size_t)L::kAlloc, stream,
                    dim3(1, 1, 1), tw, tx, M, N, K, splits, epi);
}


// Explicit instantiations live in gemm_big_i*.cu (parallel compilation).
#define SRL_BIG_LAUNCH_ARGS                                                                  \
  const CUtensorMap&, const CUtensorMap&, int, int, int, int, const EpiParams&, cudaStream_t
#define SRL_BIG_EXTERN(TOK, AMN, BMN, EK) \
  extern template cudaError_t launch_big<TOK, AMN, BMN, EK>(SRL_BIG_LAUNCH_ARGS);
#define SRL_BIG_INSTANTIATE(TOK, AMN, BMN, EK) \
  template cudaError_t launch_big<TOK, AMN, BMN, EK>(SRL_BIG_LAUNCH_ARGS);
#define SRL_BIG_ALL(X)                                                                      \
  X(256, false, false, 0) X(256, false, false, 1) X(256, false, false, 2) X(256, false, false, 3) \
  X(256, false, false, 4) X(256, false, false, 5) X(256, false, false, 6) X(256, false, false, 7) \
  X(128, false, false, 0) X(128, false, false, 1) X(128, false, false, 2) X(128, false, false, 3) \
  X(128, false, false, 4) X(128, false, false, 5) X(128, false, false, 6) X(128, false, false, 7) \
  X(256, true, true, 0) X(256, true, true, 6) X(128, true, true, 0) X(128, true, true, 6)        \
  X(256, true, false, 0) X(256, true, false, 6) X(256, true, false, 8)                          \
  X(128, true, false, 0) X(128, true, false, 6) X(128, true, false, 8)
SRL_BIG_ALL(SRL_BIG_EXTERN)

}  // namespace bigk
}  // namespace srl
