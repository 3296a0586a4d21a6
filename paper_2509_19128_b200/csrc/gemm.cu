// gemm.cu -- warp-specialised tcgen05 GEMM for sm_100a with fused epilogues.
//
// One CTA = 4 warps computes a [128 weight rows x TOK tokens] fp32 tile in
// TMEM.  warp0/elected lane streams W and X k-blocks with TMA into a STAGES-
// deep 128B-swizzled ring; warp1/elected lane issues tcgen05.mma (UMMA
// 128 x TOK x 16) and releases ring slots with tcgen05.commit; afterwards all
// four warps drain TMEM (tcgen05.ld 32x32b) into a shared tile and run the
// epilogue.
//
// Skinny (decode) GEMMs split K across a thread-block cluster of CS CTAs:
// every CTA stages its fp32 partial tile in its own shared memory, and after a
// cluster barrier CTA r reduces rows [r*TOK/CS, (r+1)*TOK/CS) by reading the
// CS partials through distributed shared memory in rank order -- so the
// result is bit-reproducible and no partial ever touches L2/HBM -- then runs
// the epilogue for those rows.
//
// Programmatic dependent launch: the weights do not depend on the previous
// kernel, so the producer issues the first STAGES weight tiles before
// griddepcontrol.wait; only the activation tiles and the epilogue inputs wait.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "gemm.cuh"
#include "gemm_epi.cuh"
#include "sm100.cuh"

namespace srl {
using namespace sm100;

namespace {

constexpr int kBlockN = 128;  // weight rows per tile (UMMA M)
constexpr int kBlockK = 64;   // bf16 elements per 128-B swizzle row
constexpr int kThreads = 128;
constexpr int kMaxCluster = 8;

// NB weight tiles of kBlockN rows per CTA share each X (token) stage: the
// token operand is read from L2 once per NB x 128 weight rows (decode GEMMs of
// 256 rows are L2-throughput bound on the X re-reads otherwise).
template <int TOK, int STAGES, int NB = 1>
struct Layout {
  static constexpr int kABytes = NB * kBlockN * kBlockK * 2;
  static constexpr int kBBytes = TOK * kBlockK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kPitch = kBlockN + 4;  // floats; rows stay 16-B aligned
  static constexpr int kEpiBytes = TOK * kPitch * 4;
  static constexpr int kMainBytes =
      STAGES * kStageBytes > kEpiBytes ? STAGES * kStageBytes : kEpiBytes;
  static constexpr int kBarOffset = kMainBytes;
  static constexpr int kMiscOffset = (kBarOffset + (2 * STAGES + 1) * 8 + 15) / 16 * 16;
  static constexpr int kRstdOffset = kMiscOffset + 16;
  static constexpr int kRowOffset = kRstdOffset + TOK * 4;   // per-row slot / pos / page / offset
  static_assert(kRowOffset % 16 == 0, "int4 row metadata must be 16-B aligned");
  static constexpr int kTotal = kRowOffset + TOK * 16;
  static constexpr int kAlloc = kTotal + 1024;  // manual 1024-B alignment slack
};


__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define SRL_STAMP(i)                                                                        \
  do {                                                                                      \
    if (epi.stamps != nullptr && threadIdx.x == 0)                                          \
      epi.stamps[((size_t)blockIdx.z * gridDim.y * gridDim.x + (size_t)blockIdx.y * gridDim.x + \
                  blockIdx.x) * 8 + (i)] = gtimer();                                          \
  } while (0)


template <int TOK, int STAGES, int EK, int NB = 1>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_bf16_kernel(const __grid_constant__ CUtensorMap tw, const __grid_constant__ CUtensorMap tx,
                     int M, int N, int K, int cs, float* __restrict__ ws, const EpiParams epi) {
  using L = Layout<TOK, STAGES, NB>;
  constexpr int XB = TOK > 128 ? TOK / 128 : 1;  // X boxes of <= 128 rows per stage
  constexpr int XBOX = TOK / XB;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kBarOffset);
  uint64_t* empty = full + STAGES;
  uint64_t* done = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::kMiscOffset);
  float* s_rstd = reinterpret_cast<float*>(smem + L::kRstdOffset);
  int4* s_row = reinterpret_cast<int4*>(smem + L::kRowOffset);
  float* tile = reinterpret_cast<float*>(smem);  // epilogue view, aliases the ring

  const int warp = threadIdx.x >> 5;
  const int split = blockIdx.y, tok_tile = blockIdx.z;
  const int n_tiles = (N + kBlockN - 1) / kBlockN;  // 128-row tiles (epilogue / partial index)
  const int n0 = blockIdx.x * NB * kBlockN, t0 = tok_tile * TOK;
  const int kb_total = K / kBlockK;
  const int kb_begin = (split * kb_total) / cs;
  const int nkb = ((split + 1) * kb_total) / cs - kb_begin;  // >= 1 (host: cs <= kb_total)
  SRL_STAMP(0);

  if (warp == 0) {
    if (elect_one()) {
      tma_prefetch_desc(&tw);
      tma_prefetch_desc(&tx);
    }
    __syncwarp();
    tmem_alloc<NB * TOK>(tmem_slot);
  } else if (warp == 1) {
    if (elect_one()) {
      for (int s = 0; s < STAGES; ++s) {
        mbar_init(&full[s], 1);
        mbar_init(&empty[s], 1);
      }
      mbar_init(done, 1);
      fence_barrier_init();
    }
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  griddep_launch_dependents();  // the next kernel may start its prologue now
  SRL_STAMP(1);

  if (warp == 0) {
    if (elect_one()) {  // ---- TMA producer
      const uint64_t w_policy = policy_evict_first();
      const int pre = nkb < STAGES ? nkb : STAGES;
      auto load_w = [&](int s, int kc) {
#pragma unroll
        for (int h = 0; h < NB; ++h)
          tma_load_2d_hint(smem + s * L::kStageBytes + h * (kBlockN * kBlockK * 2), &tw, &full[s], kc,
                           n0 + h * kBlockN, w_policy);
      };
      auto load_x = [&](int s, int kc) {
#pragma unroll
        for (int b = 0; b < XB; ++b)
          tma_load_2d(smem + s * L::kStageBytes + L::kABytes + b * (XBOX * kBlockK * 2), &tx, &full[s], kc,
                      t0 + b * XBOX);
      };
      for (int i = 0; i < pre; ++i) {  // weights first: independent of the previous kernel
        mbar_arrive_expect_tx(&full[i], L::kStageBytes);
        load_w(i, (kb_begin + i) * kBlockK);
      }
      griddep_wait();  // activations are produced by the previous kernel
      for (int i = 0; i < pre; ++i) load_x(i, (kb_begin + i) * kBlockK);
      for (int i = pre; i < nkb; ++i) {
        const int s = i % STAGES;
        const uint32_t ph = (i / STAGES) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&full[s], L::kStageBytes);
        const int kc = (kb_begin + i) * kBlockK;
        load_w(s, kc);
        load_x(s, kc);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (elect_one()) {  // ---- MMA issuer
      constexpr uint32_t idesc = idesc_bf16_f32(128, TOK);
      for (int i = 0; i < nkb; ++i) {
        const int s = i % STAGES;
        const uint32_t ph = (i / STAGES) & 1;
        mbar_wait(&full[s], ph);
        tc_fence_after();
        const uint32_t a = smem_u32(smem + s * L::kStageBytes);
        const uint32_t b = a + L::kABytes;
#pragma unroll
        for (int h = 0; h < NB; ++h)
#pragma unroll
          for (int kk = 0; kk < kBlockK / 16; ++kk)
            mma_bf16_ss(tmem + h * TOK, umma_desc_k_sw128(a + h * (kBlockN * kBlockK * 2), kk * 32),
                        umma_desc_k_sw128(b, kk * 32), idesc, (i | kk) != 0);
        mma_commit(&empty[s]);
      }
      mma_commit(done);
    }
    __syncwarp();
  }

  // ---- drain TMEM: thread = weight row (TMEM lane), columns = tokens; one
  // 128-row tile (accumulator half h of NB) at a time.  cs == 1: into the
  // shared tile, then its epilogue.  cs > 1: into this split's fp32 partial in
  // global memory (coalesced across rows), exchanged through L2 -- the DSMEM
  // port (~20 B/clk/SM) is slower than L2 for whole-tile partials.
  mbar_wait(done, 0);
  tc_fence_after();
  const int row = threadIdx.x;
  const size_t tiles_total = (size_t)n_tiles * gridDim.z;
  const int nh = NB == 1 ? 1 : min(NB, n_tiles - (int)blockIdx.x * NB);  // halves inside N
  auto tile_id = [&](int h) { return (size_t)tok_tile * n_tiles + blockIdx.x * NB + h; };
  auto drain = [&](int h) {
    const uint32_t lane_addr = tmem + h * TOK + ((uint32_t)(warp * 32) << 16);
    float* part = cs > 1 ? ws + ((size_t)split * tiles_total + tile_id(h)) * (TOK * kBlockN) : nullptr;
#pragma unroll
    for (int c0 = 0; c0 < TOK; c0 += 64) {  // two 32-column loads in flight, one wait
      uint32_t ra[32], rb[32];
      tmem_ld_32x32b_x32(lane_addr + c0, ra);
      tmem_ld_32x32b_x32(lane_addr + c0 + 32, rb);
      tmem_ld_wait();
      if (cs == 1) {
#pragma unroll
        for (int j = 0; j < 32; ++j) tile[(c0 + j) * L::kPitch + row] = __uint_as_float(ra[j]);
#pragma unroll
        for (int j = 0; j < 32; ++j) tile[(c0 + 32 + j) * L::kPitch + row] = __uint_as_float(rb[j]);
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) __stcg(&part[(c0 + j) * kBlockN + row], __uint_as_float(ra[j]));
#pragma unroll
        for (int j = 0; j < 32; ++j) __stcg(&part[(c0 + 32 + j) * kBlockN + row], __uint_as_float(rb[j]));
      }
    }
  };
  int r0 = 0, r1 = TOK;
  if (cs > 1) {
    r0 = (split * TOK) / cs;
    r1 = ((split + 1) * TOK) / cs;
  }
  // split-K: CTA r sums rows [r0, r1) of all partials of tile h in rank order
  // -- deterministic -- into its shared tile
  auto reduce = [&](int h) {
    const int n4 = (r1 - r0) * (kBlockN / 4);
    constexpr int kMinCs = TOK > 128 ? 4 : 2;  // the host keeps cs >= kMinCs (or 1)
    constexpr int kMaxPer = (TOK / kMinCs) * (kBlockN / 4) / kThreads + 1;
    float4 acc[kMaxPer];
#pragma unroll
    for (int k = 0; k < kMaxPer; ++k) acc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    const float4* base = reinterpret_cast<const float4*>(ws + tile_id(h) * (TOK * kBlockN)) +
                         (size_t)r0 * (kBlockN / 4);
    const size_t split_stride4 = tiles_total * (TOK * kBlockN) / 4;
    constexpr int kQ = TOK == 64 ? 4 : 2;  // partials in flight (register budget)
    for (int q0 = 0; q0 < cs; q0 += kQ) {
      float4 v[kQ][kMaxPer];
#pragma unroll
      for (int dq = 0; dq < kQ; ++dq)
#pragma unroll
        for (int k = 0; k < kMaxPer; ++k) {
          const int i = threadIdx.x + k * kThreads;
          if (q0 + dq < cs && i < n4) v[dq][k] = __ldcg(base + (size_t)(q0 + dq) * split_stride4 + i);
        }
#pragma unroll
      for (int dq = 0; dq < kQ; ++dq)
#pragma unroll
        for (int k = 0; k < kMaxPer; ++k) {
          const int i = threadIdx.x + k * kThreads;
          if (q0 + dq < cs && i < n4) {
            acc[k].x += v[dq][k].x; acc[k].y += v[dq][k].y;
            acc[k].z += v[dq][k].z; acc[k].w += v[dq][k].w;
          }
        }
    }
#pragma unroll
    for (int k = 0; k < kMaxPer; ++k) {
      const int i = threadIdx.x + k * kThreads;
      if (i < n4) {
        const int j = r0 + i / (kBlockN / 4), c = (i % (kBlockN / 4)) * 4;
        *reinterpret_cast<float4*>(&tile[j * L::kPitch + c]) = acc[k];
      }
    }
    __syncthreads();
  };
  // ---- epilogue of tile h over rows [r0, r1) (gemm_epi.cuh)
  auto epilogue = [&](int h) {
    const int nt = (int)blockIdx.x * NB + h;
    SRL_STAMP(4);
    griddep_wait();  // epilogue inputs (ssq, residual) come from earlier kernels
    gemm_detail::epi_row_meta<EK>(epi, r0, r1, t0, M, s_rstd, s_row, threadIdx.x, kThreads);
    __syncthreads();
    SRL_STAMP(5);
    gemm_detail::epi_apply<EK>(epi, tile, L::kPitch, r0, r1, t0, nt * kBlockN, nt, n_tiles, M, N, s_rstd,
                               s_row, threadIdx.x, kThreads, [] { __syncthreads(); });
    __syncthreads();
    SRL_STAMP(6);
  };
  if (cs == 1) {
    for (int h = 0; h < nh; ++h) {
      drain(h);
      tc_fence_before();
      __syncthreads();
      if (h == nh - 1 && warp == 0) tmem_free<NB * TOK>(tmem);
      SRL_STAMP(3);
      epilogue(h);
    }
  } else {
    for (int h = 0; h < nh; ++h) drain(h);
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_free<NB * TOK>(tmem);
    SRL_STAMP(3);
    // after one cluster barrier (release/acquire orders the global partials)
    cluster_sync();
    SRL_STAMP(7);
    for (int h = 0; h < nh; ++h) {
      reduce(h);
      epilogue(h);
    }
  }
}

// One instance per epilogue kind (only its own epilogue in the instruction stream).
template <int TOK, int STAGES, int EK, int NB = 1>
cudaError_t launch_impl(const CUtensorMap& tw, const CUtensorMap& tx, int M, int N, int K, int cs,
                        const GemmWorkspace& ws, const EpiParams& epi, cudaStream_t stream) {
  using L = Layout<TOK, STAGES, NB>;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(gemm_bf16_kernel<TOK, STAGES, EK, NB>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, L::kAlloc);
  });
  if (attr_err != cudaSuccess) return attr_err;
  const int n_tiles = (N + kBlockN - 1) / kBlockN;
  const int tok_tiles = (M + TOK - 1) / TOK;
  if (cs > 1) {
    const size_t need = (size_t)cs * n_tiles * tok_tiles * TOK * kBlockN;
    if (ws.partials == nullptr || need > ws.partial_floats) return cudaErrorInvalidValue;
  }
  return launch_pdl(gemm_bf16_kernel<TOK, STAGES, EK, NB>, dim3((n_tiles + NB - 1) / NB, cs, tok_tiles),
                    dim3(kThreads), (size_t)L::kAlloc, stream, dim3(1, cs, 1), tw, tx, M, N, K, cs,
                    ws.partials, epi);
}

// 128 < M <= 256 token rows (e.g. the 7B batch-256 decode): one 256-token tile
// and two 128-row weight tiles per CTA (X read once per 256 weight rows),
// split-K over a cluster of kSkinnyCs CTAs.  Kinds with per-tile-pair
// epilogues (SwiGLU) or a vocabulary-wide N keep the other paths.
constexpr int kSkinnyCs = 8;
int skinny256_splits(int M, int N, int K, int kind, int num_sms) {
  static const bool off = [] {
    const char* v = std::getenv("SRL_GEMM_SKINNY");
    return v && v[0] == '0';
  }();
  if (off || M <= 128 || M > 256) return 0;
  if (kind != EPI_STORE_F32 && kind != EPI_RESID && kind != EPI_STORE_BF16 && kind != EPI_QKV) return 0;
  const int tiles = (N + 2 * kBlockN - 1) / (2 * kBlockN);
  // >= 32 k-blocks per split: a 256 x 256 fp32 partial pair (256 KB per CTA)
  // costs more than the X re-reads it saves on short K (7B O / QKV, K = 3584:
  // 29 -> 38 / 30 -> 81 us; down, K = 18944: 74 -> 59.5 us)
  auto fits = [&](int cs) { return tiles * cs <= (3 * num_sms) / 2 && K / kBlockK >= 32 * cs; };
  int cs = kSkinnyCs;
  while (cs > 4 && !fits(cs)) cs /= 2;
  if (!fits(cs)) return 0;
  return cs;
}
size_t skinny256_ws_floats(int N) {
  return (size_t)kSkinnyCs * ((N + kBlockN - 1) / kBlockN) * 256 * kBlockN;
}
cudaError_t launch_skinny256(const CUtensorMap& tw, const CUtensorMap& tx, int M, int N, int K, int cs,
                             const GemmWorkspace& ws, const EpiParams& epi, cudaStream_t stream) {
  switch (epi.kind) {
    case EPI_STORE_F32: return launch_impl<256, 3, EPI_STORE_F32, 2>(tw, tx, M, N, K, cs, ws, epi, stream);
    case EPI_RESID: return launch_impl<256, 3, EPI_RESID, 2>(tw, tx, M, N, K, cs, ws, epi, stream);
    case EPI_STORE_BF16: return launch_impl<256, 3, EPI_STORE_BF16, 2>(tw, tx, M, N, K, cs, ws, epi, stream);
    case EPI_QKV: return launch_impl<256, 3, EPI_QKV, 2>(tw, tx, M, N, K, cs, ws, epi, stream);
    default: return cudaErrorInvalidValue;
  }
}

template <int TOK>
cudaError_t launch_kind(const CUtensorMap& tw, const CUtensorMap& tx, int M, int N, int K, int cs,
                        const GemmWorkspace& ws, const EpiParams& epi, cudaStream_t stream) {
  switch (epi.kind) {
    case 0: return launch_impl<TOK, 4, 0>(tw, tx, M, N, K, cs, ws, epi, stream);
    case 1: return launch_impl<TOK, 4, 1>(tw, tx, M, N, K, cs, ws, epi, stream);
    case 2: return launch_impl<TOK, 4, 2>(tw, tx, M, N, K, cs, ws, epi, stream);
    case 3: return launch_impl<TOK, 4, 3>(tw, tx, M, N, K, cs, ws, epi, stream);
    case 4: return launch_impl<TOK, 4, 4>(tw, tx, M, N, K, cs, ws, epi, stream);
    case 5: return launch_impl<TOK, 4, 5>(tw, tx, M, N, K, cs, ws, epi, stream);
    case 6: return launch_impl<TOK, 4, 6>(tw, tx, M, N, K, cs, ws, epi, stream);
    case 7: return launch_impl<TOK, 4, 7>(tw, tx, M, N, K, cs, ws, epi, stream);
    default: return cudaErrorInvalidValue;
  }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn get_encode() {
  static EncodeFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<EncodeFn>(nullptr);
    return reinterpret_cast<EncodeFn>(p);
  }();
  return fn;
}

}  // namespace

CUtensorMap make_tmap_bf16(const void* ptr, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  CUtensorMap m;
  std::memset(&m, 0, sizeof(m));
  EncodeFn enc = get_encode();
  if (enc == nullptr) {
    std::fprintf(stderr, "srl: cuTensorMapEncodeTiled unavailable\n");
    std::abort();
  }
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {cols * 2};
  const cuuint32_t box[2] = {64, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims,
                         strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    std::fprintf(stderr, "srl: cuTensorMapEncodeTiled failed (%d) rows=%llu cols=%llu\n", (int)r,
                 (unsigned long long)rows, (unsigned long long)cols);
    std::abort();
  }
  return m;
}

int gemm_tok_tile(int M) { return M <= 64 ? 64 : 128; }

// Cluster split-K factor: a power of two <= 8, at least two k-blocks per
// split, growing while the grid is below ~1.5 waves of the machine.
int gemm_auto_splits(int M, int N, int K, int num_sms) {
  const int tok = gemm_tok_tile(M);
  const int tiles = ((N + kBlockN - 1) / kBlockN) * ((M + tok - 1) / tok);
  const int kb = K / kBlockK;
  int cs = 1;
  while (cs * 2 <= kMaxCluster && kb >= 2 * (cs * 2) && tiles * cs * 2 <= (3 * num_sms) / 2) cs *= 2;
  return cs;
}

size_t gemm_workspace_floats(int M, int N, int splits) {
  const int tok = gemm_tok_tile(M);
  int cs = 1;
  while (cs * 2 <= splits && cs * 2 <= kMaxCluster) cs *= 2;
  // (128, 256] rows may take the skinny 256-token path instead (gemm_bf16_launch)
  const size_t skinny = (M > 128 && M <= 256) ? skinny256_ws_floats(N) : 0;
  if (cs == 1) return skinny;
  return std::max(skinny, (size_t)cs * ((N + kBlockN - 1) / kBlockN) * ((M + tok - 1) / tok) * tok * kBlockN);
}

cudaError_t gemm_bf16_launch(const CUtensorMap& tw, const CUtensorMap& tx, int M, int N, int K,
                             int splits, const GemmWorkspace& ws, const EpiParams& epi,
                             cudaStream_t stream) {
  if (M < 1 || N < 1 || K < kBlockK || K % kBlockK != 0 || splits < 1)
    return cudaErrorInvalidValue;
  if (epi.kind == EPI_SWIGLU && N % kBlockN != 0) return cudaErrorInvalidValue;
  // many token rows: the persistent double-buffered kernel (gemm_big.cu);
  // SRL_GEMM_BIG=0 disables it, =1 forces it for every M > 64 (A/B tests)
  static const char* big_env = std::getenv("SRL_GEMM_BIG");
  static const int sms = [] {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  if (const int scs = skinny256_splits(M, N, K, epi.kind, sms)) {
    if (ws.partials != nullptr && (size_t)scs * ((N + kBlockN - 1) / kBlockN) * 256 * kBlockN <= ws.partial_floats) {
      static const bool log = std::getenv("SRL_GEMM_LOG") != nullptr;
      if (log) std::fprintf(stderr, "srl gemm M=%d N=%d K=%d kind=%d path=skinny256x%d\n", M, N, K, epi.kind, scs);
      return launch_skinny256(tw, tx, M, N, K, scs, ws, epi, stream);
    }
  }
  int big = gemm_big_tok(M, N, K, sms);
  if (big_env && big_env[0] == '0') big = 0;
  if (big_env && big_env[0] == '1' && M > 64 && big == 0) big = 128;
  static const bool log = std::getenv("SRL_GEMM_LOG") != nullptr;  // launch trace (profiling)
  if (log) std::fprintf(stderr, "srl gemm M=%d N=%d K=%d kind=%d path=%s\n", M, N, K, epi.kind,
                        big ? (big == 256 ? "big256" : "big128") : "splitk");
  if (big) return gemm_big_launch(tw, tx, M, N, K, big, epi, stream);
  int cs = 1;
  while (cs * 2 <= splits && cs * 2 <= kMaxCluster && cs * 2 <= K / kBlockK) cs *= 2;
  if (gemm_tok_tile(M) == 64) return launch_kind<64>(tw, tx, M, N, K, cs, ws, epi, stream);
  return launch_kind<128>(tw, tx, M, N, K, cs, ws, epi, stream);
}

}  // namespace srl
