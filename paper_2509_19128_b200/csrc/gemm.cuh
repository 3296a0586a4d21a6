// gemm.cuh -- host-visible interface of the tcgen05 GEMM used by every
// projection of the decoder policy (QKV, O, gate/up, down, LM head).
//
//   Y[m, n] = epilogue( sum_k X[m, k] * W[n, k] )       X: [M x K] bf16 (tokens)
//                                                       W: [N x K] bf16 (weights)
// The kernel is "swap-AB": weight rows fill the UMMA M=128 dimension and the
// token rows are the UMMA N (64 or 128), so a decode batch of 64 tokens still
// issues full-height tensor-core tiles while the weights stream from HBM.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace srl {

enum EpiKind : int {
  EPI_STORE_F32 = 0,   // out_f32[m, n] = rstd[m] * acc (+ bias[n])
  EPI_RESID = 1,       // resid[m, n] += acc; xg[m, n] = bf16(resid * gain[n]); ssq partials
  EPI_SWIGLU = 2,      // tile = 64 gate | 64 up rows: act[m, j] = bf16(silu(g) * u), g,u scaled by rstd
  EPI_STORE_BF16 = 3,  // out_bf16[m, n] = bf16(rstd[m] * acc (+ bias[n]))
  EPI_QKV = 4,         // rstd*acc + bias, RoPE on q/k, q -> bf16 rows, k/v -> paged KV cache
  EPI_LOGITS = 5,      // out_f32 = rstd*acc; per (row, 128-col tile): max and fp64 sum exp(x - max)
  EPI_ACCUM_F32 = 6,   // out_f32[m, n] += scale * acc  (gradient accumulation)
  EPI_DLOGITS = 7,     // x = rstd*acc; d = coef[m] * (onehot(tgt[m]) - exp(x - lse[m])) -> bf16
  EPI_SWIGLU_BWD = 8,  // acc = dact[m, j]: dgu (bf16, gate | up 64-col interleave of gu_in) = SwiGLU'
                       // out_bf16[m, n] and (outT_bf16) the transpose [n, m]
};

struct EpiParams {
  int kind = EPI_STORE_F32;
  // Deferred RMSNorm: rstd[m] = rsqrt(sum_p ssq_in[m * ssq_in_parts + p] * inv_dim + eps).
  const float* ssq_in = nullptr;
  int ssq_in_parts = 0;
  float inv_dim = 0.f;
  float eps = 0.f;
  const __nv_bfloat16* bias = nullptr;  // [N]
  float* out_f32 = nullptr;
  int ld_out = 0;
  __nv_bfloat16* out_bf16 = nullptr;
  int ld_bf16 = 0;
  // EPI_RESID
  float* resid = nullptr;               // [M x N] fp32, ld = N
  const __nv_bfloat16* gain = nullptr;  // next RMSNorm gain [N]
  __nv_bfloat16* xg = nullptr;          // [M x N] bf16
  float* ssq_out = nullptr;             // [M x ceil(N/128)]
  // EPI_QKV
  int nq = 0, nkv = 0, hd = 0, pages_per_seq = 0;
  const int32_t* row_slot = nullptr;    // plan: slot of each row (-1 = padding)
  const int32_t* row_pos = nullptr;     // plan: position of each row
  const int32_t* block_table = nullptr; // [slots x pages_per_seq]
  const float* cos_sin = nullptr;       // [max_pos x hd] (cos | sin)
  __nv_bfloat16* q_out = nullptr;       // [M x nq*hd]
  __nv_bfloat16* kc = nullptr;          // [pages][nkv][64][hd] (this layer)
  __nv_bfloat16* vc = nullptr;
  // EPI_LOGITS
  float* part_max = nullptr;            // [M x ceil(N/128)]
  double* part_sum = nullptr;           // [M x ceil(N/128)]
  float scale = 1.f;                    // EPI_ACCUM_F32
  // EPI_LOGITS (optional): out_f32 may be null (statistics only); the logit of
  // column tgt_row[m] is stored to tgt_out[m].  EPI_DLOGITS: see above.
  const int32_t* tgt_row = nullptr;
  float* tgt_out = nullptr;
  const double* lse_in = nullptr;
  const float* row_coef = nullptr;
  __nv_bfloat16* outT_bf16 = nullptr;
  // EPI_SWIGLU also keeps the rstd-scaled gate | up for the backward, and
  // EPI_SWIGLU_BWD reads it back, in the token-blocked layout of gu_index():
  // a (32-token block, column) pair is 32 contiguous values, which is exactly
  // what one epilogue thread holds (column = TMEM lane, 32 tokens) -- 16-byte
  // vector stores / loads instead of 32 strided scalars.  Rows padded to 32.
  __nv_bfloat16* out2_bf16 = nullptr;   // EPI_SWIGLU: bf16 gate | up [M x N], gu_index layout
  const __nv_bfloat16* gu_in = nullptr; // EPI_SWIGLU_BWD: gate | up pre-activations [M x 2N], gu_index layout
  int ldT = 0;
  int* tile_flags = nullptr;            // gemm_mn_launch split-K ordering (>= tiles ints, zeroed once)
  // Split operands (gemm_big only; the trainer's precise mode carries a value
  // as two bf16 halves hi + lo = fp32 to ~2^-17).  The K loop is the
  // concatenation of up to 3 segments of seg_kb k-blocks each (K = segments *
  // seg_kb * 64); segment s reads X and W shifted by x_off[s] / w_off[s]
  // elements -- along K for a K-major operand, along MN for an MN-major one.
  // (hi + lo) W = [hi | lo] . [W ; W]: 2 segments, x_off = {0, lo}, w_off = 0;
  // (dh + dl)^T (uh + ul) ~ dh uh + dh ul + dl uh: 3 segments.
  int seg_kb = 0;                       // 0: one plain segment
  int x_off0 = 0, x_off1 = 0, x_off2 = 0;
  int w_off0 = 0, w_off1 = 0, w_off2 = 0;
  // Split bf16 outputs (EPI_RESID xg, EPI_SWIGLU act, EPI_DLOGITS, EPI_SWIGLU_BWD):
  // hi at column c, lo = bf16(v - hi) at column c + lo_off (0: hi only).
  // EPI_RESID's xg row stride is N + lo_off.
  int lo_off = 0;
  float* out2_f32 = nullptr;            // EPI_SWIGLU: fp32 gate | up [M x N], gu_index layout
  const float* gu_in_f32 = nullptr;     // EPI_SWIGLU_BWD: fp32 gate | up (instead of gu_in), gu_index layout
  const float* row_scale = nullptr;     // EPI_SWIGLU_BWD: dgu[m, :] *= row_scale[m]
  int fold_rstd = 0;                    // EPI_DLOGITS: d *= rstd[m] (the LM head's rstd folded in)
  // debug: per-CTA %globaltimer phase stamps [ctas x 8] (null = off)
  unsigned long long* stamps = nullptr;
};

// token-blocked gate | up layout (EPI_SWIGLU out2_*, EPI_SWIGLU_BWD gu_in*) of
// an [M x N] matrix (M padded to 32, N % 32 == 0): 32 tokens x 32 columns
// blocks, inside a block V-token groups (V = 4 fp32 / 8 bf16 = 16 bytes) of
// the 32 columns, each column's V tokens contiguous.  An epilogue warp holds
// 32 columns x 32 tokens (lane = column), so each 16-byte vector store / load
// of the warp covers 512 contiguous bytes.
template <int V>
__host__ __device__ __forceinline__ size_t gu_index_v(size_t m, size_t col, size_t N) {
  return ((((m >> 5) * (N >> 5) + (col >> 5)) * (32 / V) + ((m & 31) / V)) << 5 | (col & 31)) * V + (m % V);
}
__host__ __device__ __forceinline__ size_t gu_index(size_t m, size_t col, size_t N) {  // bf16
  return gu_index_v<8>(m, col, N);
}
__host__ __device__ __forceinline__ size_t gu_index_f32(size_t m, size_t col, size_t N) {
  return gu_index_v<4>(m, col, N);
}
__host__ __device__ __forceinline__ size_t gu_rows_padded(size_t M) { return (M + 31) & ~size_t(31); }


// Build a 2-D bf16 TMA descriptor for a row-major [rows x cols] matrix with a
// box of [box_rows x 64] elements and 128-B swizzle (the UMMA K-major layout).
CUtensorMap make_tmap_bf16(const void* ptr, uint64_t rows, uint64_t cols, uint32_t box_rows);

struct GemmWorkspace {
  float* partials = nullptr;  // split-K partial tiles
  size_t partial_floats = 0;
  int* counters = nullptr;    // per output tile arrival counters (self-resetting)
  int counter_count = 0;
};

// Number of output tiles the kernel will use for (M, N); tok_tile is 64 or 128.
int gemm_tok_tile(int M);
// Choose a split-K factor that fills the machine for skinny (decode) GEMMs.
int gemm_auto_splits(int M, int N, int K, int num_sms);
size_t gemm_workspace_floats(int M, int N, int splits);

// Persistent large-M kernel (gemm_big.cu): token tile 256 or 128 when the
// tile count fills `num_sms`, else 0 (use the split-K kernel).
int gemm_big_tok(int M, int N, int K, int num_sms);
cudaError_t gemm_big_launch(const CUtensorMap& tw, const CUtensorMap& tx, int M, int N, int K, int tok,
                            const EpiParams& epi, cudaStream_t stream);

// W operand MN-major: tw maps W as [K x N] with 64 x 64 boxes
// (make_tmap_bf16(p, K_rows, N, 64)); rows past the map's K read as zero, so
// K may be rounded up to 64.  x_mn: X is MN-major too ([K x M], 64 x 64
// boxes), else K-major [M x K] with a box of `tok` rows.  C[m, n] = sum_k
// X(m, k) W[k, n] through EPI_STORE_F32 / EPI_ACCUM_F32 / EPI_SWIGLU_BWD (no rstd / bias);
// splits > 1 (ordered K slices) needs EPI_ACCUM_F32 and epi.tile_flags.
int gemm_mn_plan(int M, int N, int K, int num_sms, int* splits);
cudaError_t gemm_mn_launch(const CUtensorMap& tw, const CUtensorMap& tx, int M, int N, int K, int tok,
                           int splits, bool x_mn, const EpiParams& epi, cudaStream_t stream);

// Launch.  tw: W [N x K] (box 128 rows); tx: X [>=M x K] (box gemm_tok_tile(M) rows).
// Dispatches to gemm_big_launch when gemm_big_tok() says so (splits ignored).
cudaError_t gemm_bf16_launch(const CUtensorMap& tw, const CUtensorMap& tx, int M, int N, int K,
                             int splits, const GemmWorkspace& ws, const EpiParams& epi,
                             cudaStream_t stream);

}  // namespace srl
