// gemm_big.cu -- persistent, warp-specialised tcgen05 GEMM for many token
// rows (prefill chunks, the trainer's forward and backward GEMMs).
//
// Same contract and fused epilogues as gemm.cu (swap-AB: 128 weight rows are
// the UMMA M, TOK = 128 or 256 token rows the UMMA N), but built for
// throughput instead of decode latency:
//   * one CTA per SM walks output tiles n-fastest (concurrent CTAs share the
//     activation block, the weights stay L2-resident);
//   * warp 0 streams A (16 KB) + B (TOK x 128 B) k-blocks by TMA into a
//     STAGES-deep ring across tile boundaries; warp 1 issues
//     tcgen05.mma 128 x TOK x 16 into one of TWO TMEM accumulators
//     (2 x TOK fp32 columns) and moves on to the next tile at once;
//   * warps 4-11 drain the other accumulator and run the epilogue while the
//     next tile's MMAs run: two groups of four warps (each group covers the
//     128 TMEM lanes) take alternate 32-token chunks, stage them in shared
//     memory and run gemm_epi.cuh on them.
// No split-K: it is chosen only when the tile count fills the machine.
#include "gemm_big_impl.cuh"

namespace srl {
using bigk::launch_big;

namespace {
template <int TOK, bool AMN, bool BMN>
cudaError_t by_kind(const CUtensorMap& tw, const CUtensorMap& tx, int M, int N, int K, int splits,
                    const EpiParams& epi, cudaStream_t stream) {
  if constexpr (!AMN) {
    switch (epi.kind) {
      case 0: return launch_big<TOK, false, false, 0>(tw, tx, M, N, K, splits, epi, stream);
      case 1: return launch_big<TOK, false, false, 1>(tw, tx, M, N, K, splits, epi, stream);
      case 2: return launch_big<TOK, false, false, 2>(tw, tx, M, N, K, splits, epi, stream);
      case 3: return launch_big<TOK, false, false, 3>(tw, tx, M, N, K, splits, epi, stream);
      case 4: return launch_big<TOK, false, false, 4>(tw, tx, M, N, K, splits, epi, stream);
      case 5: return launch_big<TOK, false, false, 5>(tw, tx, M, N, K, splits, epi, stream);
      case 6: return launch_big<TOK, false, false, 6>(tw, tx, M, N, K, splits, epi, stream);
      case 7: return launch_big<TOK, false, false, 7>(tw, tx, M, N, K, splits, epi, stream);
      default: return cudaErrorInvalidValue;
    }
  } else if constexpr (BMN) {
    switch (epi.kind) {
      case 0: return launch_big<TOK, true, true, 0>(tw, tx, M, N, K, splits, epi, stream);
      case 6: return launch_big<TOK, true, true, 6>(tw, tx, M, N, K, splits, epi, stream);
      default: return cudaErrorInvalidValue;
    }
  } else {
    switch (epi.kind) {
      case 0: return launch_big<TOK, true, false, 0>(tw, tx, M, N, K, splits, epi, stream);
      case 6: return launch_big<TOK, true, false, 6>(tw, tx, M, N, K, splits, epi, stream);
      case 8: return launch_big<TOK, true, false, 8>(tw, tx, M, N, K, splits, epi, stream);
      default: return cudaErrorInvalidValue;
    }
  }
}
}  // namespace

// Measured on B200 (tools/gemm_bench.py --graph, Qwen2.5 0.5B/1.5B/7B
// shapes, M = 200..20480): with per-kind instances the persistent kernel
// beats the cluster split-K kernel from M = 200 on for every 0.5B shape but
// a long K on very few tiles (down projection at M = 200: 14 tiles), and the
// 7B down projection on less than a wave.  256-token tiles pay off once
// there are two waves of them.
int gemm_big_tok(int M, int N, int K, int num_sms) {
  if (M <= 64) return 0;
  const int n_tiles = (N + bigk::kBN - 1) / bigk::kBN;
  if (n_tiles * ((M + 255) / 256) >= 2 * num_sms) return 256;
  const int t128 = n_tiles * ((M + 127) / 128);
  if ((K >= 2048 && t128 < 16) || (K >= 8192 && t128 < num_sms)) return 0;
  return 128;
}

cudaError_t gemm_big_launch(const CUtensorMap& tw, const CUtensorMap& tx, int M, int N, int K, int tok,
                            const EpiParams& epi, cudaStream_t stream) {
  if (tok == 256) return by_kind<256, false, false>(tw, tx, M, N, K, 1, epi, stream);
  if (tok == 128) return by_kind<128, false, false>(tw, tx, M, N, K, 1, epi, stream);
  return cudaErrorInvalidValue;
}

// MN-major plan: 256-token tiles when they give two waves, else 128; long-K
// outputs of less than half a wave get K slices (>= 8 k-blocks each) up to
// about one wave.
int gemm_mn_plan(int M, int N, int K, int num_sms, int* splits) {
  const int n_tiles = (N + bigk::kBN - 1) / bigk::kBN;
  const int tok = n_tiles * ((M + 255) / 256) >= 2 * num_sms ? 256 : 128;
  const int tiles = n_tiles * ((M + tok - 1) / tok);
  int s = 1;
  if (2 * tiles <= num_sms)
    while ((s + 1) * tiles <= num_sms && (K / bigk::kBK) / (s + 1) >= 8) ++s;
  *splits = s;
  return tok;
}

cudaError_t gemm_mn_launch(const CUtensorMap& tw, const CUtensorMap& tx, int M, int N, int K, int tok,
                           int splits, bool x_mn, const EpiParams& epi, cudaStream_t stream) {
  if (M < 1 || N < 1 || K < bigk::kBK || K % bigk::kBK != 0 || splits < 1 || splits > K / bigk::kBK)
    return cudaErrorInvalidValue;
  const bool direct = epi.kind == EPI_ACCUM_F32 || epi.kind == EPI_STORE_F32 || epi.kind == EPI_SWIGLU_BWD;
  if (epi.kind == EPI_SWIGLU_BWD &&  // 16-byte rows of the dgu tile
      (N % 64 != 0 || epi.ld_bf16 % 8 != 0 || (reinterpret_cast<uintptr_t>(epi.out_bf16) & 15) != 0))
    return cudaErrorInvalidValue;
  if (!direct || (splits > 1 && (epi.kind != EPI_ACCUM_F32 || epi.tile_flags == nullptr)) ||
      epi.ssq_in != nullptr || epi.bias != nullptr)
    return cudaErrorInvalidValue;
  if (x_mn) {
    if (tok == 256) return by_kind<256, true, true>(tw, tx, M, N, K, splits, epi, stream);
    if (tok == 128) return by_kind<128, true, true>(tw, tx, M, N, K, splits, epi, stream);
  } else {
    if (tok == 256) return by_kind<256, true, false>(tw, tx, M, N, K, splits, epi, stream);
    if (tok == 128) return by_kind<128, true, false>(tw, tx, M, N, K, splits, epi, stream);
  }
  return cudaErrorInvalidValue;
}

}  // namespace srl
