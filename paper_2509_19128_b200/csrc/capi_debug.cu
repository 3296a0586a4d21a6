// capi_debug.cu -- kernel-level C entry points used by the parity tests and
// bench.py to exercise single kernels through the same shared library the
// engine uses (declared in include/streamrl_b200.h, "kernel entry points").
#include <cuda_runtime.h>

#include "decoder.cuh"
#include "gemm.cuh"
#include "train.cuh"
#include "streamrl_b200.h"

using namespace srl;

namespace {
int cuda_status(cudaError_t e) { return e == cudaSuccess ? SRL_OK : SRL_CUDA_ERROR; }
int num_sms() {
  int dev = 0, n = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}
}  // namespace

static unsigned long long* g_stamps = nullptr;  // debug phase stamps (srl_debug_gemm_stamps)
extern "C" void srl_debug_gemm_stamps(unsigned long long* device_buf) { g_stamps = device_buf; }

extern "C" int srl_kernel_gemm_bf16(const void* w, const void* x, int32_t M, int32_t N, int32_t K,
                                    int32_t splits, int32_t epi_kind, const void* bias,
                                    const float* ssq_in, int32_t ssq_parts, float inv_dim,
                                    float eps, void* out, float* resid, const void* gain,
                                    void* xg, float* ssq_out, void* stream) {
  if (!w || !x || M < 1 || N < 1 || K < 64 || K % 64) return SRL_INVALID_ARGUMENT;
  const int tok = gemm_tok_tile(M);
  const CUtensorMap tw = make_tmap_bf16(w, (uint64_t)N, (uint64_t)K, 128);
  const CUtensorMap tx = make_tmap_bf16(x, (uint64_t)M, (uint64_t)K, (uint32_t)tok);
  if (splits <= 0) splits = gemm_auto_splits(M, N, K, num_sms());
  GemmWorkspace ws;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  static float* g_ws = nullptr;
  static size_t g_ws_floats = 0;
  const size_t need = gemm_workspace_floats(M, N, splits);
  if (need > g_ws_floats) {
    if (g_ws) cudaFree(g_ws);
    if (cudaMalloc(&g_ws, need * sizeof(float)) != cudaSuccess) return SRL_OUT_OF_MEMORY;
    g_ws_floats = need;
  }
  ws.partials = g_ws;
  ws.partial_floats = g_ws_floats;
  EpiParams epi;
  epi.stamps = g_stamps;
  epi.kind = epi_kind;
  epi.ssq_in = ssq_in;
  epi.ssq_in_parts = ssq_parts;
  epi.inv_dim = inv_dim;
  epi.eps = eps;
  epi.bias = static_cast<const __nv_bfloat16*>(bias);
  if (epi_kind == EPI_STORE_F32) {
    epi.out_f32 = static_cast<float*>(out);
    epi.ld_out = N;
  } else if (epi_kind == EPI_STORE_BF16) {
    epi.out_bf16 = static_cast<__nv_bfloat16*>(out);
    epi.ld_bf16 = N;
  } else if (epi_kind == EPI_SWIGLU) {
    epi.out_bf16 = static_cast<__nv_bfloat16*>(out);
    epi.ld_bf16 = N / 2;
  } else if (epi_kind == EPI_RESID) {
    epi.resid = resid;
    epi.gain = static_cast<const __nv_bfloat16*>(gain);
    epi.xg = static_cast<__nv_bfloat16*>(xg);
    epi.ssq_out = ssq_out;
  }
  return cuda_status(gemm_bf16_launch(tw, tx, M, N, K, splits, ws, epi, st));
}

extern "C" int srl_kernel_gemm_mn(const void* w, const void* x, int32_t M, int32_t N, int32_t k_rows,
                                  int32_t x_kmajor, int32_t splits, int32_t accumulate, float scale,
                                  float* out, void* stream) {
  if (!w || !x || !out || M < 1 || N < 1 || k_rows < 1 || N % 8) return SRL_INVALID_ARGUMENT;
  if (x_kmajor ? k_rows % 64 != 0 : M % 8 != 0) return SRL_INVALID_ARGUMENT;
  const int K = (k_rows + 63) / 64 * 64;
  const CUtensorMap tw = make_tmap_bf16(w, (uint64_t)k_rows, (uint64_t)N, 64);
  const CUtensorMap tx = x_kmajor ? make_tmap_bf16(x, (uint64_t)M, (uint64_t)K, 128)
                                  : make_tmap_bf16(x, (uint64_t)k_rows, (uint64_t)M, 64);
  int planned = 1;
  const int tok = gemm_mn_plan(M, N, K, num_sms(), &planned);
  if (splits <= 0) splits = planned;
  static int* g_flags = nullptr;  // split-K ordering counters (self-resetting)
  constexpr int kFlags = 1 << 16;
  if (g_flags == nullptr) {
    if (cudaMalloc(&g_flags, kFlags * sizeof(int)) != cudaSuccess) return SRL_OUT_OF_MEMORY;
    if (cudaMemset(g_flags, 0, kFlags * sizeof(int)) != cudaSuccess) return SRL_CUDA_ERROR;
  }
  if ((size_t)((N + 127) / 128) * ((M + tok - 1) / tok) > (size_t)kFlags) return SRL_INVALID_ARGUMENT;
  EpiParams epi;
  epi.kind = accumulate ? EPI_ACCUM_F32 : EPI_STORE_F32;
  epi.out_f32 = out;
  epi.ld_out = N;
  epi.scale = scale;
  epi.tile_flags = g_flags;
  if (!accumulate && splits > 1) return SRL_INVALID_ARGUMENT;
  return cuda_status(gemm_mn_launch(tw, tx, M, N, K, tok, splits, !x_kmajor, epi, static_cast<cudaStream_t>(stream)));
}

extern "C" int srl_kernel_sample_logits(const float* logits, int32_t vocab, int32_t rows,
                                        const uint64_t* seeds, const int32_t* draw_index,
                                        int32_t greedy, int32_t* tokens_out, double* logprobs_out,
                                        void* stream) {
  if (!logits || vocab < 1 || rows < 0 || !seeds || !draw_index || !tokens_out || !logprobs_out)
    return SRL_INVALID_ARGUMENT;
  launch_sample_logits(logits, vocab, rows, seeds, draw_index, greedy, tokens_out, logprobs_out,
                       static_cast<cudaStream_t>(stream));
  return cuda_status(cudaGetLastError());
}

// Single-query paged GQA attention (the multi-kernel round's attention_kernel,
// decoder.cu) on caller buffers: q [rows x nq x hd] bf16, K / V caches
// [pages][nkv][64][hd] bf16, block_table [slots x pages_per_seq], per row its
// slot and position (keys 0..pos).  out [rows x nq x hd] bf16.
extern "C" int srl_kernel_attention_decode(const void* q, const void* kc, const void* vc,
                                           const int32_t* block_table, int32_t pages_per_seq,
                                           const int32_t* row_slot, const int32_t* row_pos, int32_t rows,
                                           int32_t nq, int32_t nkv, int32_t hd, int32_t max_ctx, void* out,
                                           void* stream) {
  if (!q || !kc || !vc || !block_table || !row_slot || !row_pos || !out || rows < 1 || nkv < 1 ||
      nq % nkv != 0 || (hd != 64 && hd != 128) || max_ctx < 1)
    return SRL_INVALID_ARGUMENT;
  DecoderDims d{};
  d.nq = nq;
  d.nkv = nkv;
  d.hd = hd;
  RoundPlan plan{const_cast<int32_t*>(row_slot), const_cast<int32_t*>(row_pos), nullptr, nullptr};
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t wsf = attention_ws_floats(d, rows, max_ctx);
  float* ws = nullptr;
  int* ctr = nullptr;
  if (cudaMallocAsync(&ws, sizeof(float) * wsf, st) != cudaSuccess ||
      cudaMallocAsync(&ctr, sizeof(int) * (size_t)rows * nkv, st) != cudaSuccess)
    return SRL_CUDA_ERROR;
  cudaMemsetAsync(ctr, 0, sizeof(int) * (size_t)rows * nkv, st);
  launch_attention(static_cast<const __nv_bfloat16*>(q), d, plan, rows, block_table, pages_per_seq,
                   static_cast<const __nv_bfloat16*>(kc), static_cast<const __nv_bfloat16*>(vc), max_ctx, ws,
                   ctr, wsf, static_cast<__nv_bfloat16*>(out), st);
  cudaFreeAsync(ws, st);
  cudaFreeAsync(ctr, st);
  return cuda_status(cudaGetLastError());
}

// Causal multi-query attention over packed segments (train_attn.cu
// attn_fwd_mma): the trainer's forward and a prefill round's prompt rows.
extern "C" int srl_kernel_attention_prefill(const void* q, const void* kc, const void* vc,
                                            const int32_t* block_table, int32_t pages_per_seq,
                                            const int32_t* seq_start, const int32_t* seq_len,
                                            const int32_t* seg_pos0, const int32_t* seg_slot, int32_t n_seg,
                                            int32_t max_rows, int32_t nq, int32_t nkv, int32_t hd, void* out,
                                            float* lse, int32_t out_lo, void* stream) {
  if (!q || !kc || !vc || !block_table || !seq_start || !seq_len || !out || n_seg < 1 || max_rows < 1 ||
      nkv < 1 || nq % nkv != 0 || (hd != 64 && hd != 128) || out_lo < 0 || pages_per_seq < 1)
    return SRL_INVALID_ARGUMENT;
  return cuda_status(launch_attention_fwd_mma(
      static_cast<const __nv_bfloat16*>(q), static_cast<const __nv_bfloat16*>(kc),
      static_cast<const __nv_bfloat16*>(vc), seq_start, seq_len, block_table, pages_per_seq, n_seg, nq, nkv, hd,
      static_cast<__nv_bfloat16*>(out), lse, static_cast<cudaStream_t>(stream), seg_pos0, seg_slot, max_rows,
      out_lo));
}

// Device-to-device cudaMemcpyAsync on the caller's stream (e.g. a one-GPU
// weight update into the standby buffer on a side stream).  Measured beside
// the persistent decode megakernel it advances only in the gaps between
// rounds (~27 GB/s over a 110 ms step): hidden, but not a copy-engine path.
extern "C" int srl_device_copy_async(void* dst, const void* src, size_t nbytes, void* stream) {
  if ((!dst || !src) && nbytes) return SRL_INVALID_ARGUMENT;
  return cuda_status(cudaMemcpyAsync(dst, src, nbytes, cudaMemcpyDeviceToDevice, static_cast<cudaStream_t>(stream)));
}
