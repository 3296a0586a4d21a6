// decoder.cuh -- the decoder policy ("streamrl.policy/1" type "decoder"):
// configuration, flat bf16 weight layout, and the non-GEMM kernels of one
// decode/prefill round.  The GEMMs are in gemm.cu.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "streamrl_b200.h"

namespace srl {

constexpr int kPageTokens = 64;  // paged KV block size (tokens)

// Offsets (in bf16 elements) of every tensor inside the flat weight buffer.
// Each tensor starts on a 128-byte boundary so TMA descriptors can address it.
struct LayerOffsets {
  size_t ln1, qkv_w, qkv_b, o_w, ln2, gate_up_w, down_w;
};
struct WeightLayout {
  size_t embed = 0, final_norm = 0, lm_head = 0;
  LayerOffsets* layers = nullptr;  // host array [n_layers]
  size_t total = 0;                // elements
};

struct DecoderDims {
  int V, H, L, nq, nkv, hd, I, tie, bos, max_pos;
  float theta, eps;
  int qkv() const { return (nq + 2 * nkv) * hd; }
  int qdim() const { return nq * hd; }
  int ssq_parts() const { return (H + 127) / 128; }
};

DecoderDims dims_from(const srl_decoder_config& c);
bool dims_valid(const DecoderDims& d, const char** why);
// Fills `out` (layers array allocated with new[]); returns total elements.
size_t make_layout(const DecoderDims& d, WeightLayout& out);

// One round's row plan (device arrays, M rows): which stream slot, which
// position, which input token.  last_row[s] >= 0 marks the row whose logits
// produce slot s's next token.
struct RoundPlan {
  int32_t* row_slot;
  int32_t* row_pos;
  int32_t* row_token;
  int32_t* last_row;  // [slots]
};

// Per-slot device state.
struct SlotState {
  int32_t* live;        // 1 = emitting
  int32_t* seq_len;     // tokens in the KV cache
  int32_t* gen_count;   // tokens emitted (= event position of the next token)
  int32_t* max_tokens;
  int32_t* terminator;
  uint64_t* seed;       // SplitMix64 stream seed (engine.cpp:35)
  int32_t* history;     // [slots x max_seq] every token fed to the cache
  int32_t max_seq;
};

// Events of one round for every slot (array of records, one D2H copy).
struct DevEvent {
  int32_t flag;  // 0 none, 1 emitted, 2 emitted+Length, 3 emitted+Terminator
  int32_t token;
  int32_t position;
  int32_t version;
  double logprob;
};
struct EventRing {
  DevEvent* ev;    // [rounds x slots]
  int32_t rounds;  // R
};

// ------------------------------------------------------------ kernels ---
void launch_init_weights(__nv_bfloat16* w, const DecoderDims& d, const WeightLayout& lay,
                         uint64_t seed, double scale, cudaStream_t st);
void launch_perturb(__nv_bfloat16* w, size_t n, uint64_t seed, double magnitude, cudaStream_t st);
void launch_rope_table(float* cos_sin, int max_pos, int hd, double theta, cudaStream_t st);

// x = E[token]; xg = bf16(x * gain); ssq partial sums of x^2 per 128 cols.
void launch_embed(const __nv_bfloat16* embed, const __nv_bfloat16* gain, const int32_t* row_token,
                  int M, int H, int V, float* x, __nv_bfloat16* xg, float* ssq, cudaStream_t st);

// RoPE on q,k of qkv (fp32, bias already added) -> q bf16; k,v -> paged cache.
void launch_rope_append(const float* qkv, const DecoderDims& d, const RoundPlan& plan, int M,
                        const float* cos_sin, const int32_t* block_table, int pages_per_seq,
                        __nv_bfloat16* kc, __nv_bfloat16* vc, __nv_bfloat16* q_out,
                        cudaStream_t st);

// Causal paged GQA attention: row m attends keys [0, row_pos[m]] of its slot.
void launch_attention(const __nv_bfloat16* q, const DecoderDims& d, const RoundPlan& plan, int M,
                      const int32_t* block_table, int pages_per_seq, const __nv_bfloat16* kc,
                      const __nv_bfloat16* vc, int max_ctx, float* ws, int* counters,
                      size_t ws_floats, __nv_bfloat16* out, cudaStream_t st,
                      float* lse_out = nullptr /* [M x nq] natural-log LSE, for backward */,
                      int out_lo = 0 /* > 0: out rows are [hi | lo] split pairs, lo at + out_lo */);
size_t attention_ws_floats(const DecoderDims& d, int M, int max_ctx);

// Gather the last row of each emitting slot (decode rounds use identity).
void launch_slot_set(const SlotState& ss, int slot, int live, int reset, int max_tokens, int terminator,
                     uint64_t seed, cudaStream_t st);
void launch_gather_rows(const __nv_bfloat16* xg, const float* ssq, const int32_t* last_row,
                        int slots, int H, int parts, __nv_bfloat16* xg_out, float* ssq_out,
                        cudaStream_t st);

// fp64 log-softmax + SplitMix64 inverse-CDF (or greedy argmax) sampling of
// each emitting slot's logits row; emits events, advances slot state and
// writes next round's decode plan.
void launch_sample(const float* logits, const float* pmax, const double* psum, int V, int slots,
                   const RoundPlan& plan, RoundPlan next_plan, SlotState ss, EventRing ring,
                   const int32_t* round_ctr, const int32_t* version, int greedy, cudaStream_t st);

// Sampler over raw logits rows (row r draws uniform #draw[r] of seeds[r]).
void launch_sample_logits(const float* logits, int V, int rows, const uint64_t* seeds,
                          const int32_t* draw, int greedy, int32_t* tok, double* lp, cudaStream_t st);

// out[r] = logits[r, targets[r]] - logsumexp(logits[r, :]) in fp64.
// KL(softmax(p row) || softmax(q row)) per row, fp64 (numeric.hpp:34-46).
void launch_row_kl(const float* logits_p, const float* logits_q, int V, int rows, double* out, cudaStream_t st);
void launch_row_logprobs(const float* logits, int V, int rows, const int32_t* targets, double* out,
                         cudaStream_t st);

// Copy next_plan -> plan and bump the device round counter (the first
// kernel of every round; the sampler writes events to ring[(ctr-1) % R]).
void launch_plan_copy(RoundPlan dst, RoundPlan src, int rows, int slots, int32_t* round_ctr,
                      cudaStream_t st);

// Lag statistics over a consumed batch (integer, bit-exact): hist[lag]++,
// per-sequence lag sums, max lag, total lag.  See sim.cpp:63-87.
void launch_lag_stats(const int32_t* versions, const int64_t* seq_offsets, int n_seq,
                      int version_before, int64_t* hist, int hist_cap, int64_t* seq_lag_sums,
                      int64_t* totals /* [0]=tokens [1]=lag_sum [2]=max_lag [3]=bad */,
                      cudaStream_t st);

}  // namespace srl
