// train.cuh -- trainer-side kernels of the decoder policy: the fused
// truncated-IS policy-gradient loss -> dlogits, and the backward pieces that
// are not GEMMs (transposes feeding the K-major tcgen05 GEMM, RMSNorm,
// SwiGLU, RoPE and causal-attention backward, bias/embedding gradients) plus
// the Adam update.  See trainer.cpp for how they compose.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace srl {

// dst[c, r] = bf16(src[r, c]) for a row-major [rows x cols] source.
// dst row stride is ld_dst (>= rows; padding columns are left untouched).
void launch_transpose_bf16(const __nv_bfloat16* src, int rows, int cols, __nv_bfloat16* dst,
                           int ld_dst, cudaStream_t st);
void launch_transpose_f32_bf16(const float* src, int rows, int cols, __nv_bfloat16* dst,
                               int ld_dst, cudaStream_t st);
// dst[r, :] = bf16(scale[r] * src[r, :]) then transposed (xn^T for weight gradients).
void launch_scale_transpose_bf16(const __nv_bfloat16* src, const float* row_scale, int rows,
                                 int cols, __nv_bfloat16* dst, int ld_dst, cudaStream_t st);
// dst[r, :] = bf16(scale[r] * src[r, :]) (xn for the MN-major weight gradients); cols % 8 == 0.
void launch_scale_rows_bf16(const __nv_bfloat16* src, const float* row_scale, int rows, int cols,
                            __nv_bfloat16* dst, cudaStream_t st);
// act[t, j] = bf16(silu(g) * u) from the interleaved fp32 gate|up pre-activations.
void launch_swiglu_fwd(const float* gu, int T, int I, __nv_bfloat16* act, cudaStream_t st);
void launch_f32_to_bf16(const float* src, size_t n, __nv_bfloat16* dst, cudaStream_t st);
void launch_bf16_to_f32(const __nv_bfloat16* src, size_t n, float* dst, cudaStream_t st);
void launch_zero(float* p, size_t n, cudaStream_t st);

// Per row r: lse from the EPI_LOGITS tile partials, logprob[r] =
// logits[r, tgt] - lse (fp64), dlogits[r, :] = coef[r] * (onehot(tgt) -
// softmax) in bf16 -- the gradient of J = sum_r coef[r] * log pi(tgt_r) w.r.t.
// the logits (rl_math.cpp:239-256 for one row).
// lse and log pi(target) per row from the LM-head epilogue's tile partials.
void launch_lse_logprob(const float* pmax, const double* psum, int V, int rows, const float* tgt_logit,
                        double* lse, double* logprob, cudaStream_t st);
void launch_loss_dlogits(const float* logits, const float* pmax, const double* psum, int V,
                         int rows, const int32_t* targets, const float* coef, double* logprob,
                         __nv_bfloat16* dlogits, cudaStream_t st);

// RMSNorm backward for y = rstd(x) * (x . g) W^T with dzw = dy W:
//   du = rstd * dzw ; drstd = sum_k dzw * x_k g_k
//   dx += du . g - rstd^3 / H * drstd * x ;  dg += sum_rows du . x
// prescaled: dzw already carries the row's rstd (dzw' = rstd * dy W, the
// trainer's precise mode folds rstd into dy): du = dzw'.
void launch_rmsnorm_bwd(const float* dzw, const float* x, const __nv_bfloat16* g,
                        const float* rstd, int T, int H, float* dx, float* dg, cudaStream_t st,
                        bool prescaled = false);
// Split bf16 pair of v = src[r, c] * row_scale[r] * col_gain[c] (either may be
// null): dst row r = [hi (cols) | lo (cols)], hi = bf16(v), lo = bf16(v - hi).
// cols % 4 == 0.
void launch_split_bf16(const float* src, int rows, int cols, const float* row_scale,
                       const __nv_bfloat16* col_gain, __nv_bfloat16* dst, cudaStream_t st);
// rstd[t] = 1/sqrt(mean(x^2) + eps)
void launch_row_rstd(const float* x, int T, int H, float eps, float* rstd, cudaStream_t st);

// SwiGLU backward (interleaved 64-col gate|up blocks): dgu = d[silu(g) u];
// gu in the token-blocked layout (gemm.cuh gu_index), dgu row-major.
void launch_swiglu_bwd(const float* dact, const __nv_bfloat16* gu, int T, int I, __nv_bfloat16* dgu,
                       float* dgu_f32, cudaStream_t st);

// Attention backward (causal, paged K/V as in the forward).  dq/dk/dv are
// written into dqkv [T x (nq+2nkv)hd] fp32 (pre-RoPE rotation applied after).
void launch_attention_bwd(const __nv_bfloat16* q, const __nv_bfloat16* o, const float* d_o,
                          const float* lse, const __nv_bfloat16* kc, const __nv_bfloat16* vc,
                          const int32_t* row_slot, const int32_t* row_pos,
                          const int32_t* seq_start, const int32_t* seq_len,
                          const int32_t* block_table, int pages_per_seq, int T, int n_seq, int nq,
                          int nkv, int hd, float* dqkv, cudaStream_t st, bool split = false);
// Causal attention forward over packed sequences on the tensor cores
// (train_attn.cu): O [T x nq*hd] bf16 and lse [T x nq] (scaled scores).
cudaError_t launch_attention_fwd_mma(const __nv_bfloat16* q, const __nv_bfloat16* kc, const __nv_bfloat16* vc,
                                     const int32_t* seq_start, const int32_t* seq_len,
                                     const int32_t* block_table, int pages_per_seq, int n_seq, int nq,
                                     int nkv, int hd, __nv_bfloat16* out, float* lse, cudaStream_t st,
                                     const int32_t* seg_pos0 = nullptr, const int32_t* seg_slot = nullptr,
                                     int max_rows = 0, int out_lo = 0);
// The tensor-core path of the above (train_attn.cu); D = rowsum(dO * O).
cudaError_t launch_attention_bwd_mma(const __nv_bfloat16* q, const __nv_bfloat16* dob, const __nv_bfloat16* dol,
                                     const float* lse, const float* D, const __nv_bfloat16* kc,
                                     const __nv_bfloat16* vc, const int32_t* seq_start, const int32_t* seq_len,
                                     const int32_t* block_table, int pages_per_seq, int n_seq, int nq,
                                     int nkv, int hd, float* dqkv, cudaStream_t st, bool split = false);
// Undo RoPE on the q/k part of dqkv in place (rotation by -angle).
void launch_rope_bwd(float* dqkv, const int32_t* row_pos, const float* cos_sin, int T, int nq,
                     int nkv, int hd, cudaStream_t st);

// out[n] += sum_rows src[r, n] (column sums, fp32)
void launch_colsum_accum(const float* src, int rows, int cols, float* out, cudaStream_t st);
// dE[tok[r], :] += dx[r, :]
void launch_embed_bwd(const float* dx, const int32_t* tokens, int T, int H, float* dE,
                      cudaStream_t st);

// Adam (ascent when sign = +1): m,v fp32; master fp32; w bf16 (the broadcast payload).
void launch_adam(float* master, __nv_bfloat16* w, const float* grad, float* m, float* v, size_t n,
                 float lr, float beta1, float beta2, float eps, float bias1, float bias2,
                 float sign, cudaStream_t st);

}  // namespace srl
