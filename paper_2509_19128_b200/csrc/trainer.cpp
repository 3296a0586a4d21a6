// trainer.cpp -- trainer-side device computations of the decoder policy.
//
//  * decoder_policy_logprobs: per-token current-policy log-prob recompute
//    (rl_math.cpp:128-142) as a chunked varlen forward.
//  * DecoderTrainer: one truncated-IS REINFORCE step (rl_math.cpp:211-276
//    generalised from tabular logits to the decoder's parameters):
//      forward over the packed batch, saving activations
//      pass 1: LM head -> log pi(y_t) for every row (fp64)
//      IS weights: w = min(c, exp(sum lp - sum mu)) per sequence, or per token
//      coef_t = (1/m) * w * A_t  (m = number of trajectories, stop-gradient on w)
//      pass 2: LM head again per row chunk -> dlogits = coef (onehot - softmax)
//      backward through the layers (tcgen05 GEMMs reading MN-major operands in
//      place for dX = dY W and dW = dY^T X, the SwiGLU backward fused into the
//      dact GEMM's epilogue, tensor-core (mma.sync) attention backward, per-row
//      RMSNorm / RoPE backward) into one fp32 gradient buffer laid out like
//      the weights -- the ascent direction of J, as in the reference.
//  * precise mode (default): every activation and backward operand a bf16
//    hi + lo pair (K-segmented GEMMs, split epilogues); fast mode: single bf16.
//  * Adam on fp32 master weights writes the bf16 weights that the generator
//    receives (ncclBroadcast payload).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "decoder_engine.hpp"
#include "train.cuh"
#include "trainer.hpp"

namespace srl {

int decoder_policy_logprobs(const DecoderWeights& w, const std::vector<int32_t>& tokens,
                            std::vector<double>& out) {
  const int n = (int)tokens.size();
  out.assign(n, 0.0);
  if (n == 0) return SRL_OK;
  if (n + 1 > w.dims.max_pos) return fail(SRL_INVALID_ARGUMENT, "sequence longer than max_positions");
  SRL_CUDA(cudaSetDevice(w.device));
  cudaStream_t st = nullptr;
  SRL_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  const int chunk = std::min(n, 512);
  DecoderRunner r;
  int status = r.init(w.dims, w.layout, 1, n + 1, chunk, chunk, w.device, st);
  if (status != SRL_OK) { cudaStreamDestroy(st); return status; }
  const WeightMaps maps = build_weight_maps(w.dims, w.layout, w.w);
  int32_t* dtarget = nullptr;
  double* dout = nullptr;
  SRL_CUDA(cudaMalloc(&dtarget, 4 * (size_t)n));
  SRL_CUDA(cudaMalloc(&dout, 8 * (size_t)n));
  SRL_CUDA(cudaMemcpy(dtarget, tokens.data(), 4 * (size_t)n, cudaMemcpyHostToDevice));
  std::vector<int32_t> rs(chunk, 0), rp(chunk), rt(chunk);
  for (int c0 = 0; c0 < n && status == SRL_OK; c0 += chunk) {
    const int M = std::min(chunk, n - c0);
    for (int i = 0; i < M; ++i) {
      const int p = c0 + i;
      rp[i] = p;
      rt[i] = p == 0 ? w.dims.bos : tokens[p - 1];  // input at position p predicts tokens[p]
    }
    cudaMemcpyAsync(r.plan.row_slot, rs.data(), 4 * (size_t)M, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(r.plan.row_pos, rp.data(), 4 * (size_t)M, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(r.plan.row_token, rt.data(), 4 * (size_t)M, cudaMemcpyHostToDevice, st);
    if ((status = r.forward(M, w.w, maps)) != SRL_OK) break;
    if ((status = r.lm_head(M, maps, false)) != SRL_OK) break;
    launch_row_logprobs(r.logits, w.dims.V, M, dtarget + c0, dout + c0, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) status = cuda_fail(cudaGetLastError(), "logprobs");
  }
  if (status == SRL_OK) {
    if (cudaMemcpy(out.data(), dout, 8 * (size_t)n, cudaMemcpyDeviceToHost) != cudaSuccess)
      status = cuda_fail(cudaGetLastError(), "logprobs copy");
  }
  cudaFree(dtarget);
  cudaFree(dout);
  cudaStreamDestroy(st);
  return status;
}

// ----------------------------------------------------------- trainer ---
namespace {
// rows per LM-head pass: the logits chunk is [chunk x V] fp32.  Large chunks
// keep the LM-head GEMMs efficient and, above all, accumulate the [V x H] fp32
// LM-head gradient (a read-modify-write of 0.5 GB at V = 152k) few times.
constexpr int kLogitChunkMax = 16384;
constexpr int kTileFlags = 4096;
int pad64(int x) { return (x + 63) / 64 * 64; }
}  // namespace

DecoderTrainer::~DecoderTrainer() {
  if (st_) cudaStreamSynchronize(st_);
  for (void* p : allocs_) cudaFree(p);
  if (ws_) cudaFree(ws_);
  if (kc_) cudaFree(kc_);
  if (vc_) cudaFree(vc_);
  if (st_) cudaStreamDestroy(st_);
}

template <typename T>
int DecoderTrainer::alloc(T** p, size_t n) {
  SRL_CUDA(cudaMalloc(p, std::max<size_t>(n, 1) * sizeof(T)));
  SRL_CUDA(cudaMemsetAsync(*p, 0, std::max<size_t>(n, 1) * sizeof(T), st_));
  allocs_.push_back(*p);
  return SRL_OK;
}

int DecoderTrainer::init(const DecoderWeights& w, const srl_trainer_options& o) {
  opts_ = o;
  d_ = w.dims;
  dev_ = o.device >= 0 ? o.device : w.device;  // the trainer lives on opts.device
  SRL_CUDA(cudaSetDevice(dev_));
  SRL_CUDA(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
  {  // the step's stream-ordered scratch (block tables, attention partials) stays
     // mapped between steps instead of returning to the driver at every sync
    cudaMemPool_t pool;
    uint64_t keep = UINT64_MAX;
    if (cudaDeviceGetDefaultMemPool(&pool, dev_) == cudaSuccess)
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  int st;
  if ((st = clone_decoder(w, weights_, dev_))) return st;
  lay_ = weights_->layout;
  n_ = lay_.total;
  T_max_ = pad64(std::max(64, o.max_tokens));
  chunk_ = std::min(o.logit_chunk > 0 ? pad64(o.logit_chunk) : kLogitChunkMax, T_max_);
  precise_ = o.fast_bf16 == 0;
  sp_ = precise_ ? 2 : 1;
  if (precise_ && (d_.H % 64 || d_.I % 64 || d_.qdim() % 64 || d_.qkv() % 64 || d_.V % 64))
    return fail(SRL_INVALID_ARGUMENT, "trainer: precise mode needs every width a multiple of 64");
  const int H = d_.H, L = d_.L, I = d_.I, qd = d_.qdim(), qkv = d_.qkv();
  // fp32 master weights, Adam moments, gradient
  if ((st = alloc(&master_, n_)) || (st = alloc(&grad_, n_)) || (st = alloc(&adam_m_, n_)) ||
      (st = alloc(&adam_v_, n_)) || (st = alloc(&tile_flags_, kTileFlags)))
    return st;
  SRL_CUDA(cudaMemsetAsync(tile_flags_, 0, sizeof(int) * kTileFlags, st_));
  launch_bf16_to_f32(weights_->w, n_, master_, st_);
  // saved activations
  acts_.resize(L);
  for (int l = 0; l < L; ++l) {
    LayerActs& a = acts_[l];
    // split (precise) activations are [hi | lo] rows: sp_ x the width
    if ((st = alloc(&a.x_in, (size_t)T_max_ * H)) || (st = alloc(&a.xg1, (size_t)T_max_ * H * sp_)) ||
        (st = alloc(&a.rstd1, T_max_)) || (st = alloc(&a.q, (size_t)T_max_ * qd)) ||
        (st = alloc(&a.attn, (size_t)T_max_ * qd * sp_)) || (st = alloc(&a.lse, (size_t)T_max_ * d_.nq)) ||
        (st = alloc(&a.x_mid, (size_t)T_max_ * H)) || (st = alloc(&a.xg2, (size_t)T_max_ * H * sp_)) ||
        (st = alloc(&a.rstd2, T_max_)) || (st = alloc(&a.act, (size_t)T_max_ * I * sp_)))
      return st;
    const size_t gu_elems = gu_rows_padded((size_t)T_max_) * 2 * I;  // token-blocked (gemm.cuh gu_index)
    if (precise_ ? (st = alloc(&a.gu32, gu_elems)) : (st = alloc(&a.gu, gu_elems)))
      return st;
  }
  if ((st = alloc(&x_, (size_t)T_max_ * H)) || (st = alloc(&xgF_, (size_t)T_max_ * H * sp_)) ||
      (st = alloc(&rstdF_, T_max_)) || (st = alloc(&ssq_, (size_t)T_max_ * d_.ssq_parts())) ||
      (st = alloc(&pmax_, (size_t)chunk_ * ((d_.V + 127) / 128))) ||
      (st = alloc(&psum_, (size_t)chunk_ * ((d_.V + 127) / 128))) ||
      (st = alloc(&dlogits_, (size_t)chunk_ * d_.V * sp_)) || (st = alloc(&dx_, (size_t)T_max_ * H)) ||
      (st = alloc(&dz_, (size_t)T_max_ * std::max(H, 2 * I))) ||
      (st = alloc(&dbig_, (size_t)T_max_ * std::max({2 * I, qkv, qd}))) ||
      (st = alloc(&dbig_bf_, (size_t)T_max_ * std::max({2 * I, qkv, qd, H}) * sp_)) ||
      (st = alloc(&xn_, (size_t)T_max_ * H)) || (st = alloc(&dgu_, (size_t)T_max_ * 2 * I * sp_)) ||
      (st = alloc(&ones_, T_max_)) || (st = alloc(&row_slot_, T_max_)) ||
      (st = alloc(&row_pos_, T_max_)) || (st = alloc(&row_tok_, T_max_)) ||
      (st = alloc(&row_tgt_, T_max_)) || (st = alloc(&coef_, T_max_)) ||
      (st = alloc(&lp_, T_max_)) || (st = alloc(&lse_, T_max_)) || (st = alloc(&tgt_logit_, T_max_)) || (st = alloc(&cos_sin_, (size_t)d_.max_pos * d_.hd)))
    return st;
  launch_rope_table(cos_sin_, d_.max_pos, d_.hd, (double)d_.theta, st_);
  std::vector<float> ones(T_max_, 1.f);
  SRL_CUDA(cudaMemcpyAsync(ones_, ones.data(), 4 * (size_t)T_max_, cudaMemcpyHostToDevice, st_));
  SRL_CUDA(cudaStreamSynchronize(st_));
  sms_ = 148;
  cudaDeviceGetAttribute(&sms_, cudaDevAttrMultiProcessorCount, dev_);
  return SRL_OK;
}

void DecoderTrainer::apply_seg(EpiParams& e, const Seg* seg, int K) {
  if (seg == nullptr || seg->n <= 1) return;
  e.seg_kb = K / 64;
  e.x_off0 = seg->x_off[0]; e.x_off1 = seg->x_off[1]; e.x_off2 = seg->x_off[2];
  e.w_off0 = seg->w_off[0]; e.w_off1 = seg->w_off[1]; e.w_off2 = seg->w_off[2];
}

// C[m, n] (epilogue) = sum_k X[m, k] * W[n, k]; X, W bf16 K-major.  Precise
// mode: X rows are [hi (K) | lo (K)] and the persistent kernel runs the two
// K segments (hi W + lo W) into one accumulator.
int DecoderTrainer::gemm(const __nv_bfloat16* X, int x_rows_alloc, int M, const __nv_bfloat16* W,
                         int N, int K, const EpiParams& e) {
  if (precise_) {
    const CUtensorMap tx = make_tmap_bf16(X, (uint64_t)std::max(x_rows_alloc, M), (uint64_t)(2 * K), 128);
    const CUtensorMap tw = make_tmap_bf16(W, (uint64_t)N, (uint64_t)K, 128);
    EpiParams es = e;
    const Seg sg = seg_x(K);
    apply_seg(es, &sg, K);
    int tok = gemm_big_tok(M, N, 2 * K, sms_);
    if (tok == 0) tok = 128;
    const cudaError_t err = gemm_big_launch(tw, tx, M, N, 2 * K, tok, es, st_);
    if (err != cudaSuccess) return cuda_fail(err, "trainer gemm (split)");
    return SRL_OK;
  }
  const int tok = gemm_tok_tile(M);
  const CUtensorMap tx = make_tmap_bf16(X, (uint64_t)std::max(x_rows_alloc, M), (uint64_t)K, (uint32_t)tok);
  const CUtensorMap tw = make_tmap_bf16(W, (uint64_t)N, (uint64_t)K, 128);
  const int splits = gemm_auto_splits(M, N, K, sms_);
  const size_t need = gemm_workspace_floats(M, N, splits);
  if (need > ws_floats_) {
    if (ws_) cudaFree(ws_);
    SRL_CUDA(cudaMalloc(&ws_, need * sizeof(float)));
    ws_floats_ = need;
  }
  GemmWorkspace ws;
  ws.partials = ws_;
  ws.partial_floats = ws_floats_;
  const cudaError_t err = gemm_bf16_launch(tw, tx, M, N, K, splits, ws, e, st_);
  if (err != cudaSuccess) return cuda_fail(err, "trainer gemm");
  return SRL_OK;
}

int DecoderTrainer::gemm_store(const __nv_bfloat16* X, int M, const __nv_bfloat16* W, int N, int K,
                               float* out) {
  EpiParams e;
  e.kind = EPI_STORE_F32;
  e.out_f32 = out;
  e.ld_out = N;
  return gemm(X, M, M, W, N, K, e);
}

int DecoderTrainer::gemm_accum(const __nv_bfloat16* X, int M, const __nv_bfloat16* W, int N, int K,
                               float* out) {
  EpiParams e;
  e.kind = EPI_ACCUM_F32;
  e.out_f32 = out;
  e.ld_out = N;
  return gemm(X, M, M, W, N, K, e);
}

// C[m, n] (+)= sum_k X(m, k) W[k, n] with W MN-major ([k_rows x N] row-major:
// an activation with tokens as K, or a weight matrix used as dX = dY W) and X
// MN-major [k_rows x M] or K-major [M x k_rows] -- no transposed copies.
// dgu = SwiGLU'(gu) applied to dact = dY W (W MN-major [k_rows x I]): fused
// into the GEMM epilogue when the plan needs no K slices, else through dz_.
int DecoderTrainer::gemm_swiglu_bwd(const __nv_bfloat16* dY, int M, const __nv_bfloat16* W, int I, int k_rows,
                                    const __nv_bfloat16* gu, __nv_bfloat16* dgu, const LayerActs* a) {
  const int K = pad64(k_rows);
  if (precise_) {
    // dact = (dYh + dYl) W_down, SwiGLU backward on the fp32 gate | up with
    // rstd2 folded in, dgu' written as [hi (2I) | lo (2I)] rows
    const Seg sg = seg_x(k_rows);
    const CUtensorMap tw = make_tmap_bf16(W, (uint64_t)k_rows, (uint64_t)I, 64);
    const CUtensorMap tx = make_tmap_bf16(dY, (uint64_t)M, (uint64_t)(2 * k_rows), 128);
    int splits = 1;
    const int tok = gemm_mn_plan(M, I, 2 * K, sms_, &splits);
    EpiParams e;
    e.kind = EPI_SWIGLU_BWD;
    e.gu_in_f32 = a->gu32;
    e.row_scale = a->rstd2;
    e.out_bf16 = dgu;
    e.ld_bf16 = 4 * I;
    e.lo_off = 2 * I;
    apply_seg(e, &sg, K);
    const cudaError_t err = gemm_mn_launch(tw, tx, M, I, 2 * K, tok, 1, false, e, st_);
    if (err != cudaSuccess) return cuda_fail(err, "trainer gemm_swiglu_bwd (split)");
    return SRL_OK;
  }
  int splits = 1;
  const int tok = gemm_mn_plan(M, I, K, sms_, &splits);
  if (splits > 1) {
    int s = gemm_mn(dY, true, M, W, I, k_rows, dz_, false);
    if (s) return s;
    launch_swiglu_bwd(dz_, gu, M, I, dgu, nullptr, st_);
    return SRL_OK;
  }
  const CUtensorMap tw = make_tmap_bf16(W, (uint64_t)k_rows, (uint64_t)I, 64);
  const CUtensorMap tx = make_tmap_bf16(dY, (uint64_t)M, (uint64_t)k_rows, 128);
  EpiParams e;
  e.kind = EPI_SWIGLU_BWD;
  e.gu_in = gu;
  e.out_bf16 = dgu;
  e.ld_bf16 = 2 * I;
  const cudaError_t err = gemm_mn_launch(tw, tx, M, I, K, tok, 1, false, e, st_);
  if (err != cudaSuccess) return cuda_fail(err, "trainer gemm_swiglu_bwd");
  return SRL_OK;
}

int DecoderTrainer::gemm_mn(const __nv_bfloat16* X, bool x_kmajor, int M, const __nv_bfloat16* W, int N,
                            int k_rows, float* out, bool accumulate, const Seg* seg) {
  const int K = pad64(k_rows);
  const int nseg = seg ? seg->n : 1;
  if (nseg > 1 && x_kmajor && k_rows % 64 != 0)
    return fail(SRL_INVALID_ARGUMENT, "trainer gemm_mn: split K-major operand needs K % 64 == 0");
  const uint64_t wc = seg && seg->w_cols ? seg->w_cols : N;
  const uint64_t xc = seg && seg->x_cols ? seg->x_cols : (x_kmajor ? k_rows : M);
  const CUtensorMap tw = make_tmap_bf16(W, (uint64_t)k_rows, wc, 64);
  const CUtensorMap tx = x_kmajor ? make_tmap_bf16(X, (uint64_t)M, xc, 128)
                                  : make_tmap_bf16(X, (uint64_t)k_rows, xc, 64);
  int splits = 1;
  const int tok = gemm_mn_plan(M, N, K * nseg, sms_, &splits);
  if ((size_t)((N + 127) / 128) * ((M + tok - 1) / tok) > (size_t)kTileFlags) splits = 1;
  if (splits > 1 && !accumulate) {  // ordered K slices add into a zeroed output
    SRL_CUDA(cudaMemsetAsync(out, 0, sizeof(float) * (size_t)M * N, st_));
    accumulate = true;
  }
  EpiParams e;
  e.kind = accumulate ? EPI_ACCUM_F32 : EPI_STORE_F32;
  e.out_f32 = out;
  e.ld_out = N;
  e.tile_flags = tile_flags_;
  apply_seg(e, seg, K);
  const cudaError_t err = gemm_mn_launch(tw, tx, M, N, K * nseg, tok, splits, !x_kmajor, e, st_);
  if (err != cudaSuccess) return cuda_fail(err, "trainer gemm_mn");
  return SRL_OK;
}

int DecoderTrainer::step(const TrainBatch& b, srl_trainer_stats* stats) {
  const int T = b.rows, Tp = pad64(T);
  if (T < 1 || Tp > T_max_) return fail(SRL_INVALID_ARGUMENT, "trainer: batch exceeds max_tokens");
  const int H = d_.H, I = d_.I, L = d_.L, qd = d_.qdim(), qkv = d_.qkv(), V = d_.V;
  const int parts = d_.ssq_parts();
  const float inv_h = 1.f / (float)H;
  const __nv_bfloat16* w = weights_->w;
  cudaStream_t st = st_;
  SRL_CUDA(cudaSetDevice(dev_));
  int s;

  // ---- batch layout: rows (seq, pos); KV pages per sequence
  const int n_seq = (int)b.seq_len.size();
  int pps = 1;
  for (int l : b.seq_len) pps = std::max(pps, (l + kPageTokens - 1) / kPageTokens);
  const size_t n_pages = (size_t)n_seq * pps;
  const size_t kv_elems = n_pages * d_.nkv * kPageTokens * d_.hd;
  if (kv_elems * L > kv_cap_) {
    if (kc_) { cudaFree(kc_); cudaFree(vc_); }
    SRL_CUDA(cudaMalloc(&kc_, kv_elems * L * 2));
    SRL_CUDA(cudaMalloc(&vc_, kv_elems * L * 2));
    kv_cap_ = kv_elems * L;
  }
  std::vector<int32_t> bt(n_pages);
  for (size_t i = 0; i < n_pages; ++i) bt[i] = (int32_t)i;
  int32_t *d_bt = nullptr, *d_sstart = nullptr, *d_slen = nullptr;
  SRL_CUDA(cudaMallocAsync(&d_bt, 4 * n_pages, st));
  SRL_CUDA(cudaMallocAsync(&d_sstart, 4 * (size_t)n_seq, st));
  SRL_CUDA(cudaMallocAsync(&d_slen, 4 * (size_t)n_seq, st));
  SRL_CUDA(cudaMemcpyAsync(d_bt, bt.data(), 4 * n_pages, cudaMemcpyHostToDevice, st));
  SRL_CUDA(cudaMemcpyAsync(d_sstart, b.seq_start.data(), 4 * (size_t)n_seq, cudaMemcpyHostToDevice, st));
  SRL_CUDA(cudaMemcpyAsync(d_slen, b.seq_len.data(), 4 * (size_t)n_seq, cudaMemcpyHostToDevice, st));
  SRL_CUDA(cudaMemcpyAsync(row_slot_, b.row_slot.data(), 4 * (size_t)T, cudaMemcpyHostToDevice, st));
  SRL_CUDA(cudaMemcpyAsync(row_pos_, b.row_pos.data(), 4 * (size_t)T, cudaMemcpyHostToDevice, st));
  SRL_CUDA(cudaMemcpyAsync(row_tok_, b.row_token.data(), 4 * (size_t)T, cudaMemcpyHostToDevice, st));
  SRL_CUDA(cudaMemcpyAsync(row_tgt_, b.row_target.data(), 4 * (size_t)T, cudaMemcpyHostToDevice, st));

  cudaEvent_t e0, e1, e2;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventCreate(&e2);
  cudaEventRecord(e0, st);

  // ---- forward with saved activations
  const bool P = precise_;
  if (P) {  // xg1 of layer 0 as the split pair of x * ln1 (the embed kernel's bf16 xg is scratch)
    launch_embed(w + lay_.embed, w + lay_.layers[0].ln1, row_tok_, T, H, V, x_, xn_, ssq_, st);
    launch_split_bf16(x_, T, H, nullptr, w + lay_.layers[0].ln1, acts_[0].xg1, st);
  } else {
    launch_embed(w + lay_.embed, w + lay_.layers[0].ln1, row_tok_, T, H, V, x_, acts_[0].xg1, ssq_, st);
  }
  for (int l = 0; l < L; ++l) {
    LayerActs& a = acts_[l];
    const LayerOffsets& o = lay_.layers[l];
    SRL_CUDA(cudaMemcpyAsync(a.x_in, x_, sizeof(float) * T * H, cudaMemcpyDeviceToDevice, st));
    launch_row_rstd(a.x_in, T, H, d_.eps, a.rstd1, st);
    __nv_bfloat16* kcl = kc_ + kv_elems * l;
    __nv_bfloat16* vcl = vc_ + kv_elems * l;
    EpiParams e;
    e.kind = EPI_QKV;
    e.ssq_in = ssq_; e.ssq_in_parts = parts; e.inv_dim = inv_h; e.eps = d_.eps;
    e.bias = w + o.qkv_b;
    e.nq = d_.nq; e.nkv = d_.nkv; e.hd = d_.hd; e.pages_per_seq = pps;
    e.row_slot = row_slot_; e.row_pos = row_pos_; e.block_table = d_bt; e.cos_sin = cos_sin_;
    e.q_out = a.q; e.kc = kcl; e.vc = vcl;
    if ((s = gemm(a.xg1, T_max_, T, w + o.qkv_w, qkv, H, e))) return s;
    static const bool scalar_fwd = std::getenv("SRL_ATTN_FWD_SCALAR") != nullptr;  // A/B switch
    if (!scalar_fwd || P) {
      SRL_CUDA(launch_attention_fwd_mma(a.q, kcl, vcl, d_sstart, d_slen, d_bt, pps, n_seq, d_.nq, d_.nkv,
                                        d_.hd, a.attn, a.lse, st, nullptr, nullptr, 0, P ? qd : 0));
    } else {
    RoundPlan plan{row_slot_, row_pos_, row_tok_, nullptr};
    float* attn_ws = nullptr;
    int* attn_cnt = nullptr;
    const size_t aws = attention_ws_floats(d_, T, d_.max_pos);
    SRL_CUDA(cudaMallocAsync(&attn_ws, sizeof(float) * aws, st));
    SRL_CUDA(cudaMallocAsync(&attn_cnt, sizeof(int) * (size_t)T * d_.nkv, st));
    SRL_CUDA(cudaMemsetAsync(attn_cnt, 0, sizeof(int) * (size_t)T * d_.nkv, st));
    int max_ctx = 1;
    for (int len : b.seq_len) max_ctx = std::max(max_ctx, len);
    launch_attention(a.q, d_, plan, T, d_bt, pps, kcl, vcl, max_ctx, attn_ws, attn_cnt, aws, a.attn,
                     st, a.lse);
    cudaFreeAsync(attn_ws, st);
    cudaFreeAsync(attn_cnt, st);
    }
    EpiParams r;
    r.kind = EPI_RESID; r.resid = x_; r.gain = w + o.ln2; r.xg = a.xg2; r.ssq_out = ssq_;
    r.lo_off = P ? H : 0;
    if ((s = gemm(a.attn, T_max_, T, w + o.o_w, H, qd, r))) return s;
    SRL_CUDA(cudaMemcpyAsync(a.x_mid, x_, sizeof(float) * T * H, cudaMemcpyDeviceToDevice, st));
    launch_row_rstd(a.x_mid, T, H, d_.eps, a.rstd2, st);
    EpiParams g;  // SwiGLU fused: act for the down GEMM, gate | up kept (bf16) for the backward
    g.kind = EPI_SWIGLU;
    g.ssq_in = ssq_; g.ssq_in_parts = parts; g.inv_dim = inv_h; g.eps = d_.eps;
    g.out_bf16 = a.act; g.ld_bf16 = I * sp_; g.lo_off = P ? I : 0;
    g.out2_bf16 = a.gu; g.out2_f32 = a.gu32;
    if ((s = gemm(a.xg2, T_max_, T, w + o.gate_up_w, 2 * I, H, g))) return s;
    EpiParams r2;
    r2.kind = EPI_RESID; r2.resid = x_; r2.ssq_out = ssq_; r2.lo_off = P ? H : 0;
    r2.xg = l + 1 < L ? acts_[l + 1].xg1 : xgF_;
    r2.gain = w + (l + 1 < L ? lay_.layers[l + 1].ln1 : lay_.final_norm);
    if ((s = gemm(a.act, T_max_, T, w + o.down_w, H, I, r2))) return s;
  }
  launch_row_rstd(x_, T, H, d_.eps, rstdF_, st);

  // ---- pass 1: log pi(target) of every row
  const int nT = (V + 127) / 128;
  // LM-head row chunks of equal size (<= chunk_, a multiple of 256): a short
  // tail chunk ran at half the rate of a full one
  const int n_chunks = (T + chunk_ - 1) / chunk_;
  const int cb = std::min(chunk_, ((T + n_chunks - 1) / n_chunks + 255) / 256 * 256);
  for (int c0 = 0; c0 < T; c0 += cb) {
    const int C = std::min(cb, T - c0);
    EpiParams e;
    e.kind = EPI_LOGITS;
    e.ssq_in = ssq_ + (size_t)c0 * parts; e.ssq_in_parts = parts; e.inv_dim = inv_h; e.eps = d_.eps;
    // statistics and the target's logit only: the [C x V] logits are never stored
    e.out_f32 = nullptr; e.part_max = pmax_; e.part_sum = psum_;
    e.tgt_row = row_tgt_ + c0; e.tgt_out = tgt_logit_ + c0;
    if ((s = gemm(xgF_ + (size_t)c0 * H * sp_, C, C, w + lay_.lm_head, V, H, e))) return s;
    launch_lse_logprob(pmax_, psum_, V, C, tgt_logit_ + c0, lse_ + c0, lp_ + c0, st);
  }
  cudaEventRecord(e1, st);
  std::vector<double> lp(T);
  SRL_CUDA(cudaMemcpyAsync(lp.data(), lp_, 8 * (size_t)T, cudaMemcpyDeviceToHost, st));
  SRL_CUDA(cudaStreamSynchronize(st));

  // ---- truncated IS weights and per-row coefficients (host: O(tokens) scalars)
  std::vector<float> coef(T, 0.f);
  const double inv_m = 1.0 / (double)std::max(1, b.n_trajectories);
  std::vector<double> seq_w(n_seq, 1.0);
  double loss = 0.0, ess_num = 0.0, ess_den = 0.0;
  int clamped = 0;
  for (int q = 0; q < n_seq; ++q) {
    double pi = 0.0, mu = 0.0;
    for (int p = b.loss_begin[q]; p < b.seq_len[q]; ++p) {
      pi += lp[b.seq_start[q] + p];
      mu += b.row_mu[b.seq_start[q] + p];
    }
    if (b.granularity == 0) {
      const double r = std::exp(pi - mu);
      seq_w[q] = std::min(b.clamp, r);  // truncated_is_weight (rl_math.cpp:144-150)
      if (r > b.clamp) ++clamped;
      ess_num += seq_w[q];
      ess_den += seq_w[q] * seq_w[q];
    }
    for (int p = b.loss_begin[q]; p < b.seq_len[q]; ++p) {
      const int row = b.seq_start[q] + p;
      double wgt = seq_w[q];
      if (b.granularity == 1) {
        const double r = std::exp(lp[row] - b.row_mu[row]);
        wgt = std::min(b.clamp, r);
        if (r > b.clamp) ++clamped;
        ess_num += wgt;
        ess_den += wgt * wgt;
      }
      const double c = inv_m * wgt * b.row_adv[row];
      coef[row] = (float)c;
      loss += c * lp[row];
    }
  }
  SRL_CUDA(cudaMemcpyAsync(coef_, coef.data(), 4 * (size_t)T, cudaMemcpyHostToDevice, st));

  // ---- backward
  launch_zero(grad_, n_, st);
  launch_zero(dx_, (size_t)T_max_ * H, st);
  // Every backward GEMM reads its operands in place: weight gradients take
  // both operands MN-major (tokens as K), input gradients take W MN-major.
  // pass 2: dlogits per chunk -> d(final xg) and dE(lm_head)
  float* g_lm = grad_ + lay_.lm_head;
  for (int c0 = 0; c0 < T; c0 += cb) {
    const int C = std::min(cb, T - c0);
    // dlogits = coef (onehot - softmax) straight from the LM-head accumulator
    // (lse of pass 1: same weights, same logits)
    EpiParams e;
    e.kind = EPI_DLOGITS;
    e.ssq_in = ssq_ + (size_t)c0 * parts; e.ssq_in_parts = parts; e.inv_dim = inv_h; e.eps = d_.eps;
    e.lse_in = lse_ + c0; e.row_coef = coef_ + c0; e.tgt_row = row_tgt_ + c0;
    e.out_bf16 = dlogits_; e.ld_bf16 = V * sp_;
    if (P) {  // dlogits' = rstd * dlogits as [hi | lo] rows
      e.fold_rstd = 1;
      e.lo_off = V;
    }
    if ((s = gemm(xgF_ + (size_t)c0 * H * sp_, C, C, w + lay_.lm_head, V, H, e))) return s;
    if (P) {
      const Seg sx = seg_x(V), sxw = seg_xw(V, H);
      // dzw'[t, h] = sum_v dlogits'[t, v] E[v, h]  (rstd already in)
      if ((s = gemm_mn(dlogits_, true, C, w + lay_.lm_head, H, V, dz_, false, &sx))) return s;
      launch_rmsnorm_bwd(dz_, x_ + (size_t)c0 * H, w + lay_.final_norm, rstdF_ + c0, C, H,
                         dx_ + (size_t)c0 * H, grad_ + lay_.final_norm, st, true);
      // dE[v, h] += sum_t dlogits'[t, v] * u[t, h], u = x * final_norm (split)
      if ((s = gemm_mn(dlogits_, false, V, xgF_ + (size_t)c0 * H * 2, H, C, g_lm, true, &sxw))) return s;
      continue;
    }
    // dzw[t, h] = sum_v dlogits[t, v] E[v, h]
    if ((s = gemm_mn(dlogits_, true, C, w + lay_.lm_head, H, V, dz_, false))) return s;
    launch_rmsnorm_bwd(dz_, x_ + (size_t)c0 * H, w + lay_.final_norm, rstdF_ + c0, C, H,
                       dx_ + (size_t)c0 * H, grad_ + lay_.final_norm, st);
    // dE[v, h] += sum_t dlogits[t, v] * rstd[t] xg[t, h]
    launch_scale_rows_bf16(xgF_ + (size_t)c0 * H, rstdF_ + c0, C, H, xn_, st);
    if ((s = gemm_mn(dlogits_, false, V, xn_, H, C, g_lm, true))) return s;
  }
  // layers in reverse; dx_ holds dJ/dx_out of the layer being processed
  for (int l = L - 1; l >= 0 && P; --l) {
    // precise mode: every GEMM operand that is not a weight is a [hi | lo] pair;
    // rstd is folded into the dY of the normalised GEMMs (QKV, gate/up), whose
    // weight gradients then read the split u = x * gain directly
    LayerActs& a = acts_[l];
    const LayerOffsets& o = lay_.layers[l];
    const Seg sH = seg_x(H), s2I = seg_x(2 * I), sQKV = seg_x(qkv);
    const Seg dWd = seg_xw(H, I), dWgu = seg_xw(2 * I, H), dWo = seg_xw(H, qd), dWqkv = seg_xw(qkv, H);
    // down: x_out = x_mid + act W_down^T
    launch_split_bf16(dx_, T, H, nullptr, nullptr, dbig_bf_, st);                 // dY [T x 2H]
    if ((s = gemm_mn(dbig_bf_, false, H, a.act, I, T, grad_ + o.down_w, true, &dWd))) return s;
    if ((s = gemm_swiglu_bwd(dbig_bf_, T, w + o.down_w, I, H, nullptr, dgu_, &a))) return s;  // dgu' [T x 4I]
    // gate_up: gu = rstd2 * (u2 W_gu^T), rstd2 folded into dgu'
    if ((s = gemm_mn(dgu_, true, T, w + o.gate_up_w, H, 2 * I, dz_, false, &s2I))) return s;
    if ((s = gemm_mn(dgu_, false, 2 * I, a.xg2, H, T, grad_ + o.gate_up_w, true, &dWgu))) return s;
    launch_rmsnorm_bwd(dz_, a.x_mid, w + o.ln2, a.rstd2, T, H, dx_, grad_ + o.ln2, st, true);
    // O: x_mid = x_in + attn W_o^T
    launch_split_bf16(dx_, T, H, nullptr, nullptr, dbig_bf_, st);
    if ((s = gemm_mn(dbig_bf_, true, T, w + o.o_w, qd, H, dz_, false, &sH))) return s;          // dO [T x qd]
    if ((s = gemm_mn(dbig_bf_, false, H, a.attn, qd, T, grad_ + o.o_w, true, &dWo))) return s;
    launch_attention_bwd(a.q, a.attn, dz_, a.lse, kc_ + kv_elems * l, vc_ + kv_elems * l, row_slot_,
                         row_pos_, d_sstart, d_slen, d_bt, pps, T, n_seq, d_.nq, d_.nkv, d_.hd, dbig_, st,
                         true);
    launch_rope_bwd(dbig_, row_pos_, cos_sin_, T, d_.nq, d_.nkv, d_.hd, st);
    launch_colsum_accum(dbig_, T, qkv, grad_ + o.qkv_b, st);
    launch_split_bf16(dbig_, T, qkv, a.rstd1, nullptr, dbig_bf_, st);            // dqkv' = rstd1 dqkv
    if ((s = gemm_mn(dbig_bf_, true, T, w + o.qkv_w, H, qkv, dz_, false, &sQKV))) return s;
    if ((s = gemm_mn(dbig_bf_, false, qkv, a.xg1, H, T, grad_ + o.qkv_w, true, &dWqkv))) return s;
    launch_rmsnorm_bwd(dz_, a.x_in, w + o.ln1, a.rstd1, T, H, dx_, grad_ + o.ln1, st, true);
  }
  for (int l = L - 1; l >= 0 && !P; --l) {
    LayerActs& a = acts_[l];
    const LayerOffsets& o = lay_.layers[l];
    // down: x_out = x_mid + act W_down^T
    launch_f32_to_bf16(dx_, (size_t)T * H, dbig_bf_, st);                       // dY bf16 [T x H]
    if ((s = gemm_mn(dbig_bf_, false, H, a.act, I, T, grad_ + o.down_w, true))) return s;  // dW_down [H x I]
    // dact [T x I] = dY W_down, SwiGLU backward in its epilogue -> dgu bf16 [T x 2I]
    if ((s = gemm_swiglu_bwd(dbig_bf_, T, w + o.down_w, I, H, a.gu, dgu_))) return s;
    // gate_up: gu = rstd2 * (xg2 W_gu^T)
    if ((s = gemm_mn(dgu_, true, T, w + o.gate_up_w, H, 2 * I, dz_, false))) return s;  // dzw [T x H]
    launch_scale_rows_bf16(a.xg2, a.rstd2, T, H, xn_, st);                      // xn2 [T x H]
    if ((s = gemm_mn(dgu_, false, 2 * I, xn_, H, T, grad_ + o.gate_up_w, true))) return s;
    launch_rmsnorm_bwd(dz_, a.x_mid, w + o.ln2, a.rstd2, T, H, dx_, grad_ + o.ln2, st);
    // O: x_mid = x_in + attn W_o^T   (dx_ now = dJ/dx_mid)
    launch_f32_to_bf16(dx_, (size_t)T * H, dbig_bf_, st);
    if ((s = gemm_mn(dbig_bf_, true, T, w + o.o_w, qd, H, dz_, false))) return s;          // dO [T x qd]
    if ((s = gemm_mn(dbig_bf_, false, H, a.attn, qd, T, grad_ + o.o_w, true))) return s;   // dW_o [H x qd]
    // attention + RoPE backward -> dqkv (pre-RoPE, pre-bias) fp32
    launch_attention_bwd(a.q, a.attn, dz_, a.lse, kc_ + kv_elems * l, vc_ + kv_elems * l, row_slot_,
                         row_pos_, d_sstart, d_slen, d_bt, pps, T, n_seq, d_.nq, d_.nkv, d_.hd, dbig_, st);
    launch_rope_bwd(dbig_, row_pos_, cos_sin_, T, d_.nq, d_.nkv, d_.hd, st);
    launch_colsum_accum(dbig_, T, qkv, grad_ + o.qkv_b, st);
    launch_f32_to_bf16(dbig_, (size_t)T * qkv, dbig_bf_, st);
    if ((s = gemm_mn(dbig_bf_, true, T, w + o.qkv_w, H, qkv, dz_, false))) return s;     // dzw [T x H]
    launch_scale_rows_bf16(a.xg1, a.rstd1, T, H, xn_, st);
    if ((s = gemm_mn(dbig_bf_, false, qkv, xn_, H, T, grad_ + o.qkv_w, true))) return s;
    launch_rmsnorm_bwd(dz_, a.x_in, w + o.ln1, a.rstd1, T, H, dx_, grad_ + o.ln1, st);
  }
  launch_embed_bwd(dx_, row_tok_, T, H, grad_ + lay_.embed, st);
  cudaEventRecord(e2, st);
  cudaFreeAsync(d_bt, st);
  cudaFreeAsync(d_sstart, st);
  cudaFreeAsync(d_slen, st);
  SRL_CUDA(cudaStreamSynchronize(st));
  SRL_CUDA(cudaGetLastError());
  float fwd_ms = 0.f, all_ms = 0.f;
  cudaEventElapsedTime(&fwd_ms, e0, e1);
  cudaEventElapsedTime(&all_ms, e0, e2);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaEventDestroy(e2);
  if (stats) {
    stats->objective = loss;
    // ess over the IS weights actually used (rl_math.cpp:152-163)
    const double nw = b.granularity == 0 ? (double)n_seq : (double)b.n_loss_rows;
    stats->ess = (ess_den > 0 && nw > 0) ? (ess_num * ess_num) / (nw * ess_den) : 0.0;
    stats->clamped = clamped;
    stats->tokens = T;
    stats->forward_ms = fwd_ms;
    stats->step_ms = all_ms;
  }
  lp_host_ = std::move(lp);
  return SRL_OK;
}

int DecoderTrainer::apply_adam(float lr, float beta1, float beta2, float eps) {
  ++adam_t_;
  const float b1 = 1.f - std::pow(beta1, (float)adam_t_), b2 = 1.f - std::pow(beta2, (float)adam_t_);
  launch_adam(master_, weights_->w, grad_, adam_m_, adam_v_, n_, lr, beta1, beta2, eps, b1, b2, +1.f,
              st_);
  SRL_CUDA(cudaStreamSynchronize(st_));
  return SRL_OK;
}

}  // namespace srl
