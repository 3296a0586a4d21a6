// decoder_engine.cpp -- the decoder policy on the device: DecoderRunner (the
// varlen forward over a row plan: embedding, L x [QKV GEMM -> RoPE/KV append
// -> paged attention -> O GEMM(+residual, next RMSNorm stats) -> gate/up GEMM
// (SwiGLU) -> down GEMM(+residual)], LM head, sampler) and DecoderBackend
// (stream slots at a constant generation batch, prefill of new streams,
// CUDA-graph decode rounds, double-buffered weights with a pointer swap at
// token boundaries, optional KV recompute after a swap).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "decoder_engine.hpp"
#include "train.cuh"

namespace srl {

namespace {
int sm_count(int device) {
  int n = 148;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device);
  return n;
}
}  // namespace

WeightMaps build_weight_maps(const DecoderDims& d, const WeightLayout& lay, const __nv_bfloat16* w) {
  WeightMaps m;
  m.qkv.resize(d.L);
  m.o.resize(d.L);
  m.gate_up.resize(d.L);
  m.down.resize(d.L);
  for (int l = 0; l < d.L; ++l) {
    const LayerOffsets& o = lay.layers[l];
    m.qkv[l] = make_tmap_bf16(w + o.qkv_w, d.qkv(), d.H, 128);
    m.o[l] = make_tmap_bf16(w + o.o_w, d.H, d.qdim(), 128);
    m.gate_up[l] = make_tmap_bf16(w + o.gate_up_w, 2 * (uint64_t)d.I, d.H, 128);
    m.down[l] = make_tmap_bf16(w + o.down_w, d.H, d.I, 128);
  }
  m.lm_head = make_tmap_bf16(w + lay.lm_head, d.V, d.H, 128);
  return m;
}

// -------------------------------------------------------------- timer ---
void KernelTimer::begin(int kind) {
  while (pool.size() < used + 2) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    pool.push_back(e);
  }
  kinds.push_back(kind);
  cudaEventRecord(pool[used++], st);
}
void KernelTimer::end() { cudaEventRecord(pool[used++], st); }
void KernelTimer::collect(srl_kernel_profile* out) {
  *out = srl_kernel_profile{};
  for (size_t i = 0; i < kinds.size(); ++i) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, pool[2 * i], pool[2 * i + 1]);
    out->ms[kinds[i]] += ms;
    out->launches[kinds[i]] += 1;
  }
  out->valid = 1;
}
KernelTimer::~KernelTimer() {
  for (cudaEvent_t e : pool) cudaEventDestroy(e);
}

// ------------------------------------------------------------- runner ---
DecoderRunner::~DecoderRunner() {
  for (void* p : allocs_) cudaFree(p);
  if (fork_) cudaEventDestroy(fork_);
  if (join_) cudaEventDestroy(join_);
  if (side_) cudaStreamDestroy(side_);
}

int DecoderRunner::init(const DecoderDims& dims, const WeightLayout& layout, int slots, int max_seq,
                        int m_max, int logits_rows, int device, cudaStream_t st, bool precise_mode) {
  d = dims;
  precise = precise_mode;
  sp = precise ? 2 : 1;
  if (precise && (d.H % 64 || d.I % 64 || d.qdim() % 64))
    return fail(SRL_INVALID_ARGUMENT, "precise engine: every GEMM width a multiple of 64");
  lay = layout;  // offsets only (layers array owned by the weights object)
  S = slots;
  max_seq = max_seq;
  this->max_seq = max_seq;
  pages_per_seq = (max_seq + kPageTokens - 1) / kPageTokens;
  M_max = std::max(m_max, slots);
  this->logits_rows = std::max(logits_rows, slots);
  dev = device;
  st_ = st;
  sms = sm_count(device);
  SRL_CUDA(cudaStreamCreateWithFlags(&side_, cudaStreamNonBlocking));
  SRL_CUDA(cudaEventCreateWithFlags(&fork_, cudaEventDisableTiming));
  SRL_CUDA(cudaEventCreateWithFlags(&join_, cudaEventDisableTiming));
  unfused_qkv = std::getenv("SRL_UNFUSED_QKV") != nullptr;  // A/B switch: separate RoPE kernel
  const int H = d.H, parts = d.ssq_parts();
  auto alloc = [&](auto** p, size_t n) -> int {
    SRL_CUDA(cudaMalloc(p, std::max<size_t>(n, 1) * sizeof(**p)));
    SRL_CUDA(cudaMemset(*p, 0, std::max<size_t>(n, 1) * sizeof(**p)));
    allocs_.push_back(*p);
    return SRL_OK;
  };
  int st2;
  const size_t n_pages = (size_t)S * pages_per_seq;
  kv_layer_elems = n_pages * d.nkv * kPageTokens * d.hd;
  if ((st2 = alloc(&x, (size_t)M_max * H)) || (st2 = alloc(&xg, (size_t)M_max * H * sp)) ||
      (st2 = alloc(&ssq, (size_t)M_max * parts)) || (st2 = alloc(&qkv, (size_t)M_max * d.qkv())) ||
      (st2 = alloc(&q, (size_t)M_max * d.qdim())) || (st2 = alloc(&attn, (size_t)M_max * d.qdim() * sp)) ||
      (st2 = alloc(&act, (size_t)M_max * d.I * sp)) ||
      (st2 = alloc(&xg_last, (size_t)this->logits_rows * H * sp)) ||
      (st2 = alloc(&ssq_last, (size_t)this->logits_rows * parts)) ||
      (st2 = alloc(&logits, (size_t)this->logits_rows * d.V)) ||
      (st2 = alloc(&lse_max, (size_t)this->logits_rows * ((d.V + 127) / 128))) ||
      (st2 = alloc(&lse_sum, (size_t)this->logits_rows * ((d.V + 127) / 128))) ||
      (st2 = alloc(&kc, kv_layer_elems * d.L)) || (st2 = alloc(&vc, kv_layer_elems * d.L)) ||
      (st2 = alloc(&block_table, n_pages)) || (st2 = alloc(&cos_sin, (size_t)max_seq * d.hd)) ||
      (st2 = alloc(&plan.row_slot, M_max)) || (st2 = alloc(&plan.row_pos, M_max)) ||
      (st2 = alloc(&plan.row_token, M_max)) || (st2 = alloc(&plan.last_row, std::max(S, this->logits_rows))) ||
      (st2 = alloc(&next.row_slot, M_max)) || (st2 = alloc(&next.row_pos, M_max)) ||
      (st2 = alloc(&next.row_token, M_max)) || (st2 = alloc(&next.last_row, std::max(S, this->logits_rows))))
    return st2;
  // static page assignment: slot s owns pages [s*pps, (s+1)*pps)
  std::vector<int32_t> bt(n_pages);
  for (size_t i = 0; i < n_pages; ++i) bt[i] = (int32_t)i;
  SRL_CUDA(cudaMemcpy(block_table, bt.data(), bt.size() * 4, cudaMemcpyHostToDevice));
  launch_rope_table(cos_sin, max_seq, d.hd, (double)d.theta, st_);
  // activation TMA maps (box 64 and box 128 rows)
  for (int b = 0; b < 2; ++b) {
    const uint32_t box = b == 0 ? 64 : 128;
    xg_map[b] = make_tmap_bf16(xg, M_max, (uint64_t)H * sp, box);
    attn_map[b] = make_tmap_bf16(attn, M_max, (uint64_t)d.qdim() * sp, box);
    act_map[b] = make_tmap_bf16(act, M_max, (uint64_t)d.I * sp, box);
    last_map[b] = make_tmap_bf16(xg_last, this->logits_rows, (uint64_t)H * sp, box);
  }
  // GEMM workspace: the largest split-K need over every row count we may launch
  size_t need = 0;
  int counters = 1;
  const int shapes[5][2] = {{d.qkv(), H}, {H, d.qdim()}, {2 * d.I, H}, {H, d.I}, {d.V, H}};
  const int m_hi = std::max(M_max, this->logits_rows);
  // every row count the engine may launch: 1, 64, 128, ... and m_hi itself
  // (a row count between two multiples of 64 can need the larger token tile)
  for (int M = 1;; M = (M < 64) ? 64 : M + 64) {
    const int Mc = std::min(M, m_hi);
    const int tok = gemm_tok_tile(Mc);
    for (auto& sh : shapes) {
      const int sp = gemm_auto_splits(Mc, sh[0], sh[1], sms);
      need = std::max(need, sp > 1 ? gemm_workspace_floats(Mc, sh[0], sp) : 0);
      counters = std::max(counters, ((sh[0] + 127) / 128) * ((Mc + tok - 1) / tok));
    }
    if (M >= m_hi) break;
  }
  gws.partial_floats = need;
  gws.counter_count = counters;
  if ((st2 = alloc(&gws.partials, need)) || (st2 = alloc(&gws.counters, counters))) return st2;
  attn_ws_floats = std::max(attention_ws_floats(d, S, max_seq), attention_ws_floats(d, M_max, max_seq));
  if ((st2 = alloc(&seg, 4 * (size_t)std::max(S, 1)))) return st2;
  if ((st2 = alloc(&attn_ws, attn_ws_floats)) || (st2 = alloc(&attn_counters, (size_t)M_max * d.nkv)))
    return st2;
  SRL_CUDA(cudaStreamSynchronize(st_));
  return SRL_OK;
}

int DecoderRunner::gemm(const CUtensorMap& tw, const CUtensorMap* tx, int M, int N, int K,
                        const EpiParams& e) {
  if (precise) {  // X rows [hi (K) | lo (K)]: two K segments into one accumulator (persistent kernel)
    EpiParams es = e;
    es.seg_kb = K / 64;
    es.x_off1 = K;
    int tok = gemm_big_tok(M, N, 2 * K, sms);
    if (tok == 0) tok = 128;
    const cudaError_t err = gemm_big_launch(tw, tx[1], M, N, 2 * K, tok, es, st_);
    if (err != cudaSuccess) return cuda_fail(err, "gemm_big_launch (precise)");
    return SRL_OK;
  }
  static const bool lm_big = [] {
    const char* v = std::getenv("SRL_LM_BIG");
    return !(v && v[0] == '0');
  }();
  if (lm_big && M <= 64 && e.kind == EPI_LOGITS && (N + 127) / 128 >= 4 * sms) {
    // the LM head of <= 64 rows (a prefill round's slots, the multi-kernel
    // decode): the persistent kernel streams the vocabulary tiles through its
    // ring (the split-K kernel pays a pipeline fill per 128-row tile)
    const cudaError_t err = gemm_big_launch(tw, tx[1], M, N, K, 128, e, st_);
    if (err != cudaSuccess) return cuda_fail(err, "gemm_big_launch (lm head)");
    return SRL_OK;
  }
  const int splits = gemm_auto_splits(M, N, K, sms);
  const CUtensorMap& x_map = tx[gemm_tok_tile(M) == 64 ? 0 : 1];
  const cudaError_t err = gemm_bf16_launch(tw, x_map, M, N, K, splits, gws, e, st_);
  if (err != cudaSuccess) return cuda_fail(err, "gemm_bf16_launch");
  return SRL_OK;
}

int DecoderRunner::forward(int M, const __nv_bfloat16* w, const WeightMaps& wm) {
  const int H = d.H, parts = d.ssq_parts();
  const float inv_h = 1.0f / (float)H;
  tb(1);
  launch_embed(w + lay.embed, w + lay.layers[0].ln1, plan.row_token, M, H, d.V, x, xg, ssq, st_);
  if (precise) launch_split_bf16(x, M, H, nullptr, w + lay.layers[0].ln1, xg, st_);  // xg = split(x * ln1)
  te();
  int st;
  for (int l = 0; l < d.L; ++l) {
    const LayerOffsets& o = lay.layers[l];
    __nv_bfloat16* kcl = kc + kv_layer_elems * l;
    __nv_bfloat16* vcl = vc + kv_layer_elems * l;
    EpiParams e;  // QKV + bias + RoPE + paged KV append, fused
    e.kind = unfused_qkv ? EPI_STORE_F32 : EPI_QKV;
    e.out_f32 = qkv;
    e.ld_out = d.qkv();
    e.ssq_in = ssq; e.ssq_in_parts = parts; e.inv_dim = inv_h; e.eps = d.eps;
    e.bias = w + o.qkv_b;
    e.nq = d.nq; e.nkv = d.nkv; e.hd = d.hd; e.pages_per_seq = pages_per_seq;
    e.row_slot = plan.row_slot; e.row_pos = plan.row_pos; e.block_table = block_table;
    e.cos_sin = cos_sin; e.q_out = q; e.kc = kcl; e.vc = vcl;
    tb(2);
    if ((st = gemm(wm.qkv[l], xg_map, M, d.qkv(), H, e))) return st;
    te();
    if (unfused_qkv) {
      tb(3);
      launch_rope_append(qkv, d, plan, M, cos_sin, block_table, pages_per_seq, kcl, vcl, q, st_);
      te();
    }
    tb(4);
    if (n_seg > 0) {
      // prompt segments on the tensor cores, the single decode rows per row --
      // on a side stream, concurrently (disjoint output rows; both small)
      const bool side = n_single > 0 && timer == nullptr;
      if (n_single > 0) {
        if (side) {
          SRL_CUDA(cudaEventRecord(fork_, st_));
          SRL_CUDA(cudaStreamWaitEvent(side_, fork_, 0));
        }
        launch_attention(q, d, plan, n_single, block_table, pages_per_seq, kcl, vcl, max_seq, attn_ws,
                         attn_counters, attn_ws_floats, attn, side ? side_ : st_, nullptr,
                         precise ? d.qdim() : 0);
        if (side) SRL_CUDA(cudaEventRecord(join_, side_));
      }
      SRL_CUDA(launch_attention_fwd_mma(q, kcl, vcl, seg, seg + S, block_table, pages_per_seq, n_seg, d.nq,
                                        d.nkv, d.hd, attn, nullptr, st_, seg + 2 * S, seg + 3 * S,
                                        seg_max_rows, precise ? d.qdim() : 0));
      if (side) SRL_CUDA(cudaStreamWaitEvent(st_, join_, 0));
    } else {
      launch_attention(q, d, plan, M, block_table, pages_per_seq, kcl, vcl, max_seq, attn_ws,
                       attn_counters, attn_ws_floats, attn, st_, nullptr, precise ? d.qdim() : 0);
    }
    te();
    EpiParams r;
    r.kind = EPI_RESID; r.resid = x; r.gain = w + o.ln2; r.xg = xg; r.ssq_out = ssq;
    r.lo_off = precise ? H : 0;
    tb(5);
    if ((st = gemm(wm.o[l], attn_map, M, H, d.qdim(), r))) return st;
    te();
    EpiParams g;
    g.kind = EPI_SWIGLU;
    g.ssq_in = ssq; g.ssq_in_parts = parts; g.inv_dim = inv_h; g.eps = d.eps;
    g.out_bf16 = act; g.ld_bf16 = d.I * sp; g.lo_off = precise ? d.I : 0;
    tb(6);
    if ((st = gemm(wm.gate_up[l], xg_map, M, 2 * d.I, H, g))) return st;
    te();
    EpiParams r2;
    r2.kind = EPI_RESID; r2.resid = x; r2.xg = xg; r2.ssq_out = ssq; r2.lo_off = precise ? H : 0;
    r2.gain = w + (l + 1 < d.L ? lay.layers[l + 1].ln1 : lay.final_norm);
    tb(7);
    if ((st = gemm(wm.down[l], act_map, M, H, d.I, r2))) return st;
    te();
  }
  return SRL_OK;
}

int DecoderRunner::lm_head(int rows, const WeightMaps& wm, bool gathered) {
  EpiParams e;
  e.kind = EPI_LOGITS;
  e.part_max = lse_max;
  e.part_sum = lse_sum;
  e.ssq_in = gathered ? ssq_last : ssq;
  e.ssq_in_parts = d.ssq_parts();
  e.inv_dim = 1.0f / (float)d.H;
  e.eps = d.eps;
  e.out_f32 = logits;
  e.ld_out = d.V;
  tb(8);
  const int st = gemm(wm.lm_head, gathered ? last_map : xg_map, rows, d.V, d.H, e);
  te();
  return st;
}

// ------------------------------------------------------------ backend ---
DecoderBackend::DecoderBackend(const Policy& p, const srl_engine_options& o) : opts_(o) {
  (void)p;
}

DecoderBackend::~DecoderBackend() {
  if (st_) cudaStreamSynchronize(st_);
  for (int b = 0; b < 2; ++b)
    if (mk_.wmaps[b]) cudaFree(mk_.wmaps[b]);
  if (mk_.mem) cudaFree(mk_.mem);
  if (mk_.ws) cudaFree(mk_.ws);
  if (mk_.qkv_part) cudaFree(mk_.qkv_part);
  if (mk_.trace) cudaFree(mk_.trace);
  if (mk_.stamps_host) cudaFreeHost(mk_.stamps_host);
  for (int b = 0; b < 2; ++b)
    if (exec_[b]) cudaGraphExecDestroy(exec_[b]);
  if (dev_state_) cudaFree(dev_state_);
  if (pinned_) cudaFreeHost(pinned_);
  if (slot_stage_) cudaFreeHost(slot_stage_);
  if (ev_start_) cudaEventDestroy(ev_start_);
  if (ev_stop_) cudaEventDestroy(ev_stop_);
  for (cudaEvent_t& ev : ev_prof_)
    if (ev) cudaEventDestroy(ev);
  for (cudaEvent_t& ev : ev_pf_)
    if (ev) cudaEventDestroy(ev);
  runner_.reset();
  if (st_) cudaStreamDestroy(st_);
}

int DecoderBackend::init(const Policy& p) {
  SRL_CUDA(cudaSetDevice(opts_.device));
  SRL_CUDA(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
  SRL_CUDA(cudaEventCreate(&ev_start_));
  SRL_CUDA(cudaEventCreate(&ev_stop_));
  for (cudaEvent_t& ev : ev_prof_) SRL_CUDA(cudaEventCreate(&ev));
  for (cudaEvent_t& ev : ev_pf_) SRL_CUDA(cudaEventCreate(&ev));
  const DecoderWeights& src = *p.dec;
  d_ = src.dims;
  S_ = std::max(1, opts_.max_streams);
  max_seq_ = std::min(std::max(2, opts_.max_seq_len), d_.max_pos);
  R_ = std::max(opts_.event_ring, std::max(1, opts_.rounds_per_sync));
  prefill_budget_ = std::max(opts_.prefill_budget, 1);
  int st;
  for (int b = 0; b < 2; ++b) {
    if ((st = clone_decoder(src, buf_[b], opts_.device))) return st;
    maps_[b] = build_weight_maps(d_, buf_[b]->layout, buf_[b]->w);
  }
  runner_ = std::make_unique<DecoderRunner>();
  if ((st = runner_->init(d_, buf_[0]->layout, S_, max_seq_, S_ + prefill_budget_, S_,
                          opts_.device, st_, opts_.precise != 0)))
    return st;
  // slot state + ring + counters in one allocation
  const size_t ints = (size_t)S_ * 6 + 4;
  const size_t bytes = ints * 4 + (size_t)S_ * 8 + (size_t)S_ * max_seq_ * 4 +
                       (size_t)R_ * S_ * sizeof(DevEvent) + 256;
  SRL_CUDA(cudaMalloc(&dev_state_, bytes));
  SRL_CUDA(cudaMemset(dev_state_, 0, bytes));
  uint8_t* p8 = static_cast<uint8_t*>(dev_state_);
  auto take = [&](size_t n) {
    uint8_t* at = p8;
    p8 += (n + 15) / 16 * 16;
    return at;
  };
  ring_.ev = reinterpret_cast<DevEvent*>(take((size_t)R_ * S_ * sizeof(DevEvent)));
  ring_.rounds = R_;
  ss_.seed = reinterpret_cast<uint64_t*>(take((size_t)S_ * 8));
  ss_.live = reinterpret_cast<int32_t*>(take((size_t)S_ * 4));
  ss_.seq_len = reinterpret_cast<int32_t*>(take((size_t)S_ * 4));
  ss_.gen_count = reinterpret_cast<int32_t*>(take((size_t)S_ * 4));
  ss_.max_tokens = reinterpret_cast<int32_t*>(take((size_t)S_ * 4));
  ss_.terminator = reinterpret_cast<int32_t*>(take((size_t)S_ * 4));
  ss_.history = reinterpret_cast<int32_t*>(take((size_t)S_ * max_seq_ * 4));
  ss_.max_seq = max_seq_;
  version_dev_ = reinterpret_cast<int32_t*>(take(4));
  round_ctr_dev_ = reinterpret_cast<int32_t*>(take(4));
  // pinned staging: events + plan upload + scalars
  pinned_bytes_ = (size_t)R_ * S_ * sizeof(DevEvent) + (size_t)(runner_->M_max * 3 + S_ + 64) * 4 +
                  (size_t)S_ * 64;
  SRL_CUDA(cudaMallocHost(&pinned_, pinned_bytes_));
  SRL_CUDA(cudaMallocHost(&slot_stage_, 4 * (size_t)S_ * max_seq_));
  host_.assign(S_, HostSlot{});
  // next plan: every slot dead
  std::vector<int32_t> neg(std::max(runner_->M_max, S_), -1);
  SRL_CUDA(cudaMemcpy(runner_->next.row_slot, neg.data(), 4 * (size_t)runner_->M_max, cudaMemcpyHostToDevice));
  SRL_CUDA(cudaMemcpy(runner_->next.last_row, neg.data(), 4 * (size_t)S_, cudaMemcpyHostToDevice));
  SRL_CUDA(cudaMemcpy(runner_->plan.row_slot, neg.data(), 4 * (size_t)runner_->M_max, cudaMemcpyHostToDevice));
  SRL_CUDA(cudaMemcpy(runner_->plan.last_row, neg.data(), 4 * (size_t)S_, cudaMemcpyHostToDevice));
  return mega_init();
}

// Phase table, device tensor maps and counters of the persistent decode
// kernel.  Off with SRL_MEGAKERNEL=0 (the multi-kernel CUDA-graph round).
int DecoderBackend::mega_init() {
  const char* env = std::getenv("SRL_MEGAKERNEL");
  if ((env && env[0] == '0') || !megakernel_supported(d_, S_)) return SRL_OK;
  DecoderRunner& r = *runner_;
  const int grid = r.sms;
  if (megakernel_occupancy(d_) < 1) return SRL_OK;  // not co-resident: multi-kernel round
  if (opts_.precise) return SRL_OK;                  // precise engine: the multi-kernel round
  // keys per attention item (SRL_MK_ATTN_CHUNK: 64..8192, a multiple of 64).  A
  // 1.5B round at steady-state 8k contexts, items handed out longest first:
  // 1024 -> 3.49 ms, 2048 -> 3.12, 4096 -> 2.88, 6144 -> 3.47, 8192 -> 3.95 (the
  // item's q / k / v prologue and split merge amortised over more keys, until
  // there are fewer items than SMs)
  const int chunk_env = [] {  // read per engine (tests set it)
    const char* v = std::getenv("SRL_MK_ATTN_CHUNK");
    const int c = v ? std::atoi(v) : kMkAttnChunk;
    return std::max(64, std::min(8192, c / 64 * 64));
  }();
  // the per-round item order (mk_attn_order) keeps 2 ints per item in the
  // scratch area: at most kMkMaxAttnItems items, so coarser splits if needed
  int attn_chunk = chunk_env;
  while ((size_t)S_ * d_.nkv * ((max_seq_ + attn_chunk - 1) / attn_chunk) > (size_t)kMkMaxAttnItems)
    attn_chunk += 64;
  const int L = d_.L, splits = (max_seq_ + attn_chunk - 1) / attn_chunk;
  // pair mode (SRL_MK_PAIRS=1): cluster of two CTAs, DSMEM split-K for QKV and
  // O, attention reads finished q / K / V
  const char* pe = std::getenv("SRL_MK_PAIRS");
  // (measured slower at 0.5B / B = 64: the 32-row pair epilogues are latency-bound; off by default)
  const bool pairs = pe && pe[0] == '1' && grid % 2 == 0 && megakernel_pair_clusters(d_) * 2 >= grid;
  std::vector<MkPhase> ph;
  int ctr = 0, items_total = 0;
  size_t ws = (size_t)S_ * d_.nkv * splits * (d_.nq / d_.nkv) * (d_.hd + 2);
  auto add = [&](int kind, int layer, int n_items, int cs, int N, int K, int wmap, int xmap,
                 int counters) {
    MkPhase f{kind, layer, n_items, cs, N, K, wmap, xmap, ctr, items_total % grid, -1, -1, 0, 0, -1};
    if (pairs && cs == 2 && (kind == MK_QKV || kind == MK_O)) f.rot &= ~1;  // split 0 on the even CTA
    const LayerOffsets* lo = buf_[0]->layout.layers;
    if (kind == MK_O) f.colv = (long long)lo[layer].ln2;
    if (kind == MK_ATTN) f.colv = (long long)lo[layer].qkv_b;
    if (kind == MK_DOWN)
      f.colv = (long long)(layer + 1 < d_.L ? lo[layer + 1].ln1 : buf_[0]->layout.final_norm);
    ctr += counters;
    items_total += n_items;
    ph.push_back(f);
  };
  auto cs_env = [](int kind) {  // tuning overrides: SRL_MK_CS_{QKV,O,GU,DOWN,LM}
    static const char* names[7] = {nullptr, "SRL_MK_CS_QKV", nullptr, "SRL_MK_CS_O", "SRL_MK_CS_GU",
                                   "SRL_MK_CS_DOWN", "SRL_MK_CS_LM"};
    const char* v = names[kind] ? std::getenv(names[kind]) : nullptr;
    return v ? std::max(1, std::min(16, std::atoi(v))) : 0;
  };
  auto gemm = [&](int kind, int layer, int N, int K, int wmap, int xmap) {
    int cs = megakernel_splits(N, K, grid);
    if (const int o = cs_env(kind)) cs = std::min(o, K / 64);
    const int tiles = (N + 127) / 128;
    ws = std::max(ws, megakernel_ws_floats(tiles * cs, cs, S_));
    add(kind, layer, tiles * cs, cs, N, K, wmap, xmap, cs > 1 ? tiles : 0);
  };
  // QKV: raw split partials only (no counters); the attention items reduce them
  int qkv_cs = megakernel_qkv_splits(d_, grid);
  if (const char* v = std::getenv("SRL_MK_CS_QKV")) qkv_cs = std::max(1, std::min(qkv_cs, std::atoi(v)));
  const int qkv_tiles = (d_.qkv() + 127) / 128;
  if (pairs) qkv_cs = 2;
  add(MK_EMBED, 0, S_, 1, 0, 0, 0, 0, 0);
  for (int l = 0; l < L; ++l) {
    add(MK_QKV, l, qkv_tiles * qkv_cs, qkv_cs, d_.qkv(), d_.H, 4 * l + 0, 0, 0);
    add(MK_ATTN, l, S_ * d_.nkv * splits, qkv_cs, 0, 0, 0, 0, S_ * d_.nkv + 1);  // + the work queue
    if (pairs)  // the pair reduces through DSMEM: no L2 partials, no counters
      add(MK_O, l, ((d_.H + 127) / 128) * 2, 2, d_.H, d_.qdim(), 4 * l + 1, 1, 0);
    else
      gemm(MK_O, l, d_.H, d_.qdim(), 4 * l + 1, 1);
    gemm(MK_GU, l, 2 * d_.I, d_.H, 4 * l + 2, 0);
    gemm(MK_DOWN, l, d_.H, d_.I, 4 * l + 3, 2);
  }
  gemm(MK_LM, 0, d_.V, d_.H, 4 * L, 0);
  add(MK_SAMPLE, 0, S_, 1, 0, 0, 0, 0, 0);
  // dataflow links (experiment, SRL_MK_FLOW=1 / q / d; measured slower than
  // the grid barriers at 0.5B, B = 64: the per-tile counter polls and done
  // signals cost more than the barrier they skip): QKV(l) reads xg from
  // down(l-1) tiles of 128 columns, down(l) reads act from gate/up(l) tiles of
  // 64 act columns; producer tiles count their row slices' epilogues
  const char* fe = std::getenv("SRL_MK_FLOW");
  if (fe && fe[0] != '0' && !pairs) {
    for (size_t i = 1; i < ph.size(); ++i) {
      MkPhase& f = ph[i];
      MkPhase& prev = ph[i - 1];
      const bool want_q = !fe || fe[0] != 'd', want_d = !fe || fe[0] != 'q';
      const bool link = (want_q && f.kind == MK_QKV && prev.kind == MK_DOWN) ||
                        (want_d && f.kind == MK_DOWN && prev.kind == MK_GU);
      if (!link) continue;
      const int tiles = (prev.N + 127) / 128;
      prev.done_ctr = ctr;
      ctr += tiles;
      f.flow_ctr = prev.done_ctr;
      f.flow_cols = prev.kind == MK_GU ? 64 : 128;
      f.flow_target = prev.cs;
    }
  }
  const int n = (int)ph.size();

  // one allocation: phases | layers | xmaps | phase_done | epoch | tile counters | stamps
  auto al = [](size_t v) { return (v + 127) / 128 * 128; };
  const size_t o_ph = 0, o_ly = al(o_ph + sizeof(MkPhase) * n), o_xm = al(o_ly + sizeof(MkLayer) * L),
               o_pd = al(o_xm + sizeof(CUtensorMap) * 3), o_ep = al(o_pd + 4 * 8 * (size_t)n)  /* room for 8 barrier lanes */,
               o_tc = al(o_ep + 4), o_st = al(o_tc + 4 * (size_t)std::max(ctr, 1)),
               o_ao = al(o_st + 8 * (size_t)(n + 1)),
               total = al(o_ao + 4 * (size_t)S_ * d_.nkv * splits);
  SRL_CUDA(cudaMalloc(&mk_.mem, total));
  SRL_CUDA(cudaMemset(mk_.mem, 0, total));
  SRL_CUDA(cudaMalloc(&mk_.ws, std::max<size_t>(ws, 1) * sizeof(float)));
  SRL_CUDA(cudaMalloc(&mk_.qkv_part, (size_t)qkv_cs * S_ * d_.qkv() * sizeof(float)));
  SRL_CUDA(cudaMallocHost(&mk_.stamps_host, 8 * (size_t)(n + 1)));
  uint8_t* base = static_cast<uint8_t*>(mk_.mem);
  std::vector<MkLayer> ly(L);
  for (int l = 0; l < L; ++l) {
    const LayerOffsets& o = buf_[0]->layout.layers[l];
    ly[l] = MkLayer{o.ln1, o.qkv_b, o.ln2};
  }
  const CUtensorMap xm[3] = {r.xg_map[0], r.attn_map[0], r.act_map[0]};
  SRL_CUDA(cudaMemcpy(base + o_ph, ph.data(), sizeof(MkPhase) * n, cudaMemcpyHostToDevice));
  SRL_CUDA(cudaMemcpy(base + o_ly, ly.data(), sizeof(MkLayer) * L, cudaMemcpyHostToDevice));
  SRL_CUDA(cudaMemcpy(base + o_xm, xm, sizeof(xm), cudaMemcpyHostToDevice));
  for (int b = 0; b < 2; ++b) {
    std::vector<CUtensorMap> wm(4 * L + 1);
    for (int l = 0; l < L; ++l) {
      wm[4 * l + 0] = maps_[b].qkv[l];
      wm[4 * l + 1] = maps_[b].o[l];
      wm[4 * l + 2] = maps_[b].gate_up[l];
      wm[4 * l + 3] = maps_[b].down[l];
    }
    wm[4 * L] = maps_[b].lm_head;
    SRL_CUDA(cudaMalloc(&mk_.wmaps[b], sizeof(CUtensorMap) * wm.size()));
    SRL_CUDA(cudaMemcpy(mk_.wmaps[b], wm.data(), sizeof(CUtensorMap) * wm.size(), cudaMemcpyHostToDevice));
    MkParams& P = mk_.params[b];
    P = MkParams{};
    P.S = S_; P.H = d_.H; P.I = d_.I; P.V = d_.V; P.L = L; P.nq = d_.nq; P.nkv = d_.nkv;
    P.hd = d_.hd; P.qkv = d_.qkv(); P.parts = d_.ssq_parts(); P.pps = r.pages_per_seq;
    P.attn_splits = splits; P.attn_chunk = attn_chunk; P.greedy = opts_.greedy;
    P.eps = d_.eps; P.inv_h = 1.0f / (float)d_.H; P.scale = 1.0f / sqrtf((float)d_.hd);
    P.w = buf_[b]->w;
    P.wmaps = mk_.wmaps[b];
    P.xmaps = reinterpret_cast<const CUtensorMap*>(base + o_xm);
    P.layers = reinterpret_cast<const MkLayer*>(base + o_ly);
    P.off_embed = buf_[b]->layout.embed;
    P.off_final_norm = buf_[b]->layout.final_norm;
    P.x = r.x; P.xg = r.xg; P.ssq = r.ssq; P.q = r.q; P.attn = r.attn; P.act = r.act;
    P.logits = r.logits; P.lse_max = r.lse_max; P.lse_sum = r.lse_sum;
    P.kc = r.kc; P.vc = r.vc; P.kv_layer_elems = r.kv_layer_elems;
    P.block_table = r.block_table; P.cos_sin = r.cos_sin;
    P.plan = r.plan; P.next = r.next; P.ss = ss_; P.ring = ring_;
    P.round_ctr = round_ctr_dev_; P.version = version_dev_;
    P.phase_done = reinterpret_cast<unsigned*>(base + o_pd);
    P.epoch = reinterpret_cast<unsigned*>(base + o_ep);
    P.tile_ctr = reinterpret_cast<unsigned*>(base + o_tc);
    P.attn_order = reinterpret_cast<int32_t*>(base + o_ao);
    P.ws = mk_.ws;
    P.qkv_part = mk_.qkv_part;
    P.phases = reinterpret_cast<const MkPhase*>(base + o_ph);
    P.n_phases = n;
    P.stamps = nullptr;
    if (const char* dbg = std::getenv("SRL_MK_DBG")) P.dbg = std::atoi(dbg);
    P.trace_item = 0;
    if (const char* ti = std::getenv("SRL_MK_TRACE_ITEM")) P.trace_item = std::max(0, std::atoi(ti));
    {
      const char* pf = std::getenv("SRL_MK_L2PF");
      P.l2_prefetch = pf ? (pf[0] != '0') : 0;
    }
    P.pairs = pairs ? 1 : 0;
  }
  mk_.stamps = reinterpret_cast<unsigned long long*>(base + o_st);
  if (std::getenv("SRL_MK_TRACE")) SRL_CUDA(cudaMalloc(&mk_.trace, 128 * (size_t)n * grid));
  mk_.phases = ph;
  mk_.n_phases = n;
  mk_.grid = grid;
  mk_.on = true;
  return SRL_OK;
}

int DecoderBackend::mega_round(int b, bool profile) {
  MkParams p = mk_.params[b];
  if (profile) p.stamps = mk_.stamps;
  if (profile && mk_.trace) {
    p.trace = mk_.trace;
    SRL_CUDA(cudaMemsetAsync(mk_.trace, 0, 128 * (size_t)mk_.n_phases * mk_.grid, st_));
  }
  if (profile) SRL_CUDA(cudaEventRecord(ev_prof_[0], st_));
  const cudaError_t e = launch_megakernel(p, d_, mk_.grid, st_);
  if (e != cudaSuccess) return cuda_fail(e, "launch_megakernel");
  if (profile) {
    SRL_CUDA(cudaEventRecord(ev_prof_[1], st_));
    SRL_CUDA(cudaMemcpyAsync(mk_.stamps_host, mk_.stamps, 8 * (size_t)(mk_.n_phases + 1),
                             cudaMemcpyDeviceToHost, st_));
    SRL_CUDA(cudaStreamSynchronize(st_));
    // phase durations (grid-wide completion as seen by CTA 0) -> kernel classes
    static const int cls[8] = {1, 2, 4, 5, 6, 7, 8, 9};
    profile_ = srl_kernel_profile{};
    for (int i = 0; i < mk_.n_phases; ++i) {
      const int c = cls[mk_.phases[i].kind];
      profile_.ms[c] += (double)(mk_.stamps_host[i + 1] - mk_.stamps_host[i]) * 1e-6;
      profile_.launches[c] += 1;
    }
    profile_.valid = 1;
    profile_.rows = S_;
    profile_.fused = 1;
    float fms = 0.f;
    SRL_CUDA(cudaEventElapsedTime(&fms, ev_prof_[0], ev_prof_[1]));
    profile_.fused_ms = fms;
    if (mk_.trace) {  // debugging dump: kind, cs, n_items per phase then the raw stamps
      const size_t nt = 16 * (size_t)mk_.n_phases * mk_.grid;
      std::vector<unsigned long long> h(nt);
      SRL_CUDA(cudaMemcpy(h.data(), mk_.trace, 8 * nt, cudaMemcpyDeviceToHost));
      if (FILE* f = std::fopen(std::getenv("SRL_MK_TRACE"), "wb")) {
        const int hdr[2] = {mk_.n_phases, mk_.grid};
        std::fwrite(hdr, sizeof(hdr), 1, f);
        for (const MkPhase& f2 : mk_.phases) {
          const int row[4] = {f2.kind, f2.cs, f2.n_items, f2.rot};
          std::fwrite(row, sizeof(row), 1, f);
        }
        std::fwrite(h.data(), 8, nt, f);
        std::fclose(f);
      }
    }
  }
  return SRL_OK;
}

int DecoderBackend::check_stream(const StreamSpec& spec) const {
  const int64_t n_prefix = 1 + (int64_t)spec.prompt.size();
  if (n_prefix + spec.max_tokens > max_seq_)
    return fail(SRL_INVALID_ARGUMENT, "open_stream: bos + prompt + max_tokens exceeds max_seq_len");
  return SRL_OK;
}

int DecoderBackend::open_slot(int slot, const StreamSpec& spec) {
  const int n_prefix = 1 + (int)spec.prompt.size();
  if (const int st = check_stream(spec)) return st;
  HostSlot& h = host_[slot];
  h = HostSlot{};
  h.live = true;
  h.pending = true;
  h.tokens.push_back(d_.bos);
  h.tokens.insert(h.tokens.end(), spec.prompt.begin(), spec.prompt.end());
  h.fed = 0;
  // device slot state: one tiny kernel for the scalars, the prefix from this
  // slot's own pinned staging row (alive until the slot is reopened, which
  // happens only after the stream's rounds ran): no stream synchronisation
  launch_slot_set(ss_, slot, 1, 1, spec.max_tokens, spec.terminator, spec.seed, st_);
  int32_t* stage = slot_stage_ + (size_t)slot * max_seq_;
  std::memcpy(stage, h.tokens.data(), 4 * h.tokens.size());
  SRL_CUDA(cudaMemcpyAsync(ss_.history + (size_t)slot * max_seq_, stage, 4 * h.tokens.size(),
                           cudaMemcpyHostToDevice, st_));
  any_pending_ = true;
  return SRL_OK;
}

void DecoderBackend::close_slot(int slot) {
  host_[slot].live = false;
  host_[slot].pending = false;
  launch_slot_set(ss_, slot, 0, 0, 0, -1, 0, st_);  // stream-ordered before the next round
}

int DecoderBackend::decode_round_eager(int b) {
  DecoderRunner& r = *runner_;
  r.tb(0);
  launch_plan_copy(r.plan, r.next, S_, S_, round_ctr_dev_, st_);
  r.te();
  int st;
  if ((st = r.forward(S_, buf_[b]->w, maps_[b]))) return st;
  if ((st = r.lm_head(S_, maps_[b], false))) return st;
  r.tb(9);
  launch_sample(r.logits, r.lse_max, r.lse_sum, d_.V, S_, r.plan, r.next, ss_, ring_,
                round_ctr_dev_, version_dev_, opts_.greedy, st_);
  r.te();
  return SRL_OK;
}

int DecoderBackend::capture(int b) {
  cudaGraph_t g = nullptr;
  SRL_CUDA(cudaStreamBeginCapture(st_, cudaStreamCaptureModeThreadLocal));
  const int st = decode_round_eager(b);
  const cudaError_t e = cudaStreamEndCapture(st_, &g);
  if (st != SRL_OK) {
    if (g) cudaGraphDestroy(g);
    return st;
  }
  SRL_CUDA(e);
  SRL_CUDA(cudaGraphInstantiate(&exec_[b], g, 0));
  cudaGraphDestroy(g);
  return SRL_OK;
}

// Prefill round: decode rows for running slots + prompt rows for pending slots.
int DecoderBackend::prefill_round(int b, std::vector<int>& prefilled) {
  DecoderRunner& r = *runner_;
  std::vector<int32_t> rs, rp, rt, last(S_, -1);
  for (int s = 0; s < S_; ++s) {
    HostSlot& h = host_[s];
    if (!h.live || h.pending) continue;
    last[s] = (int)rs.size();
    rs.push_back(s);
    rp.push_back(h.fed);
    rt.push_back(h.tokens.back());
  }
  int budget = prefill_budget_;
  for (int s = 0; s < S_; ++s) {
    HostSlot& h = host_[s];
    if (!h.live || !h.pending) continue;
    const int n = (int)h.tokens.size();
    if (n > budget && !prefilled.empty()) continue;  // next round
    for (int p = 0; p < n; ++p) {
      rs.push_back(s);
      rp.push_back(p);
      rt.push_back(h.tokens[p]);
    }
    last[s] = (int)rs.size() - 1;
    budget -= n;
    prefilled.push_back(s);
  }
  const int M = (int)rs.size();
  if (M > r.M_max) return fail(SRL_INVALID_ARGUMENT, "prefill exceeds the engine's row budget");
  last_prefill_rows_ = M;
  // one attention segment per prompt (rows after the running slots' decode rows)
  std::vector<int32_t> seg(4 * (size_t)S_, 0);
  int n_seg = 0, seg_max = 0;
  const int n_single = S_ > 0 ? (int)std::count_if(last.begin(), last.end(), [](int v) { return v >= 0; }) -
                                    (int)prefilled.size()
                              : 0;
  for (int s : prefilled) {
    const int n = (int)host_[s].tokens.size();
    seg[n_seg] = last[s] - n + 1;
    seg[S_ + n_seg] = n;
    seg[2 * S_ + n_seg] = 0;
    seg[3 * S_ + n_seg] = s;
    seg_max = std::max(seg_max, n);
    ++n_seg;
  }
  int32_t* pin = reinterpret_cast<int32_t*>(static_cast<uint8_t*>(pinned_) + (size_t)R_ * S_ * sizeof(DevEvent));
  std::memcpy(pin, rs.data(), 4 * M);
  std::memcpy(pin + M, rp.data(), 4 * M);
  std::memcpy(pin + 2 * M, rt.data(), 4 * M);
  std::memcpy(pin + 3 * M, last.data(), 4 * S_);
  std::memcpy(pin + 3 * M + S_, seg.data(), 16 * (size_t)S_);
  SRL_CUDA(cudaMemcpyAsync(r.seg, pin + 3 * M + S_, 16 * (size_t)S_, cudaMemcpyHostToDevice, st_));
  SRL_CUDA(cudaMemcpyAsync(r.next.row_slot, pin, 4 * M, cudaMemcpyHostToDevice, st_));
  SRL_CUDA(cudaMemcpyAsync(r.next.row_pos, pin + M, 4 * M, cudaMemcpyHostToDevice, st_));
  SRL_CUDA(cudaMemcpyAsync(r.next.row_token, pin + 2 * M, 4 * M, cudaMemcpyHostToDevice, st_));
  SRL_CUDA(cudaMemcpyAsync(r.next.last_row, pin + 3 * M, 4 * S_, cudaMemcpyHostToDevice, st_));
  launch_plan_copy(r.plan, r.next, M, S_, round_ctr_dev_, st_);
  int st;
  r.n_seg = n_seg;
  r.n_single = n_single;
  r.seg_max_rows = seg_max;
  st = r.forward(M, buf_[b]->w, maps_[b]);
  r.n_seg = 0;
  if (st) return st;
  launch_gather_rows(r.xg, r.ssq, r.plan.last_row, S_, d_.H * r.sp, d_.ssq_parts(), r.xg_last, r.ssq_last, st_);
  if ((st = r.lm_head(S_, maps_[b], true))) return st;
  launch_sample(r.logits, r.lse_max, r.lse_sum, d_.V, S_, r.plan, r.next, ss_, ring_,
                round_ctr_dev_, version_dev_, opts_.greedy, st_);
  // the staging buffer is reused by the next prefill: keep it ordered
  SRL_CUDA(cudaStreamSynchronize(st_));
  return SRL_OK;
}

int DecoderBackend::run_rounds(int n, std::vector<SlotEvent>& events, double* device_ms) {
  events.assign((size_t)n * S_, SlotEvent{});
  int done = 0;
  while (done < n) {
    int batch = std::min(n - done, R_);
    std::vector<std::vector<int>> prefilled_at(batch);
    bool profiled = false, prefilled = false;
    SRL_CUDA(cudaEventRecord(ev_start_, st_));
    const int64_t c0 = round_ctr_host_;
    for (int i = 0; i < batch; ++i) {
      int st;
      if (any_pending_ && i > 0) {
        // a prefill round builds the running slots' decode rows from host
        // state, which only learns this batch's tokens when its events are
        // copied back: end the batch here, the prefill opens the next one
        batch = i;
        break;
      }
      if (any_pending_) {
        SRL_CUDA(cudaEventRecord(ev_pf_[0], st_));
        if ((st = prefill_round(active_, prefilled_at[i]))) return st;
        SRL_CUDA(cudaEventRecord(ev_pf_[1], st_));
        prefilled = true;
        for (int s : prefilled_at[i]) host_[s].pending = false;
        any_pending_ = false;
        for (const HostSlot& h : host_)
          if (h.live && h.pending) any_pending_ = true;
        launches_ += 6 * d_.L + 5;
      } else if (mk_.on) {
        if ((st = mega_round(active_, profile_next_))) return st;
        profile_next_ = false;
        launches_ += 1;
      } else if (profile_next_) {
        timer_.st = st_;
        timer_.reset();
        runner_->timer = &timer_;
        st = decode_round_eager(active_);
        runner_->timer = nullptr;
        if (st) return st;
        profile_next_ = false;
        profiled = true;
        launches_ += 6 * d_.L + 4;
      } else if (opts_.use_graphs) {
        if (!exec_[active_] && (st = capture(active_))) return st;
        SRL_CUDA(cudaGraphLaunch(exec_[active_], st_));
        launches_ += 6 * d_.L + 4;
      } else {
        if ((st = decode_round_eager(active_))) return st;
        launches_ += 6 * d_.L + 4;
      }
      ++round_ctr_host_;
    }
    SRL_CUDA(cudaEventRecord(ev_stop_, st_));
    // copy the batch's ring rows (at most two contiguous ranges)
    DevEvent* pe = static_cast<DevEvent*>(pinned_);
    const int r0 = (int)(c0 % R_);
    const int first = std::min(batch, R_ - r0);
    SRL_CUDA(cudaMemcpyAsync(pe, ring_.ev + (size_t)r0 * S_, sizeof(DevEvent) * first * S_,
                             cudaMemcpyDeviceToHost, st_));
    if (batch > first)
      SRL_CUDA(cudaMemcpyAsync(pe + (size_t)first * S_, ring_.ev, sizeof(DevEvent) * (batch - first) * S_,
                               cudaMemcpyDeviceToHost, st_));
    SRL_CUDA(cudaStreamSynchronize(st_));
    SRL_CUDA(cudaGetLastError());
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ev_start_, ev_stop_);
    if (device_ms) *device_ms += ms;
    if (prefilled) {
      float pms = 0.f;
      cudaEventElapsedTime(&pms, ev_pf_[0], ev_pf_[1]);
      prefill_ms_ += pms;
      prefill_rounds_ += 1;
      prefill_rows_ += last_prefill_rows_;
    }
    if (profiled) {
      timer_.collect(&profile_);
      profile_.rows = S_;
    }
    for (int i = 0; i < batch; ++i) {
      for (int s = 0; s < S_; ++s) {
        const DevEvent& e = pe[(size_t)i * S_ + s];
        SlotEvent& o = events[(size_t)(done + i) * S_ + s];
        o.flag = e.flag; o.token = e.token; o.position = e.position; o.version = e.version;
        o.logprob = e.logprob;
        if (e.flag == 0) continue;
        HostSlot& h = host_[s];
        h.fed = (int)h.tokens.size();  // every token so far is now in the KV cache
        h.tokens.push_back(e.token);
        if (e.flag >= 2) h.live = false;
      }
    }
    done += batch;
  }
  return SRL_OK;
}

int DecoderBackend::check_update(const Policy& p) {
  if (!p.dec || !same_decoder_shape(p.dec->cfg, buf_[active_]->cfg))
    return fail(SRL_POLICY_MISMATCH, "policy_mismatch: decoder shape differs");
  return SRL_OK;
}

int DecoderBackend::swap_and_recompute(bool recompute, int version) {
  int32_t* pi = reinterpret_cast<int32_t*>(static_cast<uint8_t*>(pinned_) + pinned_bytes_ - 64);
  const int old_version = version - 1;  // versions are strictly sequential (engine.cpp:82-87)
  active_ ^= 1;
  pi[5] = version;
  SRL_CUDA(cudaMemcpyAsync(version_dev_, pi + 5, 4, cudaMemcpyHostToDevice, st_));
  int st = recompute ? recompute_kv() : SRL_OK;
  if (st == SRL_OK && cudaStreamSynchronize(st_) != cudaSuccess) st = SRL_CUDA_ERROR;
  if (st != SRL_OK) {
    // a rejected update leaves the engine serving the old weights at the old
    // version (engine.cpp:79-117): swap back, restore the version stamp and,
    // in recompute mode, rebuild the live caches under the old weights
    active_ ^= 1;
    pi[5] = old_version;
    cudaMemcpyAsync(version_dev_, pi + 5, 4, cudaMemcpyHostToDevice, st_);
    if (recompute) recompute_kv();
    cudaStreamSynchronize(st_);
    return st;
  }
  return SRL_OK;
}

// Recompute mode (engine.cpp:107-113): rebuild every live slot's KV cache
// from its full prefix under the new weights, chunked by position so each
// chunk only attends to already-rewritten keys.
int DecoderBackend::recompute_kv() {
  DecoderRunner& r = *runner_;
  int max_fed = 0, n_live = 0;
  for (const HostSlot& h : host_)
    if (h.live && !h.pending) {
      max_fed = std::max(max_fed, h.fed);
      ++n_live;
    }
  if (n_live == 0) return SRL_OK;
  // chunks of positions [c0, c1), rows slot-major inside a chunk: each live
  // slot's rows form one attention segment (first row, count, first position,
  // slot) for the tensor-core kernel; keys before c0 were rewritten by the
  // previous chunks, keys in [c0, p] by this chunk's QKV epilogue
  const int span = std::max(1, r.M_max / n_live);
  std::vector<int32_t> rs, rp, rt, seg(4 * (size_t)S_);
  for (int c0 = 0; c0 < max_fed; c0 += span) {
    const int c1 = std::min(max_fed, c0 + span);
    rs.clear(); rp.clear(); rt.clear();
    int n_seg = 0, seg_max = 0;
    for (int s = 0; s < S_; ++s) {
      const HostSlot& h = host_[s];
      if (!h.live || h.pending || c0 >= h.fed) continue;
      const int e = std::min(c1, h.fed);
      seg[n_seg] = (int)rs.size();
      seg[S_ + n_seg] = e - c0;
      seg[2 * S_ + n_seg] = c0;
      seg[3 * S_ + n_seg] = s;
      seg_max = std::max(seg_max, e - c0);
      ++n_seg;
      for (int p = c0; p < e; ++p) {
        rs.push_back(s);
        rp.push_back(p);
        rt.push_back(h.tokens[p]);
      }
    }
    const int M = (int)rs.size();
    if (M == 0) continue;
    int32_t* pin = reinterpret_cast<int32_t*>(static_cast<uint8_t*>(pinned_) + (size_t)R_ * S_ * sizeof(DevEvent));
    std::memcpy(pin, rs.data(), 4 * M);
    std::memcpy(pin + M, rp.data(), 4 * M);
    std::memcpy(pin + 2 * M, rt.data(), 4 * M);
    std::memcpy(pin + 3 * M + S_, seg.data(), 16 * (size_t)S_);
    SRL_CUDA(cudaMemcpyAsync(r.plan.row_slot, pin, 4 * M, cudaMemcpyHostToDevice, st_));
    SRL_CUDA(cudaMemcpyAsync(r.plan.row_pos, pin + M, 4 * M, cudaMemcpyHostToDevice, st_));
    SRL_CUDA(cudaMemcpyAsync(r.plan.row_token, pin + 2 * M, 4 * M, cudaMemcpyHostToDevice, st_));
    SRL_CUDA(cudaMemcpyAsync(r.seg, pin + 3 * M + S_, 16 * (size_t)S_, cudaMemcpyHostToDevice, st_));
    r.n_seg = n_seg;
    r.n_single = 0;
    r.seg_max_rows = seg_max;
    const int st = r.forward(M, buf_[active_]->w, maps_[active_]);
    r.n_seg = 0;
    if (st != SRL_OK) return st;
    SRL_CUDA(cudaStreamSynchronize(st_));  // the pinned staging is reused by the next chunk
  }
  return SRL_OK;
}

int DecoderBackend::apply_update(const Policy& p, bool recompute, int version) {
  SRL_CUDA(cudaMemcpyAsync(buf_[active_ ^ 1]->w, p.dec->w, p.dec->bytes, cudaMemcpyDeviceToDevice, st_));
  return swap_and_recompute(recompute, version);
}

int DecoderBackend::standby(void** ptr, size_t* bytes) {
  *ptr = buf_[active_ ^ 1]->w;
  *bytes = buf_[active_ ^ 1]->bytes;
  return SRL_OK;
}

int DecoderBackend::commit_standby(bool recompute, int version) {
  return swap_and_recompute(recompute, version);
}

int DecoderBackend::slot_history(int slot, std::vector<int32_t>& out) {
  out = host_[slot].tokens;
  return SRL_OK;
}

std::unique_ptr<Backend> make_decoder_backend(const Policy& p, const srl_engine_options& o, int* status) {
  auto b = std::make_unique<DecoderBackend>(p, o);
  *status = b->init(p);
  if (*status != SRL_OK) return nullptr;
  return b;
}

}  // namespace srl
