// toy.cu -- device backend for the reference's exactly-evaluable policies
// (TabularPolicy, RecurrentToyPolicy) in fp64.  One CTA per stream slot per
// round; every reduction whose order matters to the reference (logit
// accumulation, log-sum-exp, inverse-CDF walk, recurrent update) is done in
// the reference's sequential order with FMA contraction disabled
// (__dmul_rn/__dadd_rn), so tokens and version stamps match the reference
// bit for bit and log-probs to the last ulp of the libm differences.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "runtime.hpp"

namespace srl {
namespace {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ULL;
constexpr int kToyThreads = 256;

__device__ __forceinline__ double draw_uniform(uint64_t seed, uint64_t n) {
  uint64_t z = seed + (n + 1) * kGolden;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  z ^= z >> 31;
  return (double)(z >> 11) * 0x1.0p-53;
}

struct ToyDevice {
  int type, V, D, order, n_rows, has_default, max_len;
  // recurrent
  const double *emb, *rec, *out;
  // tabular
  const int32_t *row_prompt, *row_ctx_len, *row_ctx;
  const double *row_logits, *default_logits;
  // slots
  int32_t *live, *gen, *max_tokens, *terminator, *prompt_idx, *history;
  uint64_t* seed;
  double* state;  // [slots x D]
  // ring
  int32_t *ev_flag, *ev_token, *ev_pos, *ev_version;
  double* ev_logprob;
  int ring_rounds;
  const int32_t* version;
};

// log-softmax in the reference order (numeric.hpp:13-27): thread 0 scans.
__device__ void log_softmax_seq(double* row, int V, double* lse_out) {
  if (threadIdx.x == 0) {
    double m = -INFINITY;
    for (int k = 0; k < V; ++k) m = row[k] > m ? row[k] : m;
    double lse = m;
    if (isfinite(m)) {
      double s = 0.0;
      for (int k = 0; k < V; ++k) s = __dadd_rn(s, exp(__dadd_rn(row[k], -m)));
      lse = __dadd_rn(m, log(s));
    }
    *lse_out = lse;
  }
  __syncthreads();
  const double lse = *lse_out;
  for (int k = threadIdx.x; k < V; k += blockDim.x) row[k] = __dadd_rn(row[k], -lse);
  __syncthreads();
}

// RecurrentToyPolicy::advance_state (policy.cpp:84-95)
__device__ void rec_advance(const ToyDevice& t, double* h, double* scratch, int token) {
  for (int i = threadIdx.x; i < t.D; i += blockDim.x) {
    double acc = t.emb[(size_t)token * t.D + i];
    const double* w = t.rec + (size_t)i * t.D;
    for (int j = 0; j < t.D; ++j) acc = __dadd_rn(acc, __dmul_rn(w[j], h[j]));
    scratch[i] = tanh(acc);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < t.D; i += blockDim.x) h[i] = scratch[i];
  __syncthreads();
}

// next_token_logprobs for either policy type into lp[V]
__device__ void toy_logprobs(const ToyDevice& t, int slot, const double* h, const int32_t* prefix,
                             int n, double* lp, double* lse_scratch) {
  if (t.type == SRL_POLICY_RECURRENT) {
    // policy.cpp:104-113: logits[k] = sum_i h_i * W[i, k], i ascending
    for (int k = threadIdx.x; k < t.V; k += blockDim.x) {
      double acc = 0.0;
      for (int i = 0; i < t.D; ++i) acc = __dadd_rn(acc, __dmul_rn(h[i], t.out[(size_t)i * t.V + k]));
      lp[k] = acc;
    }
    __syncthreads();
  } else {
    // policy.cpp:44-69: (prompt, last min(order, n) tokens) -> row, else default/uniform
    __shared__ int s_row;
    if (threadIdx.x == 0) {
      const int window = t.order < n ? t.order : n;
      const int32_t* ctx = prefix + (n - window);
      int found = -1;
      for (int r = 0; r < t.n_rows && found < 0; ++r) {
        if (t.row_prompt[r] != t.prompt_idx[slot] || t.row_ctx_len[r] != window) continue;
        bool same = true;
        for (int j = 0; j < window; ++j)
          if (t.row_ctx[(size_t)r * t.order + j] != ctx[j]) { same = false; break; }
        if (same) found = r;
      }
      s_row = found;
    }
    __syncthreads();
    const int r = s_row;
    for (int k = threadIdx.x; k < t.V; k += blockDim.x)
      lp[k] = r >= 0 ? t.row_logits[(size_t)r * t.V + k] : (t.has_default ? t.default_logits[k] : 0.0);
    __syncthreads();
  }
  log_softmax_seq(lp, t.V, lse_scratch);
}

// One round of Engine::run_round_locked (engine.cpp:119-153) per slot.
__global__ void __launch_bounds__(kToyThreads) toy_round_kernel(ToyDevice t, int slots, int ring_index) {
  extern __shared__ double sm[];
  double* lp = sm;              // V
  double* h = sm + t.V;         // D
  double* scratch = h + t.D;    // D
  __shared__ double s_lse;
  __shared__ int s_tok;
  const int s = blockIdx.x;
  const size_t ev = (size_t)ring_index * slots + s;
  if (t.live[s] == 0) {
    if (threadIdx.x == 0) t.ev_flag[ev] = 0;
    return;
  }
  const int n = t.gen[s];
  const int32_t* prefix = t.history + (size_t)s * t.max_len;
  double* gstate = t.state + (size_t)s * t.D;
  if (t.type == SRL_POLICY_RECURRENT) {
    for (int i = threadIdx.x; i < t.D; i += blockDim.x) h[i] = gstate[i];
    __syncthreads();
  }
  toy_logprobs(t, s, h, prefix, n, lp, &s_lse);
  if (threadIdx.x == 0) {
    // probs = exp(lp) then sequential inverse CDF (engine.cpp:130-132, rng.hpp:61-69)
    const double u = draw_uniform(t.seed[s], (uint64_t)n);
    double cum = 0.0;
    int tok = t.V - 1;
    for (int k = 0; k < t.V; ++k) {
      cum = __dadd_rn(cum, exp(lp[k]));
      if (u < cum) { tok = k; break; }
    }
    s_tok = tok;
    int flag = 1;
    if (tok == t.terminator[s]) flag = 3;
    else if (n + 1 >= t.max_tokens[s]) flag = 2;
    t.ev_flag[ev] = flag;
    t.ev_token[ev] = tok;
    t.ev_pos[ev] = n;
    t.ev_version[ev] = *t.version;
    t.ev_logprob[ev] = lp[tok];
    t.history[(size_t)s * t.max_len + n] = tok;
    t.gen[s] = n + 1;
    if (flag != 1) t.live[s] = 0;
  }
  __syncthreads();
  if (t.type == SRL_POLICY_RECURRENT) {
    rec_advance(t, h, scratch, s_tok);
    for (int i = threadIdx.x; i < t.D; i += blockDim.x) gstate[i] = h[i];
  }
}

// Recompute mode (engine.cpp:107-113): state = state_for_prefix(tokens).
__global__ void __launch_bounds__(kToyThreads) toy_recompute_kernel(ToyDevice t) {
  extern __shared__ double sm[];
  double* h = sm;
  double* scratch = sm + t.D;
  const int s = blockIdx.x;
  if (t.live[s] == 0) return;
  for (int i = threadIdx.x; i < t.D; i += blockDim.x) h[i] = 0.0;
  __syncthreads();
  const int n = t.gen[s];
  for (int p = 0; p < n; ++p) rec_advance(t, h, scratch, t.history[(size_t)s * t.max_len + p]);
  for (int i = threadIdx.x; i < t.D; i += blockDim.x) t.state[(size_t)s * t.D + i] = h[i];
}

// policy_logprobs (rl_math.cpp:128-142) for one sequence, one CTA.
__global__ void __launch_bounds__(kToyThreads) toy_seq_logprobs_kernel(ToyDevice t, const int32_t* tokens,
                                                             int n, int prompt_idx, double* out) {
  extern __shared__ double sm[];
  double* lp = sm;
  double* h = sm + t.V;
  double* scratch = h + t.D;
  __shared__ double s_lse;
  // the tabular lookup reads prompt_idx[slot]; use a one-slot view
  for (int i = threadIdx.x; i < t.D; i += blockDim.x) h[i] = 0.0;
  if (threadIdx.x == 0) t.prompt_idx[0] = prompt_idx;
  __syncthreads();
  for (int p = 0; p < n; ++p) {
    toy_logprobs(t, 0, h, tokens, p, lp, &s_lse);
    if (threadIdx.x == 0) out[p] = lp[tokens[p]];
    __syncthreads();
    if (t.type == SRL_POLICY_RECURRENT) rec_advance(t, h, scratch, tokens[p]);
  }
}

template <typename T>
int upload(T** dst, const std::vector<T>& src) {
  *dst = nullptr;
  if (src.empty()) return SRL_OK;
  SRL_CUDA(cudaMalloc(dst, src.size() * sizeof(T)));
  SRL_CUDA(cudaMemcpy(*dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice));
  return SRL_OK;
}

// Device copy of a toy policy's weights (tabular rows keyed by interned prompt ids).
struct ToyWeights {
  double *emb = nullptr, *rec = nullptr, *out = nullptr;
  int32_t *row_prompt = nullptr, *row_ctx_len = nullptr, *row_ctx = nullptr;
  double *row_logits = nullptr, *default_logits = nullptr;
  int n_rows = 0, has_default = 0, order = 0;
  void release() {
    for (void* p : {(void*)emb, (void*)rec, (void*)out, (void*)row_prompt, (void*)row_ctx_len,
                    (void*)row_ctx, (void*)row_logits, (void*)default_logits})
      if (p) cudaFree(p);
    *this = ToyWeights{};
  }
  int load(const Policy& p, Backend& b) {
    if (p.type == SRL_POLICY_RECURRENT) {
      int st;
      if ((st = upload(&emb, p.rec.emb)) || (st = upload(&rec, p.rec.rec)) || (st = upload(&out, p.rec.out)))
        return st;
      return SRL_OK;
    }
    const TabularHost& t = p.tab;
    n_rows = (int)t.rows.size();
    order = t.order;
    std::vector<int32_t> rp, rl, rc((size_t)std::max(1, n_rows) * std::max(1, t.order), 0);
    std::vector<double> lg;
    for (int r = 0; r < n_rows; ++r) {
      rp.push_back(b.intern(t.rows[r].prompt_id));
      rl.push_back((int32_t)t.rows[r].context.size());
      for (size_t j = 0; j < t.rows[r].context.size(); ++j) rc[(size_t)r * t.order + j] = t.rows[r].context[j];
      lg.insert(lg.end(), t.rows[r].logits.begin(), t.rows[r].logits.end());
    }
    has_default = t.default_logits.empty() ? 0 : 1;
    int st;
    if ((st = upload(&row_prompt, rp)) || (st = upload(&row_ctx_len, rl)) ||
        (st = upload(&row_ctx, rc)) || (st = upload(&row_logits, lg)) ||
        (st = upload(&default_logits, t.default_logits)))
      return st;
    return SRL_OK;
  }
};

class ToyBackend final : public Backend {
 public:
  ToyBackend(const Policy& p, const srl_engine_options& o) : type_(p.type), opts_(o) {
    V_ = p.vocab();
    D_ = p.type == SRL_POLICY_RECURRENT ? p.rec.hidden : 1;
    S_ = std::max(1, o.max_streams);
    max_len_ = std::max(2, o.max_seq_len);
    R_ = std::max(o.event_ring, std::max(1, o.rounds_per_sync));
  }
  ~ToyBackend() override {
    cudaStreamSynchronize(st_);
    w_.release();
    for (void* p : allocs_) cudaFree(p);
    if (pinned_) cudaFreeHost(pinned_);
    if (st_) cudaStreamDestroy(st_);
  }

  int init(const Policy& p) {
    SRL_CUDA(cudaSetDevice(opts_.device));
    SRL_CUDA(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
    int st;
    if ((st = w_.load(p, *this))) return st;
    auto alloc = [&](auto** ptr, size_t n) -> int {
      SRL_CUDA(cudaMalloc(ptr, n * sizeof(**ptr)));
      SRL_CUDA(cudaMemset(*ptr, 0, n * sizeof(**ptr)));
      allocs_.push_back(*ptr);
      return SRL_OK;
    };
    if ((st = alloc(&live_, S_)) || (st = alloc(&gen_, S_)) || (st = alloc(&maxtok_, S_)) ||
        (st = alloc(&term_, S_)) || (st = alloc(&pidx_, S_)) || (st = alloc(&seed_, S_)) ||
        (st = alloc(&hist_, (size_t)S_ * max_len_)) || (st = alloc(&state_, (size_t)S_ * D_)) ||
        (st = alloc(&ev_flag_, (size_t)R_ * S_)) || (st = alloc(&ev_tok_, (size_t)R_ * S_)) ||
        (st = alloc(&ev_pos_, (size_t)R_ * S_)) || (st = alloc(&ev_ver_, (size_t)R_ * S_)) ||
        (st = alloc(&ev_lp_, (size_t)R_ * S_)) || (st = alloc(&version_, 1)) ||
        (st = alloc(&scratch_prompt_, 1)))
      return st;
    SRL_CUDA(cudaMallocHost(&pinned_, (size_t)R_ * S_ * (4 * sizeof(int32_t) + sizeof(double))));
    const size_t smem = sizeof(double) * ((size_t)V_ + 2 * (size_t)D_);
    if (smem > 48 * 1024) {
      SRL_CUDA(cudaFuncSetAttribute(toy_round_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      SRL_CUDA(cudaFuncSetAttribute(toy_seq_logprobs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      SRL_CUDA(cudaFuncSetAttribute(toy_recompute_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    }
    return SRL_OK;
  }

  int slots() const override { return S_; }

  int open_slot(int slot, const StreamSpec& spec) override {
    if (spec.max_tokens > max_len_)
      return fail(SRL_INVALID_ARGUMENT, "max_tokens exceeds the engine's max_seq_len");
    const int32_t one = 1, zero = 0;
    const int32_t pidx = spec.prompt_index;
    SRL_CUDA(cudaMemcpyAsync(live_ + slot, &one, 4, cudaMemcpyHostToDevice, st_));
    SRL_CUDA(cudaMemcpyAsync(gen_ + slot, &zero, 4, cudaMemcpyHostToDevice, st_));
    SRL_CUDA(cudaMemcpyAsync(maxtok_ + slot, &spec.max_tokens, 4, cudaMemcpyHostToDevice, st_));
    SRL_CUDA(cudaMemcpyAsync(term_ + slot, &spec.terminator, 4, cudaMemcpyHostToDevice, st_));
    SRL_CUDA(cudaMemcpyAsync(pidx_ + slot, &pidx, 4, cudaMemcpyHostToDevice, st_));
    SRL_CUDA(cudaMemcpyAsync(seed_ + slot, &spec.seed, 8, cudaMemcpyHostToDevice, st_));
    SRL_CUDA(cudaMemsetAsync(state_ + (size_t)slot * D_, 0, sizeof(double) * D_, st_));
    SRL_CUDA(cudaStreamSynchronize(st_));  // the host-side sources are stack temporaries
    gen_host_.resize(S_, 0);
    gen_host_[slot] = 0;
    return SRL_OK;
  }

  void close_slot(int slot) override {
    const int32_t zero = 0;
    cudaMemcpyAsync(live_ + slot, &zero, 4, cudaMemcpyHostToDevice, st_);
    cudaStreamSynchronize(st_);
  }

  ToyDevice view() const {
    ToyDevice t{};
    t.type = type_; t.V = V_; t.D = D_; t.order = w_.order; t.n_rows = w_.n_rows;
    t.has_default = w_.has_default; t.max_len = max_len_;
    t.emb = w_.emb; t.rec = w_.rec; t.out = w_.out;
    t.row_prompt = w_.row_prompt; t.row_ctx_len = w_.row_ctx_len; t.row_ctx = w_.row_ctx;
    t.row_logits = w_.row_logits; t.default_logits = w_.default_logits;
    t.live = live_; t.gen = gen_; t.max_tokens = maxtok_; t.terminator = term_;
    t.prompt_idx = pidx_; t.history = hist_; t.seed = seed_; t.state = state_;
    t.ev_flag = ev_flag_; t.ev_token = ev_tok_; t.ev_pos = ev_pos_; t.ev_version = ev_ver_;
    t.ev_logprob = ev_lp_; t.ring_rounds = R_; t.version = version_;
    return t;
  }

  int run_rounds(int n, std::vector<SlotEvent>& events, double* device_ms) override {
    events.assign((size_t)n * S_, SlotEvent{});
    const ToyDevice t = view();
    const size_t smem = sizeof(double) * ((size_t)V_ + 2 * (size_t)D_);
    for (int done = 0; done < n;) {
      const int batch = std::min(n - done, R_);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0, st_);
      for (int r = 0; r < batch; ++r) toy_round_kernel<<<S_, kToyThreads, smem, st_>>>(t, S_, r);
      launches_ += batch;
      cudaEventRecord(e1, st_);
      const size_t cnt = (size_t)batch * S_;
      int32_t* pf = static_cast<int32_t*>(pinned_);
      int32_t* pt = pf + cnt;
      int32_t* pp = pt + cnt;
      int32_t* pv = pp + cnt;
      double* pl = reinterpret_cast<double*>(pv + cnt + (cnt & 1));
      SRL_CUDA(cudaMemcpyAsync(pf, ev_flag_, cnt * 4, cudaMemcpyDeviceToHost, st_));
      SRL_CUDA(cudaMemcpyAsync(pt, ev_tok_, cnt * 4, cudaMemcpyDeviceToHost, st_));
      SRL_CUDA(cudaMemcpyAsync(pp, ev_pos_, cnt * 4, cudaMemcpyDeviceToHost, st_));
      SRL_CUDA(cudaMemcpyAsync(pv, ev_ver_, cnt * 4, cudaMemcpyDeviceToHost, st_));
      SRL_CUDA(cudaMemcpyAsync(pl, ev_lp_, cnt * 8, cudaMemcpyDeviceToHost, st_));
      SRL_CUDA(cudaStreamSynchronize(st_));
      SRL_CUDA(cudaGetLastError());
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
      if (device_ms) *device_ms += ms;
      for (size_t i = 0; i < cnt; ++i) {
        SlotEvent& e = events[(size_t)done * S_ + i];
        e.flag = pf[i]; e.token = pt[i]; e.position = pp[i]; e.version = pv[i]; e.logprob = pl[i];
      }
      done += batch;
    }
    return SRL_OK;
  }

  int check_update(const Policy& p) override {
    if (p.type == SRL_POLICY_RECURRENT && p.rec.hidden != D_)
      return fail(SRL_POLICY_MISMATCH, "policy_mismatch: recurrent hidden_dim differs");
    return SRL_OK;
  }

  int apply_update(const Policy& p, bool recompute, int version) override {
    ToyWeights fresh;
    int st = fresh.load(p, *this);
    if (st != SRL_OK) { fresh.release(); return st; }
    SRL_CUDA(cudaStreamSynchronize(st_));
    w_.release();
    w_ = fresh;
    SRL_CUDA(cudaMemcpyAsync(version_, &version, 4, cudaMemcpyHostToDevice, st_));
    if (recompute && type_ == SRL_POLICY_RECURRENT) {
      const size_t smem = sizeof(double) * ((size_t)V_ + 2 * (size_t)D_);
      toy_recompute_kernel<<<S_, kToyThreads, smem, st_>>>(view());
    }
    SRL_CUDA(cudaStreamSynchronize(st_));
    SRL_CUDA(cudaGetLastError());
    return SRL_OK;
  }

  int slot_history(int slot, std::vector<int32_t>& out) override {
    int32_t n = 0;
    SRL_CUDA(cudaMemcpyAsync(&n, gen_ + slot, 4, cudaMemcpyDeviceToHost, st_));
    SRL_CUDA(cudaStreamSynchronize(st_));
    out.assign(n, 0);
    if (n > 0) {
      SRL_CUDA(cudaMemcpyAsync(out.data(), hist_ + (size_t)slot * max_len_, 4 * (size_t)n,
                               cudaMemcpyDeviceToHost, st_));
      SRL_CUDA(cudaStreamSynchronize(st_));
    }
    return SRL_OK;
  }

  // policy_logprobs for toy policies (single sequence on the device).
  int seq_logprobs(const std::vector<int32_t>& tokens, int prompt_idx, std::vector<double>& out) {
    const int n = (int)tokens.size();
    out.assign(n, 0.0);
    if (n == 0) return SRL_OK;
    int32_t* dtok = nullptr;
    double* dout = nullptr;
    SRL_CUDA(cudaMalloc(&dtok, 4 * (size_t)n));
    SRL_CUDA(cudaMalloc(&dout, 8 * (size_t)n));
    SRL_CUDA(cudaMemcpy(dtok, tokens.data(), 4 * (size_t)n, cudaMemcpyHostToDevice));
    const size_t smem = sizeof(double) * ((size_t)V_ + 2 * (size_t)D_);
    ToyDevice t = view();
    t.prompt_idx = scratch_prompt_;
    toy_seq_logprobs_kernel<<<1, kToyThreads, smem, st_>>>(t, dtok, n, prompt_idx, dout);
    SRL_CUDA(cudaStreamSynchronize(st_));
    SRL_CUDA(cudaGetLastError());
    SRL_CUDA(cudaMemcpy(out.data(), dout, 8 * (size_t)n, cudaMemcpyDeviceToHost));
    cudaFree(dtok);
    cudaFree(dout);
    return SRL_OK;
  }

 private:
  int type_;
  srl_engine_options opts_;
  int V_ = 0, D_ = 1, S_ = 1, max_len_ = 2, R_ = 1;
  cudaStream_t st_ = nullptr;
  ToyWeights w_;
  int32_t *live_ = nullptr, *gen_ = nullptr, *maxtok_ = nullptr, *term_ = nullptr, *pidx_ = nullptr;
  int32_t* hist_ = nullptr;
  uint64_t* seed_ = nullptr;
  double* state_ = nullptr;
  int32_t *ev_flag_ = nullptr, *ev_tok_ = nullptr, *ev_pos_ = nullptr, *ev_ver_ = nullptr;
  double* ev_lp_ = nullptr;
  int32_t* version_ = nullptr;
  int32_t* scratch_prompt_ = nullptr;
  void* pinned_ = nullptr;
  std::vector<void*> allocs_;
  std::vector<int32_t> gen_host_;
};

}  // namespace

std::unique_ptr<Backend> make_toy_backend(const Policy& p, const srl_engine_options& o, int* status) {
  auto b = std::make_unique<ToyBackend>(p, o);
  *status = b->init(p);
  if (*status != SRL_OK) return nullptr;
  return b;
}

int toy_policy_logprobs(const Policy& p, const std::string& prompt_id,
                        const std::vector<int32_t>& tokens, std::vector<double>& out, int device) {
  srl_engine_options o{};
  o.max_streams = 1;
  o.max_seq_len = 2;
  o.rounds_per_sync = 1;
  o.event_ring = 1;
  o.device = device;
  ToyBackend b(p, o);
  const int st = b.init(p);
  if (st != SRL_OK) return st;
  return b.seq_logprobs(tokens, b.intern(prompt_id), out);
}

}  // namespace srl
