// capi.cpp -- extern "C" entry points of include/streamrl_b200.h over the C++
// runtime.  Every function validates its arguments, maps failures to the
// reference's error strings (srl_status) and never throws across the ABI.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "capi_handles.hpp"
#include "decoder_engine.hpp"

namespace srl {
int toy_policy_logprobs(const Policy& p, const std::string& prompt_id,
                        const std::vector<int32_t>& tokens, std::vector<double>& out, int device);
int decoder_policy_logprobs(const DecoderWeights& w, const std::vector<int32_t>& tokens,
                            std::vector<double>& out);
int decoder_kl_per_position(const std::vector<const DecoderWeights*>& ck, const std::vector<int>& switch_points,
                            bool recompute, const DecoderWeights& target,
                            const std::vector<std::vector<int32_t>>& prefixes, std::vector<double>& out);
int tabular_is_reinforce_gradient(const Policy& p, int n_traj, const char* const* prompt_ids,
                                  const int32_t* tokens, const int64_t* offsets, const double* mu,
                                  const double* rewards, const double* baseline, bool use_is, double clamp,
                                  int granularity, double* grad_out, int32_t* touched_out, int device);
}  // namespace srl

using namespace srl;

namespace {

int require_device(int device) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) return fail(SRL_NO_DEVICE, "no CUDA device visible");
  if (device < 0 || device >= n) return fail(SRL_INVALID_ARGUMENT, "device index out of range");
  return SRL_OK;
}

srl_engine_options default_options() {
  srl_engine_options o{};
  o.max_streams = 64;
  o.max_seq_len = 1024;
  o.greedy = 0;
  o.rounds_per_sync = 8;
  o.use_graphs = 1;
  o.device = 0;
  o.event_ring = 64;
  o.prefill_budget = 4096;
  return o;
}

template <typename F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const std::bad_alloc&) {
    return fail(SRL_OUT_OF_MEMORY, "host allocation failed");
  } catch (const std::exception& ex) {
    return fail(SRL_INVALID_ARGUMENT, ex.what());
  }
}

}  // namespace

// ------------------------------------------------------------ policies ---
extern "C" int srl_policy_tabular_create(int32_t vocab_size, int32_t context_order,
                                         const double* default_logits, int32_t n_rows,
                                         const char* const* row_prompt_ids,
                                         const int32_t* row_context_lens,
                                         const int32_t* row_contexts, const double* row_logits,
                                         srl_policy** out) {
  return guarded([&] {
    if (!out || n_rows < 0 || (n_rows > 0 && (!row_prompt_ids || !row_context_lens || !row_logits)))
      return fail(SRL_INVALID_ARGUMENT, "tabular_create: bad arguments");
    auto h = std::make_unique<srl_policy>();
    h->p.type = SRL_POLICY_TABULAR;
    TabularHost& t = h->p.tab;
    t.vocab = vocab_size;
    t.order = context_order;
    if (default_logits && vocab_size > 0) t.default_logits.assign(default_logits, default_logits + vocab_size);
    for (int r = 0; r < n_rows; ++r) {
      TabularRow row;
      row.prompt_id = row_prompt_ids[r] ? row_prompt_ids[r] : "";
      const int cl = row_context_lens[r];
      if (cl < 0 || (cl > 0 && !row_contexts)) return fail(SRL_INVALID_ARGUMENT, "bad context length");
      if (cl > context_order)  // policy.cpp:35-36
        return fail(SRL_INVALID_POLICY, "TabularPolicy: context longer than context_order");
      for (int j = 0; j < cl; ++j) row.context.push_back(row_contexts[(size_t)r * context_order + j]);
      if (vocab_size > 0) row.logits.assign(row_logits + (size_t)r * vocab_size, row_logits + (size_t)(r + 1) * vocab_size);
      t.rows.push_back(std::move(row));
    }
    // std::map<ContextKey> order: (prompt_id, context) lexicographic
    std::sort(t.rows.begin(), t.rows.end(), [](const TabularRow& a, const TabularRow& b) {
      if (a.prompt_id != b.prompt_id) return a.prompt_id < b.prompt_id;
      return a.context < b.context;
    });
    std::string why;
    if (h->p.validate(&why) != SRL_OK) return fail(SRL_INVALID_POLICY, why);
    *out = h.release();
    return (int)SRL_OK;
  });
}

extern "C" int srl_policy_recurrent_create(int32_t vocab_size, int32_t hidden_dim,
                                           const double* input_embedding, const double* recurrence,
                                           const double* output, srl_policy** out) {
  return guarded([&] {
    if (!out || !input_embedding || !recurrence || !output || vocab_size < 1 || hidden_dim < 1)
      return fail(SRL_INVALID_POLICY, "recurrent_create: bad arguments");
    auto h = std::make_unique<srl_policy>();
    h->p.type = SRL_POLICY_RECURRENT;
    RecurrentHost& r = h->p.rec;
    r.vocab = vocab_size;
    r.hidden = hidden_dim;
    r.emb.assign(input_embedding, input_embedding + (size_t)vocab_size * hidden_dim);
    r.rec.assign(recurrence, recurrence + (size_t)hidden_dim * hidden_dim);
    r.out.assign(output, output + (size_t)hidden_dim * vocab_size);
    std::string why;
    if (h->p.validate(&why) != SRL_OK) return fail(SRL_INVALID_POLICY, why);
    *out = h.release();
    return (int)SRL_OK;
  });
}

extern "C" size_t srl_decoder_weight_bytes(const srl_decoder_config* cfg) {
  if (!cfg) return 0;
  const DecoderDims d = dims_from(*cfg);
  if (!dims_valid(d, nullptr)) return 0;
  WeightLayout lay;
  const size_t n = make_layout(d, lay);
  delete[] lay.layers;
  return n * sizeof(__nv_bfloat16);
}

extern "C" int srl_policy_decoder_create(const srl_decoder_config* cfg, uint64_t init_seed,
                                         double init_scale, int32_t device, srl_policy** out) {
  return guarded([&] {
    if (!cfg || !out) return fail(SRL_INVALID_ARGUMENT, "decoder_create: null argument");
    int st;
    if ((st = require_device(device))) return st;
    auto h = std::make_unique<srl_policy>();
    h->p.type = SRL_POLICY_DECODER;
    if ((st = create_decoder(*cfg, device, h->p.dec))) return st;
    launch_init_weights(h->p.dec->w, h->p.dec->dims, h->p.dec->layout, init_seed, init_scale, 0);
    SRL_CUDA(cudaDeviceSynchronize());
    SRL_CUDA(cudaGetLastError());
    *out = h.release();
    return (int)SRL_OK;
  });
}

extern "C" int srl_policy_decoder_from_buffer(const srl_decoder_config* cfg, const void* weights,
                                              size_t nbytes, int32_t on_device, int32_t device,
                                              srl_policy** out) {
  return guarded([&] {
    if (!cfg || !out || !weights) return fail(SRL_INVALID_ARGUMENT, "decoder_from_buffer: null argument");
    int st;
    if ((st = require_device(device))) return st;
    auto h = std::make_unique<srl_policy>();
    h->p.type = SRL_POLICY_DECODER;
    if ((st = create_decoder(*cfg, device, h->p.dec))) return st;
    if (nbytes != h->p.dec->bytes) return fail(SRL_INVALID_POLICY, "decoder weight buffer size mismatch");
    SRL_CUDA(cudaMemcpy(h->p.dec->w, weights, nbytes,
                        on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice));
    *out = h.release();
    return (int)SRL_OK;
  });
}

extern "C" int srl_policy_decoder_device(const srl_policy* p, int32_t* device) {
  if (!p || !device || p->p.type != SRL_POLICY_DECODER || !p->p.dec)
    return fail(SRL_INVALID_ARGUMENT, "not a decoder policy");
  *device = p->p.dec->device;
  return SRL_OK;
}

extern "C" int srl_policy_decoder_weights(const srl_policy* p, void** device_ptr, size_t* nbytes) {
  if (!p || p->p.type != SRL_POLICY_DECODER || !p->p.dec) return fail(SRL_INVALID_ARGUMENT, "not a decoder policy");
  if (device_ptr) *device_ptr = p->p.dec->w;
  if (nbytes) *nbytes = p->p.dec->bytes;
  return SRL_OK;
}

extern "C" int srl_policy_decoder_offset(const srl_policy* p, const char* name, size_t* offset) {
  if (!p || !name || !offset || p->p.type != SRL_POLICY_DECODER) return fail(SRL_INVALID_ARGUMENT, "decoder_offset");
  const WeightLayout& L = p->p.dec->layout;
  const std::string n(name);
  if (n == "embed") { *offset = L.embed; return SRL_OK; }
  if (n == "final_norm") { *offset = L.final_norm; return SRL_OK; }
  if (n == "lm_head") { *offset = L.lm_head; return SRL_OK; }
  const size_t dot = n.find('.');
  if (dot == std::string::npos) return fail(SRL_INVALID_ARGUMENT, "unknown tensor name");
  const int l = std::atoi(n.substr(0, dot).c_str());
  if (l < 0 || l >= p->p.dec->dims.L) return fail(SRL_INVALID_ARGUMENT, "layer out of range");
  const std::string t = n.substr(dot + 1);
  const LayerOffsets& o = L.layers[l];
  if (t == "ln1") *offset = o.ln1;
  else if (t == "qkv_w") *offset = o.qkv_w;
  else if (t == "qkv_b") *offset = o.qkv_b;
  else if (t == "o_w") *offset = o.o_w;
  else if (t == "ln2") *offset = o.ln2;
  else if (t == "gate_up_w") *offset = o.gate_up_w;
  else if (t == "down_w") *offset = o.down_w;
  else return fail(SRL_INVALID_ARGUMENT, "unknown tensor name");
  return SRL_OK;
}

extern "C" int srl_policy_decoder_perturb(srl_policy* p, uint64_t seed, double magnitude) {
  if (!p || p->p.type != SRL_POLICY_DECODER) return fail(SRL_INVALID_ARGUMENT, "not a decoder policy");
  launch_perturb(p->p.dec->w, p->p.dec->layout.total, seed, magnitude, 0);
  SRL_CUDA(cudaDeviceSynchronize());
  SRL_CUDA(cudaGetLastError());
  return SRL_OK;
}

extern "C" int srl_policy_type(const srl_policy* p) { return p ? p->p.type : -1; }
extern "C" int32_t srl_policy_vocab_size(const srl_policy* p) { return p ? p->p.vocab() : 0; }
extern "C" int srl_policy_validate(const srl_policy* p) {
  if (!p) return fail(SRL_INVALID_ARGUMENT, "null policy");
  std::string why;
  const int st = p->p.validate(&why);
  return st == SRL_OK ? SRL_OK : fail(st, why);
}
extern "C" void srl_policy_destroy(srl_policy* p) { delete p; }

// -------------------------------------------------------------- engine ---
extern "C" int srl_engine_create(const srl_policy* policy, int32_t recompute_state,
                                 int32_t start_paused, const srl_engine_options* opts,
                                 srl_engine** out) {
  return guarded([&] {
    if (!policy || !out) return fail(SRL_INVALID_ARGUMENT, "engine_create: null argument");
    std::string why;
    if (policy->p.validate(&why) != SRL_OK) return fail(SRL_INVALID_POLICY, why);  // engine.cpp:39
    srl_engine_options o = opts ? *opts : default_options();
    int st;
    if ((st = require_device(o.device))) return st;
    if (o.max_streams < 1 || o.max_seq_len < 2 || o.rounds_per_sync < 1)
      return fail(SRL_INVALID_ARGUMENT, "engine options out of range");
    if (o.event_ring < o.rounds_per_sync) o.event_ring = o.rounds_per_sync;
    if (o.prefill_budget < 1) o.prefill_budget = o.max_seq_len;
    std::unique_ptr<Backend> b = policy->p.type == SRL_POLICY_DECODER
                                     ? make_decoder_backend(policy->p, o, &st)
                                     : make_toy_backend(policy->p, o, &st);
    if (!b) return st;
    auto h = std::make_unique<srl_engine>();
    Policy pol = policy->p;
    h->e = std::make_unique<Engine>(std::move(b), std::move(pol), recompute_state != 0,
                                    start_paused != 0, o);
    *out = h.release();
    return (int)SRL_OK;
  });
}

extern "C" void srl_engine_destroy(srl_engine* e) { delete e; }

extern "C" int srl_engine_open_stream(srl_engine* e, const char* prompt_id, int32_t max_tokens,
                                      uint64_t seed, int32_t terminator_token,
                                      const int32_t* prompt_tokens, int32_t n_prompt,
                                      int64_t* stream_out) {
  return guarded([&] {
    if (!e || !stream_out || n_prompt < 0 || (n_prompt > 0 && !prompt_tokens))
      return fail(SRL_INVALID_ARGUMENT, "open_stream: bad arguments");
    std::vector<int32_t> pr(prompt_tokens, prompt_tokens + n_prompt);
    return e->e->open_stream(prompt_id ? prompt_id : "", max_tokens, seed, terminator_token, pr,
                             stream_out);
  });
}

extern "C" int srl_engine_wait_events(srl_engine* e, int64_t stream, srl_token_event* buf,
                                      int32_t cap, int32_t* n_out, int32_t* finish_reason,
                                      int32_t* more) {
  return guarded([&] {
    if (!e || !buf || cap < 1 || !n_out || !finish_reason || !more)
      return fail(SRL_INVALID_ARGUMENT, "wait_events: bad arguments");
    std::vector<srl_token_event> out;
    int reason = 0, m = 0;
    const int st = e->e->wait_events(stream, out, cap, &reason, &m);
    if (st != SRL_OK) return st;
    std::copy(out.begin(), out.end(), buf);
    *n_out = (int32_t)out.size();
    *finish_reason = reason;
    *more = m;
    return (int)SRL_OK;
  });
}

namespace {
int events_many(srl_engine* e, const int64_t* streams, int32_t n_streams, srl_token_event* buf, int32_t cap,
                int32_t* counts, int32_t* finish_reasons, int32_t* more, bool block) {
  return guarded([&] {
    if (!e || !streams || n_streams < 0 || !buf || cap < 1 || !counts || !finish_reasons || !more)
      return fail(SRL_INVALID_ARGUMENT, "wait_events_many: bad arguments");
    int32_t used = 0;
    std::vector<srl_token_event> out;
    for (int32_t i = 0; i < n_streams; ++i) {
      int reason = 0, m = 0;
      out.clear();
      if (used < cap) {
        const int st = e->e->wait_events(streams[i], out, cap - used, &reason, &m, block);
        if (st != SRL_OK) return st;
      } else {
        m = 1;  // no room left: the stream keeps its events for the next call
      }
      std::copy(out.begin(), out.end(), buf + used);
      counts[i] = (int32_t)out.size();
      used += counts[i];
      finish_reasons[i] = reason;
      more[i] = m;
    }
    return (int)SRL_OK;
  });
}
}  // namespace

extern "C" int srl_engine_wait_events_many(srl_engine* e, const int64_t* streams, int32_t n_streams,
                                           srl_token_event* buf, int32_t cap, int32_t* counts,
                                           int32_t* finish_reasons, int32_t* more) {
  return events_many(e, streams, n_streams, buf, cap, counts, finish_reasons, more, true);
}

extern "C" int srl_engine_poll_events_many(srl_engine* e, const int64_t* streams, int32_t n_streams,
                                           srl_token_event* buf, int32_t cap, int32_t* counts,
                                           int32_t* finish_reasons, int32_t* more) {
  return events_many(e, streams, n_streams, buf, cap, counts, finish_reasons, more, false);
}

extern "C" int srl_engine_apply_weight_update(srl_engine* e, int32_t new_version,
                                              const srl_policy* policy, int32_t* version_out) {
  return guarded([&] {
    if (!e || !policy) return fail(SRL_INVALID_ARGUMENT, "apply_weight_update: null argument");
    int v = 0;
    const int st = e->e->apply_weight_update(new_version, policy->p, &v);
    if (version_out) *version_out = v;
    return st;
  });
}

extern "C" int srl_engine_begin_weight_update(srl_engine* e, int32_t new_version,
                                              void** standby_device_ptr, size_t* nbytes) {
  if (!e || !standby_device_ptr || !nbytes) return fail(SRL_INVALID_ARGUMENT, "begin_weight_update");
  return e->e->begin_weight_update(new_version, standby_device_ptr, nbytes);
}

extern "C" int srl_engine_commit_weight_update(srl_engine* e, int32_t new_version,
                                               int32_t* version_out, double* pause_ms) {
  if (!e) return fail(SRL_INVALID_ARGUMENT, "commit_weight_update");
  int v = 0;
  const int st = e->e->commit_weight_update(new_version, &v, pause_ms);
  if (version_out) *version_out = v;
  return st;
}

extern "C" int srl_engine_standby_bytes(srl_engine* e, size_t* nbytes) {
  if (!e || !nbytes) return fail(SRL_INVALID_ARGUMENT, "standby_bytes");
  return e->e->standby_bytes(nbytes);
}

extern "C" int srl_engine_abort_weight_update(srl_engine* e) {
  if (!e) return fail(SRL_INVALID_ARGUMENT, "abort_weight_update");
  return e->e->abort_weight_update();
}

extern "C" int srl_engine_advance(srl_engine* e, int32_t rounds, int64_t* emitted) {
  if (!e) return fail(SRL_INVALID_ARGUMENT, "advance");
  int64_t n = 0;
  const int st = e->e->advance(rounds, &n);
  if (emitted) *emitted = n;
  return st;
}

extern "C" int srl_engine_pause(srl_engine* e) {
  if (!e) return fail(SRL_INVALID_ARGUMENT, "pause");
  e->e->pause();
  return SRL_OK;
}
extern "C" int srl_engine_resume(srl_engine* e) {
  if (!e) return fail(SRL_INVALID_ARGUMENT, "resume");
  e->e->resume();
  return SRL_OK;
}
extern "C" int srl_engine_weight_version(const srl_engine* e, int32_t* out) {
  if (!e || !out) return fail(SRL_INVALID_ARGUMENT, "weight_version");
  *out = e->e->weight_version();
  return SRL_OK;
}
extern "C" int srl_engine_active_streams(const srl_engine* e, int32_t* out) {
  if (!e || !out) return fail(SRL_INVALID_ARGUMENT, "active_streams");
  *out = e->e->active_streams();
  return SRL_OK;
}
extern "C" int srl_engine_total_streams(const srl_engine* e, int64_t* out) {
  if (!e || !out) return fail(SRL_INVALID_ARGUMENT, "total_streams");
  *out = e->e->total_streams();
  return SRL_OK;
}
extern "C" int srl_engine_rounds_done(const srl_engine* e, int64_t* out) {
  if (!e || !out) return fail(SRL_INVALID_ARGUMENT, "rounds_done");
  *out = e->e->rounds_done();
  return SRL_OK;
}
extern "C" int srl_engine_recompute_state_mode(const srl_engine* e, int32_t* out) {
  if (!e || !out) return fail(SRL_INVALID_ARGUMENT, "recompute_state_mode");
  *out = e->e->recompute_state_mode() ? 1 : 0;
  return SRL_OK;
}
extern "C" int srl_engine_set_process_group(srl_engine* e, const char* group_id,
                                            const char* const* members, int32_t n_members) {
  if (!e || !group_id || n_members < 0 || (n_members > 0 && !members))
    return fail(SRL_INVALID_ARGUMENT, "set_process_group");
  std::vector<std::string> m;
  for (int i = 0; i < n_members; ++i) m.emplace_back(members[i] ? members[i] : "");
  e->e->set_process_group(group_id, std::move(m));
  return SRL_OK;
}
extern "C" int srl_engine_process_group_id(const srl_engine* e, char* buf, size_t cap,
                                           int32_t* has_group) {
  if (!e || !has_group) return fail(SRL_INVALID_ARGUMENT, "process_group_id");
  const auto g = e->e->process_group_id();
  *has_group = g.has_value() ? 1 : 0;
  if (g && buf && cap > 0) {
    const size_t n = std::min(cap - 1, g->size());
    std::memcpy(buf, g->data(), n);
    buf[n] = '\0';
  }
  return SRL_OK;
}
extern "C" int srl_engine_stop(srl_engine* e) {
  if (!e) return fail(SRL_INVALID_ARGUMENT, "stop");
  e->e->stop();
  return SRL_OK;
}
extern "C" int srl_engine_stream_tokens(srl_engine* e, int64_t stream, int32_t* buf, int32_t cap,
                                        int32_t* n_out) {
  if (!e || !n_out) return fail(SRL_INVALID_ARGUMENT, "stream_tokens");
  std::vector<int32_t> t;
  const int st = e->e->stream_tokens(stream, t);
  if (st != SRL_OK) return st;
  *n_out = (int32_t)t.size();
  if (buf) std::copy(t.begin(), t.begin() + std::min<size_t>(t.size(), std::max(cap, 0)), buf);
  return SRL_OK;
}
extern "C" int srl_engine_stats_get(const srl_engine* e, srl_engine_stats* out) {
  if (!e || !out) return fail(SRL_INVALID_ARGUMENT, "stats_get");
  *out = e->e->stats();
  return SRL_OK;
}

// -------------------------------------------------------- trainer math ---
extern "C" int srl_policy_logprobs(const srl_policy* p, const char* prompt_id,
                                   const int32_t* tokens, int32_t n, double* out) {
  return guarded([&] {
    if (!p || (n > 0 && (!tokens || !out)) || n < 0) return fail(SRL_INVALID_ARGUMENT, "policy_logprobs");
    std::string why;
    if (p->p.validate(&why) != SRL_OK) return fail(SRL_INVALID_POLICY, why);
    const int32_t V = p->p.vocab();
    for (int i = 0; i < n; ++i)  // check_tokens_in_vocab (rl_math.cpp:17-21)
      if (tokens[i] < 0 || tokens[i] >= V)
        return fail(SRL_INVALID_ARGUMENT, "token " + std::to_string(tokens[i]) + " out of vocab range");
    std::vector<int32_t> tk(tokens, tokens + n);
    std::vector<double> lp;
    int st;
    if (p->p.type == SRL_POLICY_DECODER) {
      if ((st = require_device(p->p.dec->device))) return st;
      st = decoder_policy_logprobs(*p->p.dec, tk, lp);
    } else {
      if ((st = require_device(0))) return st;
      st = toy_policy_logprobs(p->p, prompt_id ? prompt_id : "", tk, lp, 0);
    }
    if (st != SRL_OK) return st;
    std::copy(lp.begin(), lp.end(), out);
    return (int)SRL_OK;
  });
}

// truncated_is_weight (rl_math.cpp:144-150)
extern "C" int srl_truncated_is_weight(double pi_sum, double mu_sum, double clamp, double* out) {
  if (!out) return fail(SRL_INVALID_ARGUMENT, "null out");
  if (clamp <= 0.0 || !std::isfinite(clamp))
    return fail(SRL_INVALID_ARGUMENT, "truncated_is_weight: clamp must be positive");
  if (!std::isfinite(pi_sum) || !std::isfinite(mu_sum))
    return fail(SRL_INVALID_ARGUMENT, "truncated_is_weight: non-finite log-probability");
  *out = std::min(clamp, std::exp(pi_sum - mu_sum));
  return SRL_OK;
}

// is_reinforce_gradient for TabularPolicy (rl_math.cpp:211-276), tabular_grad.cu
extern "C" int srl_tabular_is_reinforce_gradient(const srl_policy* p, int32_t n_traj,
                                                 const char* const* prompt_ids, const int32_t* tokens,
                                                 const int64_t* offsets, const double* behavior_logprobs,
                                                 const double* rewards, const double* baseline, int32_t use_is,
                                                 double clamp, int32_t granularity, double* grad_rows,
                                                 int32_t* row_touched) {
  return guarded([&] {
    if (!p || !offsets || !rewards || !baseline || !grad_rows || !row_touched || !prompt_ids ||
        (use_is && !behavior_logprobs) || (granularity != 0 && granularity != 1))
      return fail(SRL_INVALID_ARGUMENT, "tabular_is_reinforce_gradient: bad arguments");
    if (p->p.type != SRL_POLICY_TABULAR) return fail(SRL_INVALID_ARGUMENT, "gradient: needs a tabular policy");
    std::string why;
    if (p->p.validate(&why) != SRL_OK) return fail(SRL_INVALID_POLICY, why);
    int st;
    if ((st = require_device(0))) return st;
    std::vector<double> zeros;
    if (!use_is) zeros.assign((size_t)std::max<int64_t>(0, offsets[std::max(0, n_traj)]), 0.0);
    return tabular_is_reinforce_gradient(p->p, n_traj, prompt_ids, tokens, offsets,
                                         use_is ? behavior_logprobs : zeros.data(), rewards, baseline,
                                         use_is != 0, clamp, granularity, grad_rows, row_touched, 0);
  });
}

// kl_per_position for the decoder policy (rl_math.cpp:336-372), kl.cpp
extern "C" int srl_decoder_kl_per_position(const srl_policy* const* checkpoints, int32_t n_checkpoints,
                                           const int32_t* switch_points, int32_t n_switch,
                                           int32_t recompute_state, const srl_policy* target,
                                           const int32_t* tokens, const int64_t* offsets, int32_t n_prefix,
                                           double* kl_out, int32_t cap) {
  return guarded([&] {
    if (!checkpoints || n_checkpoints < 1 || !target || n_prefix < 0 || (n_prefix > 0 && (!tokens || !offsets)) ||
        !kl_out || (n_switch > 0 && !switch_points))
      return fail(SRL_INVALID_ARGUMENT, "kl: bad arguments");
    if (target->p.type != SRL_POLICY_DECODER) return fail(SRL_INVALID_ARGUMENT, "kl: needs decoder policies");
    std::vector<const DecoderWeights*> ck;
    for (int i = 0; i < n_checkpoints; ++i) {
      if (!checkpoints[i] || checkpoints[i]->p.type != SRL_POLICY_DECODER)
        return fail(SRL_INVALID_ARGUMENT, "kl: needs decoder policies");
      ck.push_back(checkpoints[i]->p.dec.get());
    }
    int st;
    if ((st = require_device(target->p.dec->device))) return st;
    std::vector<std::vector<int32_t>> pre;
    size_t longest = 0;
    for (int q = 0; q < n_prefix; ++q) {
      pre.emplace_back(tokens + offsets[q], tokens + offsets[q + 1]);
      longest = std::max(longest, pre.back().size());
    }
    if ((int64_t)longest > cap) return fail(SRL_INVALID_ARGUMENT, "kl: output capacity below the longest prefix");
    std::vector<double> out;
    if ((st = decoder_kl_per_position(ck, std::vector<int>(switch_points, switch_points + std::max(0, n_switch)),
                                      recompute_state != 0, *target->p.dec, pre, out)))
      return st;
    std::copy(out.begin(), out.end(), kl_out);
    return (int)SRL_OK;
  });
}

// ess (rl_math.cpp:152-163)
extern "C" int srl_ess(const double* w, int32_t n, double* out) {
  if (!out || n < 1 || !w) return fail(SRL_INVALID_ARGUMENT, "ess: empty weight vector");
  double sum = 0.0, sq = 0.0;
  for (int i = 0; i < n; ++i) {
    if (!std::isfinite(w[i]) || w[i] < 0.0)
      return fail(SRL_INVALID_ARGUMENT, "ess: weights must be finite and nonnegative");
    sum += w[i];
    sq += w[i] * w[i];
  }
  if (sq == 0.0) return fail(SRL_ESS_UNDEFINED, "ess undefined: all weights are zero");
  *out = (sum * sum) / ((double)n * sq);
  return SRL_OK;
}

extern "C" int srl_lag_stats(const int32_t* versions, const int64_t* seq_offsets, int32_t n_seq,
                             int32_t version_before, int64_t* hist, int32_t hist_cap,
                             int64_t* seq_lag_sums, int64_t* totals, void* stream) {
  if (!seq_offsets || !hist || hist_cap < 1 || !totals || n_seq < 0 || (n_seq > 0 && (!versions || !seq_lag_sums)))
    return fail(SRL_INVALID_ARGUMENT, "lag_stats: bad arguments");
  launch_lag_stats(versions, seq_offsets, n_seq, version_before, hist, hist_cap, seq_lag_sums,
                   totals, static_cast<cudaStream_t>(stream));
  SRL_CUDA(cudaGetLastError());
  return SRL_OK;
}

// ------------------------------------------------------------ protocol ---
extern "C" uint32_t srl_crc32(const void* bytes, size_t n) {  // engine.cpp:257-274
  static uint32_t table[256];
  static bool init = [] {
    for (uint32_t i = 0; i < 256; ++i) {
      uint32_t c = i;
      for (int k = 0; k < 8; ++k) c = (c & 1) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
      table[i] = c;
    }
    return true;
  }();
  (void)init;
  const unsigned char* b = static_cast<const unsigned char*>(bytes);
  uint32_t c = 0xFFFFFFFFu;
  for (size_t i = 0; i < n; ++i) c = table[(c ^ b[i]) & 0xFFu] ^ (c >> 8);
  return c ^ 0xFFFFFFFFu;
}

extern "C" int srl_process_group_id(const char* const* members, int32_t n, char* buf, size_t cap) {
  // engine.cpp:276-291: FNV-1a over the sorted member list, '\n' separated
  if (n < 1 || !members) return fail(SRL_INVALID_ARGUMENT, "process group needs at least one member");
  if (!buf || cap < 20) return fail(SRL_INVALID_ARGUMENT, "buffer too small");
  std::vector<std::string> m;
  for (int i = 0; i < n; ++i) m.emplace_back(members[i] ? members[i] : "");
  std::sort(m.begin(), m.end());
  uint64_t h = 0xcbf29ce484222325ULL;
  for (const auto& s : m) {
    for (unsigned char c : s) {
      h ^= c;
      h *= 0x100000001b3ULL;
    }
    h ^= '\n';
    h *= 0x100000001b3ULL;
  }
  std::snprintf(buf, cap, "pg-%016llx", (unsigned long long)h);
  return SRL_OK;
}

extern "C" int srl_engine_profile_next_round(srl_engine* e) {
  if (!e) return fail(SRL_INVALID_ARGUMENT, "profile_next_round");
  e->e->profile_next_round();
  return SRL_OK;
}

extern "C" int srl_engine_kernel_profile(const srl_engine* e, srl_kernel_profile* out) {
  if (!e || !out) return fail(SRL_INVALID_ARGUMENT, "kernel_profile");
  if (!e->e->kernel_profile(out)) return fail(SRL_INVALID_ARGUMENT, "no profiled round yet");
  return SRL_OK;
}

// ------------------------------------------------------------- trainer ---
extern "C" int srl_trainer_create(const srl_policy* p, const srl_trainer_options* opts,
                                  srl_trainer** out) {
  return guarded([&] {
    if (!p || !out || p->p.type != SRL_POLICY_DECODER)
      return fail(SRL_INVALID_ARGUMENT, "trainer_create: needs a decoder policy");
    int st;
    if ((st = require_device(p->p.dec->device))) return st;
    srl_trainer_options o{};
    o.max_tokens = 4096;
    o.device = p->p.dec->device;
    if (opts) o = *opts;
    if (o.device < 0) o.device = p->p.dec->device;
    if ((st = require_device(o.device))) return st;
    auto h = std::make_unique<srl_trainer>();
    h->t = std::make_unique<DecoderTrainer>();
    if ((st = h->t->init(*p->p.dec, o))) return st;
    *out = h.release();
    return (int)SRL_OK;
  });
}

extern "C" void srl_trainer_destroy(srl_trainer* t) { delete t; }

extern "C" int srl_trainer_step(srl_trainer* t, const int32_t* tokens, const int64_t* offsets,
                                int32_t n_seq, const int32_t* loss_begin,
                                const double* behavior_logprobs, const double* advantages,
                                int32_t n_trajectories, double clamp, int32_t granularity,
                                double* logprobs_out, srl_trainer_stats* stats) {
  return guarded([&] {
    if (!t || !tokens || !offsets || n_seq < 1 || !loss_begin || !behavior_logprobs || !advantages)
      return fail(SRL_INVALID_ARGUMENT, "trainer_step: bad arguments");
    if (clamp <= 0.0 || !std::isfinite(clamp))  // truncated_is_weight (rl_math.cpp:146-147)
      return fail(SRL_INVALID_ARGUMENT, "truncated_is_weight: clamp must be positive");
    if (granularity != 0 && granularity != 1) return fail(SRL_INVALID_ARGUMENT, "granularity");
    TrainBatch b;
    b.n_trajectories = n_trajectories;
    b.clamp = clamp;
    b.granularity = granularity;
    const DecoderDims& d = t->t->weights().dims;
    for (int q = 0; q < n_seq; ++q) {
      const int64_t a = offsets[q], e = offsets[q + 1];
      const int n = (int)(e - a);
      if (n < 2 || loss_begin[q] < 1 || loss_begin[q] >= n)
        return fail(SRL_INVALID_ARGUMENT, "trainer_step: sequence needs a scored token");
      if (n > d.max_pos) return fail(SRL_INVALID_ARGUMENT, "sequence longer than max_positions");
      b.seq_start.push_back(b.rows);
      b.seq_len.push_back(n - 1);
      b.loss_begin.push_back(loss_begin[q] - 1);
      for (int p = 0; p + 1 < n; ++p) {
        const int32_t in = tokens[a + p], tg = tokens[a + p + 1];
        if (in < 0 || in >= d.V || tg < 0 || tg >= d.V)
          return fail(SRL_INVALID_ARGUMENT, "token out of vocab range");
        const double mu = behavior_logprobs[a + p + 1], adv = advantages[a + p + 1];
        const bool scored = p + 1 >= loss_begin[q];
        if (scored && (!std::isfinite(mu) || !std::isfinite(adv)))
          return fail(SRL_INVALID_ARGUMENT, "truncated_is_weight: non-finite log-probability");
        b.row_slot.push_back(q);
        b.row_pos.push_back(p);
        b.row_token.push_back(in);
        b.row_target.push_back(tg);
        b.row_mu.push_back(scored ? mu : 0.0);
        b.row_adv.push_back(scored ? adv : 0.0);
        if (scored) ++b.n_loss_rows;
        ++b.rows;
      }
    }
    srl_trainer_stats s{};
    const int st = t->t->step(b, &s);
    if (st != SRL_OK) return st;
    if (stats) *stats = s;
    if (logprobs_out) {
      const auto& lp = t->t->last_logprobs();
      for (int q = 0; q < n_seq; ++q) {
        logprobs_out[offsets[q]] = 0.0;
        for (int p = 0; p < b.seq_len[q]; ++p) logprobs_out[offsets[q] + p + 1] = lp[b.seq_start[q] + p];
      }
    }
    return (int)SRL_OK;
  });
}

extern "C" int srl_trainer_gradient(srl_trainer* t, void** device_ptr, size_t* n_elems) {
  if (!t || !device_ptr || !n_elems) return fail(SRL_INVALID_ARGUMENT, "trainer_gradient");
  *device_ptr = t->t->gradient();
  *n_elems = t->t->elements();
  return SRL_OK;
}

extern "C" int srl_trainer_apply_adam(srl_trainer* t, double lr, double b1, double b2, double eps) {
  if (!t) return fail(SRL_INVALID_ARGUMENT, "trainer_apply_adam");
  return t->t->apply_adam((float)lr, (float)b1, (float)b2, (float)eps);
}

extern "C" int srl_trainer_weights(srl_trainer* t, void** device_ptr, size_t* nbytes) {
  if (!t || !device_ptr || !nbytes) return fail(SRL_INVALID_ARGUMENT, "trainer_weights");
  *device_ptr = t->t->weights().w;
  *nbytes = t->t->weights().bytes;
  return SRL_OK;
}
