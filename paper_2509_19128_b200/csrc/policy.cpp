// policy.cpp -- policy checkpoints: validation rules of the reference
// (src/policy.cpp:14-82) and the decoder policy's flat bf16 weight buffer.
#include <cmath>
#include <limits>

#include "runtime.hpp"

namespace srl {

DecoderWeights::~DecoderWeights() {
  if (w) {
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(device);
    cudaFree(w);
    cudaSetDevice(cur);
  }
  delete[] layout.layers;
}

int32_t Policy::vocab() const {
  switch (type) {
    case SRL_POLICY_TABULAR: return tab.vocab;
    case SRL_POLICY_RECURRENT: return rec.vocab;
    default: return dec ? dec->cfg.vocab_size : 0;
  }
}

namespace {
// check_logits_row (policy.cpp:14-25): -inf allowed, +inf / NaN malformed.
bool row_ok(const std::vector<double>& row, int32_t vocab, std::string* why, const char* what) {
  if ((int32_t)row.size() != vocab) {
    if (why) *why = std::string(what) + ": row size != vocab_size";
    return false;
  }
  for (double v : row)
    if (std::isnan(v) || v == std::numeric_limits<double>::infinity()) {
      if (why) *why = std::string(what) + ": non-finite logit";
      return false;
    }
  return true;
}
}  // namespace

int Policy::validate(std::string* why) const {
  auto bad = [&](const std::string& w) -> int {
    if (why) *why = w;
    return SRL_INVALID_POLICY;
  };
  if (type == SRL_POLICY_TABULAR) {  // TabularPolicy::validate (policy.cpp:30-43)
    if (tab.vocab < 1) return bad("TabularPolicy: vocab_size must be positive");
    if (tab.order < 0) return bad("TabularPolicy: negative context_order");
    if (!tab.default_logits.empty() && !row_ok(tab.default_logits, tab.vocab, why, "default_logits"))
      return SRL_INVALID_POLICY;
    for (const auto& r : tab.rows) {
      if ((int32_t)r.context.size() > tab.order)
        return bad("TabularPolicy: context longer than context_order");
      for (int32_t t : r.context)
        if (t < 0 || t >= tab.vocab) return bad("TabularPolicy: context token out of vocab");
      if (!row_ok(r.logits, tab.vocab, why, "logits")) return SRL_INVALID_POLICY;
    }
    return SRL_OK;
  }
  if (type == SRL_POLICY_RECURRENT) {  // RecurrentToyPolicy::validate (policy.cpp:71-82)
    if (rec.vocab < 1) return bad("RecurrentToyPolicy: vocab_size must be positive");
    if (rec.hidden < 1) return bad("RecurrentToyPolicy: hidden_dim must be positive");
    auto expect = [&](const std::vector<double>& m, size_t n, const char* what) -> int {
      if (m.size() != n) return bad(std::string(what) + ": wrong element count");
      for (double v : m)
        if (!std::isfinite(v)) return bad(std::string(what) + ": non-finite weight");
      return SRL_OK;
    };
    int st;
    if ((st = expect(rec.emb, (size_t)rec.vocab * rec.hidden, "input_embedding"))) return st;
    if ((st = expect(rec.rec, (size_t)rec.hidden * rec.hidden, "recurrence"))) return st;
    if ((st = expect(rec.out, (size_t)rec.hidden * rec.vocab, "output"))) return st;
    return SRL_OK;
  }
  if (type == SRL_POLICY_DECODER) {
    if (!dec || !dec->w) return bad("decoder policy without weights");
    const char* w = nullptr;
    if (!dims_valid(dec->dims, &w)) return bad(std::string("decoder: ") + w);
    return SRL_OK;
  }
  return bad("unknown policy type");
}

bool same_decoder_shape(const srl_decoder_config& a, const srl_decoder_config& b) {
  return a.vocab_size == b.vocab_size && a.hidden == b.hidden && a.layers == b.layers &&
         a.q_heads == b.q_heads && a.kv_heads == b.kv_heads && a.head_dim == b.head_dim &&
         a.intermediate == b.intermediate && a.tie_embeddings == b.tie_embeddings &&
         a.bos_token == b.bos_token && a.rope_theta == b.rope_theta && a.rms_eps == b.rms_eps;
}

int create_decoder(const srl_decoder_config& cfg, int device, std::shared_ptr<DecoderWeights>& out) {
  auto d = std::make_shared<DecoderWeights>();
  d->cfg = cfg;
  d->dims = dims_from(cfg);
  const char* why = nullptr;
  if (!dims_valid(d->dims, &why)) return fail(SRL_INVALID_POLICY, std::string("decoder: ") + why);
  d->device = device;
  const size_t n = make_layout(d->dims, d->layout);
  d->bytes = n * sizeof(__nv_bfloat16);
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
    return fail(SRL_NO_DEVICE, "no CUDA device");
  SRL_CUDA(cudaSetDevice(device));
  SRL_CUDA(cudaMalloc(&d->w, d->bytes));
  out = d;
  return SRL_OK;
}

int clone_decoder(const DecoderWeights& src, std::shared_ptr<DecoderWeights>& out, int device) {
  if (device < 0) device = src.device;
  const int st = create_decoder(src.cfg, device, out);
  if (st != SRL_OK) return st;
  if (device == src.device)
    SRL_CUDA(cudaMemcpy(out->w, src.w, src.bytes, cudaMemcpyDeviceToDevice));
  else
    SRL_CUDA(cudaMemcpyPeer(out->w, device, src.w, src.device, src.bytes));
  return SRL_OK;
}

}  // namespace srl
