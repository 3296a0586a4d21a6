// streamrl/policy.hpp -- drop-in for the reference's policy.hpp:16-82: the
// same TabularPolicy / RecurrentToyPolicy data types and Policy variant, so
// callers construct policies unchanged.  Evaluation happens on the device:
// b200::NativePolicy uploads a Policy through srl_policy_*_create and the
// engine / rlmath entry points take it from there.
#pragma once

#include <compare>
#include <cstdint>
#include <map>
#include <span>
#include <string>
#include <variant>
#include <vector>

#include "streamrl/b200_abi.hpp"

namespace streamrl::rlmath {

struct ContextKey {  // policy.hpp:16-21
  std::string prompt_id;
  std::vector<std::int32_t> context;
  auto operator<=>(const ContextKey&) const = default;
};

struct TabularPolicy {  // policy.hpp:23-47
  std::int32_t vocab_size = 0;
  std::int32_t context_order = 0;
  std::map<ContextKey, std::vector<double>> logits;
  std::vector<double> default_logits;
  void validate() const;
};

struct RecurrentToyPolicy {  // policy.hpp:52-72
  std::int32_t vocab_size = 0;
  std::int32_t hidden_dim = 0;
  std::vector<double> input_embedding;  // vocab_size x hidden_dim
  std::vector<double> recurrence;       // hidden_dim x hidden_dim
  std::vector<double> output;           // hidden_dim x vocab_size
  void validate() const;
  std::vector<double> initial_state() const { return std::vector<double>(hidden_dim, 0.0); }
};

using Policy = std::variant<TabularPolicy, RecurrentToyPolicy>;

inline std::int32_t vocab_size_of(const Policy& p) {
  return std::visit([](const auto& q) { return q.vocab_size; }, p);
}

}  // namespace streamrl::rlmath

namespace streamrl::b200 {

// RAII device-side copy (srl_policy) of a host policy.
class NativePolicy {
 public:
  explicit NativePolicy(const rlmath::Policy& p) {
    if (const auto* t = std::get_if<rlmath::TabularPolicy>(&p)) {
      std::vector<const char*> ids;
      std::vector<std::int32_t> lens, ctx;
      std::vector<double> lg;
      const int width = t->context_order > 0 ? t->context_order : 1;
      for (const auto& [key, row] : t->logits) {
        ids.push_back(key.prompt_id.c_str());
        lens.push_back(static_cast<std::int32_t>(key.context.size()));
        for (int j = 0; j < width; ++j)
          ctx.push_back(j < static_cast<int>(key.context.size()) ? key.context[j] : 0);
        if (static_cast<std::int32_t>(row.size()) != t->vocab_size)
          throw std::invalid_argument("TabularPolicy: logits row has the wrong length");
        lg.insert(lg.end(), row.begin(), row.end());
      }
      check(srl_policy_tabular_create(t->vocab_size, t->context_order,
                                      t->default_logits.empty() ? nullptr : t->default_logits.data(),
                                      static_cast<std::int32_t>(ids.size()), ids.data(), lens.data(),
                                      ctx.data(), lg.data(), &h_),
            "TabularPolicy");
    } else {
      const auto& r = std::get<rlmath::RecurrentToyPolicy>(p);
      check(srl_policy_recurrent_create(r.vocab_size, r.hidden_dim, r.input_embedding.data(),
                                        r.recurrence.data(), r.output.data(), &h_),
            "RecurrentToyPolicy");
    }
  }
  ~NativePolicy() { srl_policy_destroy(h_); }
  NativePolicy(const NativePolicy&) = delete;
  NativePolicy& operator=(const NativePolicy&) = delete;
  srl_policy* get() const { return h_; }

 private:
  srl_policy* h_ = nullptr;
};

}  // namespace streamrl::b200

namespace streamrl::rlmath {

// validate (policy.cpp:30-43, 71-82): std::invalid_argument on a bad shape.
inline void validate(const Policy& p) { b200::check(srl_policy_validate(b200::NativePolicy(p).get()), "validate"); }
inline void TabularPolicy::validate() const { rlmath::validate(Policy{*this}); }
inline void RecurrentToyPolicy::validate() const { rlmath::validate(Policy{*this}); }

}  // namespace streamrl::rlmath

#if __has_include(<json.hpp>)
#include "streamrl/policy_json.hpp"  // policy_to_json / policy_from_json (policy.hpp:77-82)
#endif
