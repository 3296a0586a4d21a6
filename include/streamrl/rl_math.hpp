// streamrl/rl_math.hpp -- drop-in for the reference's rl_math.hpp:20-77 (the
// trainer-side math of the hot path) with the same signatures, errors and
// semantics; the per-token work runs on the device through the C ABI:
//   policy_logprobs        -> srl_policy_logprobs               (rl_math.cpp:128-142)
//   truncated_is_weight    -> srl_truncated_is_weight           (rl_math.cpp:144-150)
//   ess                    -> srl_ess                           (rl_math.cpp:152-163)
//   fit_baseline           -> host (a std::map of means, rl_math.cpp:165-179)
//   reinforce_gradient / is_reinforce_gradient
//                          -> srl_tabular_is_reinforce_gradient (rl_math.cpp:211-276)
// The oracle-only helpers of the reference (sample_trajectories,
// mixed_policy_sample, kl_per_position, random_* policies) are not part of
// the hot path and are not re-exported.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <map>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "streamrl/policy.hpp"
#include "streamrl/trajectory.hpp"

namespace streamrl::rlmath {

inline constexpr std::int32_t kNoTerminator = -1;

inline std::vector<double> policy_logprobs(const Policy& policy, const std::string& prompt_id,
                                           std::span<const std::int32_t> tokens) {
  std::vector<double> out(tokens.size());
  b200::NativePolicy h(policy);
  b200::check(srl_policy_logprobs(h.get(), prompt_id.c_str(), tokens.data(),
                                  static_cast<std::int32_t>(tokens.size()), out.data()),
              "policy_logprobs");
  return out;
}

inline double truncated_is_weight(double pi_logprob_sum, double mu_logprob_sum, double clamp) {
  double w = 0.0;
  b200::check(srl_truncated_is_weight(pi_logprob_sum, mu_logprob_sum, clamp, &w), "truncated_is_weight");
  return w;
}

struct EssUndefinedError : std::invalid_argument {  // rl_math.hpp:30-32
  EssUndefinedError() : std::invalid_argument("ess undefined: all weights are zero") {}
};

inline double ess(std::span<const double> weights) {
  double out = 0.0;
  const int st = srl_ess(weights.data(), static_cast<std::int32_t>(weights.size()), &out);
  if (st == SRL_ESS_UNDEFINED) throw EssUndefinedError();
  b200::check(st, "ess");
  return out;
}

inline BaselineTable fit_baseline(std::span<const Trajectory> trajectories) {
  if (trajectories.empty()) throw std::invalid_argument("fit_baseline: no trajectories");
  std::map<std::pair<std::string, std::size_t>, std::pair<double, long long>> cells;
  for (const auto& traj : trajectories) {
    traj.validate();
    for (std::size_t t = 0; t < traj.length(); ++t) {
      auto& c = cells[{traj.prompt_id, t}];
      c.first += traj.reward;
      c.second += 1;
    }
  }
  BaselineTable table;
  for (const auto& [key, c] : cells) table.values[key] = c.first / c.second;
  return table;
}

struct GradientTable {  // rl_math.hpp:39-46
  std::map<ContextKey, std::vector<double>> rows;
  std::vector<double> default_row;

  double max_abs() const {
    double m = 0.0;
    for (const auto& [k, r] : rows)
      for (double v : r) m = std::max(m, std::abs(v));
    for (double v : default_row) m = std::max(m, std::abs(v));
    return m;
  }
  double max_abs_diff(const GradientTable& o) const {
    double m = 0.0;
    auto diff = [&m](const std::vector<double>& a, const std::vector<double>& b) {
      for (std::size_t i = 0; i < std::max(a.size(), b.size()); ++i)
        m = std::max(m, std::abs((i < a.size() ? a[i] : 0.0) - (i < b.size() ? b[i] : 0.0)));
    };
    static const std::vector<double> none;
    for (const auto& [k, r] : rows) {
      const auto it = o.rows.find(k);
      diff(r, it == o.rows.end() ? none : it->second);
    }
    for (const auto& [k, r] : o.rows)
      if (!rows.count(k)) diff(none, r);
    diff(default_row, o.default_row);
    return m;
  }
};

enum class IsWeightGranularity { Sequence, PerToken };

namespace detail {
inline GradientTable tabular_gradient(const TabularPolicy& policy, std::span<const Trajectory> trajs,
                                      const BaselineTable& baseline, double clamp, bool use_is,
                                      IsWeightGranularity g) {
  if (trajs.empty()) throw std::invalid_argument("reinforce_gradient: no trajectories");
  std::vector<const char*> ids;
  std::vector<std::int32_t> tokens;
  std::vector<std::int64_t> offsets{0};
  std::vector<double> mu, rewards, base;
  for (const auto& t : trajs) {
    t.validate();
    ids.push_back(t.prompt_id.c_str());
    tokens.insert(tokens.end(), t.tokens.begin(), t.tokens.end());
    mu.insert(mu.end(), t.behavior_logprobs.begin(), t.behavior_logprobs.end());
    for (std::size_t p = 0; p < t.length(); ++p) base.push_back(baseline.at(t.prompt_id, p));
    offsets.push_back(static_cast<std::int64_t>(tokens.size()));
    rewards.push_back(t.reward);
  }
  const std::size_t V = static_cast<std::size_t>(policy.vocab_size), R = policy.logits.size();
  std::vector<double> grad((R + 1) * V);
  std::vector<std::int32_t> touched(R + 1);
  b200::NativePolicy h{Policy{policy}};
  b200::check(srl_tabular_is_reinforce_gradient(
                  h.get(), static_cast<std::int32_t>(trajs.size()), ids.data(), tokens.data(),
                  offsets.data(), mu.data(), rewards.data(), base.data(), use_is ? 1 : 0, clamp,
                  g == IsWeightGranularity::PerToken ? 1 : 0, grad.data(), touched.data()),
              use_is ? "is_reinforce_gradient" : "reinforce_gradient");
  GradientTable out;  // device rows are in std::map<ContextKey> order, like policy.logits
  std::size_t r = 0;
  for (const auto& [key, row] : policy.logits) {
    if (touched[r]) out.rows[key].assign(grad.begin() + r * V, grad.begin() + (r + 1) * V);
    ++r;
  }
  if (touched[R]) out.default_row.assign(grad.begin() + R * V, grad.end());
  return out;
}
}  // namespace detail

inline GradientTable reinforce_gradient(const TabularPolicy& policy, std::span<const Trajectory> trajectories,
                                        const BaselineTable& baseline) {
  return detail::tabular_gradient(policy, trajectories, baseline, 1.0, false, IsWeightGranularity::Sequence);
}

inline GradientTable is_reinforce_gradient(const TabularPolicy& policy, std::span<const Trajectory> trajectories,
                                           const BaselineTable& baseline, double clamp,
                                           IsWeightGranularity granularity = IsWeightGranularity::Sequence) {
  return detail::tabular_gradient(policy, trajectories, baseline, clamp, true, granularity);
}

}  // namespace streamrl::rlmath
