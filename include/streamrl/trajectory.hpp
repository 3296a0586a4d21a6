// streamrl/trajectory.hpp -- drop-in for the reference's trajectory.hpp:15-35
// (the actor -> trainer record and the baseline table), host-side.
#pragma once

#include <cmath>
#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace streamrl::rlmath {

struct Trajectory {
  std::string prompt_id;
  std::vector<std::int32_t> tokens;
  std::vector<double> behavior_logprobs;
  std::vector<std::int32_t> behavior_versions;
  double reward = 0.0;

  void validate() const {  // trajectory.cpp:14-25
    const std::size_t n = tokens.size();
    if (n < 1) throw std::invalid_argument("Trajectory: empty token sequence");
    if (behavior_logprobs.size() != n || behavior_versions.size() != n)
      throw std::invalid_argument("Trajectory: field lengths differ");
    for (std::size_t i = 1; i < n; ++i)
      if (behavior_versions[i] < behavior_versions[i - 1])
        throw std::invalid_argument("Trajectory: behavior_versions decrease");
    for (double lp : behavior_logprobs)
      if (std::isnan(lp)) throw std::invalid_argument("Trajectory: NaN behavior logprob");
    if (!std::isfinite(reward)) throw std::invalid_argument("Trajectory: non-finite reward");
  }
  std::size_t length() const { return tokens.size(); }
  double behavior_logprob_sum() const {
    double s = 0.0;
    for (double v : behavior_logprobs) s += v;
    return s;
  }
};

struct BaselineTable {
  std::map<std::pair<std::string, std::size_t>, double> values;
  bool contains(const std::string& prompt_id, std::size_t position) const {
    return values.count({prompt_id, position}) > 0;
  }
  double at(const std::string& prompt_id, std::size_t position) const {  // trajectory.cpp:35-41
    const auto it = values.find({prompt_id, position});
    if (it == values.end())
      throw std::invalid_argument("BaselineTable: missing cell (" + prompt_id + ", " +
                                  std::to_string(position) + ")");
    return it->second;
  }
};

}  // namespace streamrl::rlmath
