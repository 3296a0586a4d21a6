// streamrl/policy_json.hpp -- the "streamrl.policy/1" document functions of the
// reference's policy.hpp:77-82 (policy_to_json, policy_from_json,
// policy_from_file, policy_to_file) for the drop-in policy types.  Uses
// nlohmann/json, the reference's own JSON library (<json.hpp> on the include
// path, as the reference itself requires); included by streamrl/policy.hpp
// when that header is available.
#pragma once

#include <fstream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <variant>

#include <json.hpp>

#include "streamrl/policy.hpp"

namespace streamrl::rlmath {

// The document of a policy: schema id, type, shape fields, row-major weights.
inline std::string policy_to_json(const Policy& policy) {
  using nlohmann::json;
  json doc;
  if (const auto* t = std::get_if<TabularPolicy>(&policy)) {
    json rows = json::array();
    for (const auto& [key, logits] : t->logits)
      rows.push_back({{"prompt_id", key.prompt_id}, {"context", key.context}, {"logits", logits}});
    doc = {{"schema", "streamrl.policy/1"}, {"type", "tabular"}, {"vocab_size", t->vocab_size},
           {"context_order", t->context_order}, {"default_logits", t->default_logits}, {"rows", rows}};
  } else {
    const auto& r = std::get<RecurrentToyPolicy>(policy);
    doc = {{"schema", "streamrl.policy/1"}, {"type", "recurrent"}, {"vocab_size", r.vocab_size},
           {"hidden_dim", r.hidden_dim}, {"input_embedding", r.input_embedding},
           {"recurrence", r.recurrence}, {"output", r.output}};
  }
  return doc.dump(2);
}

// Parses and validates a document (std::invalid_argument on an unknown schema
// or type, or an invalid policy).
inline Policy policy_from_json(const std::string& text) {
  using nlohmann::json;
  const json doc = json::parse(text);
  if (doc.value("schema", "") != "streamrl.policy/1")
    throw std::invalid_argument("policy document: unknown schema id");
  const std::string type = doc.at("type").get<std::string>();
  Policy out;
  if (type == "tabular") {
    TabularPolicy p;
    p.vocab_size = doc.at("vocab_size").get<std::int32_t>();
    p.context_order = doc.at("context_order").get<std::int32_t>();
    p.default_logits = doc.value("default_logits", std::vector<double>{});
    for (const auto& row : doc.value("rows", json::array()))
      p.logits[{row.at("prompt_id").get<std::string>(), row.at("context").get<std::vector<std::int32_t>>()}] =
          row.at("logits").get<std::vector<double>>();
    out = std::move(p);
  } else if (type == "recurrent") {
    RecurrentToyPolicy p;
    p.vocab_size = doc.at("vocab_size").get<std::int32_t>();
    p.hidden_dim = doc.at("hidden_dim").get<std::int32_t>();
    p.input_embedding = doc.at("input_embedding").get<std::vector<double>>();
    p.recurrence = doc.at("recurrence").get<std::vector<double>>();
    p.output = doc.at("output").get<std::vector<double>>();
    out = std::move(p);
  } else {
    throw std::invalid_argument("policy document: unknown type " + type);
  }
  validate(out);
  return out;
}

inline Policy policy_from_file(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open policy file: " + path);
  std::stringstream ss;
  ss << in.rdbuf();
  return policy_from_json(ss.str());
}

inline void policy_to_file(const Policy& policy, const std::string& path) {
  std::ofstream out(path);
  if (!out) throw std::runtime_error("cannot write policy file: " + path);
  out << policy_to_json(policy);
}

}  // namespace streamrl::rlmath
