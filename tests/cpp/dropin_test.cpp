// dropin_test.cpp -- the reference's engine-level and rlmath tests, restated
// in-process against the drop-in headers (include/streamrl/*.hpp) and the
// device library (libsrl_b200.so).  The reference's own test_protocol.cpp
// drives the same Engine through its HTTP server; here the calls are direct,
// the assertions are the reference's (file:line on each case), and the
// expected values are what the unmodified reference produced
// (tests/golden/reference_vectors.json, tests/golden/make_golden.py).
//
//   g++ -std=c++20 -I include -I <nlohmann dir> tests/cpp/dropin_test.cpp
//       -L paper_2509_19128_b200 -lsrl_b200 -Wl,-rpath,... -o dropin_test
//   ./dropin_test tests/golden/reference_vectors.json
#include <cmath>
#include <cstdio>
#include <fstream>
#include <functional>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include <json.hpp>

#include "streamrl/engine.hpp"
#include "streamrl/rl_math.hpp"

using namespace streamrl;
using json = nlohmann::json;
using rlmath::Policy;

namespace {

int g_failed = 0, g_checks = 0;
#define CHECK(cond)                                                          \
  do {                                                                       \
    ++g_checks;                                                              \
    if (!(cond)) {                                                           \
      ++g_failed;                                                            \
      std::fprintf(stderr, "%s:%d: CHECK failed: %s\n", __FILE__, __LINE__, #cond); \
    }                                                                        \
  } while (0)
template <class E, class F>
void check_throws(F&& f, const char* what) {
  ++g_checks;
  try {
    f();
  } catch (const E&) {
    return;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "%s: wrong exception type: %s\n", what, e.what());
    ++g_failed;
    return;
  }
  std::fprintf(stderr, "%s: no exception\n", what);
  ++g_failed;
}
bool rel_close(double a, double b, double rel) { return std::abs(a - b) <= rel * std::max(1.0, std::abs(b)); }

// policy_from_json (policy.cpp:163-192) for the two reference types
Policy policy_of(const json& d) {
  if (d.at("type") == "tabular") {
    rlmath::TabularPolicy t;
    t.vocab_size = d.at("vocab_size");
    t.context_order = d.at("context_order");
    t.default_logits = d.value("default_logits", std::vector<double>{});
    for (const auto& r : d.at("rows"))
      t.logits[{r.at("prompt_id"), r.at("context").get<std::vector<std::int32_t>>()}] =
          r.at("logits").get<std::vector<double>>();
    return t;
  }
  rlmath::RecurrentToyPolicy r;
  r.vocab_size = d.at("vocab_size");
  r.hidden_dim = d.at("hidden_dim");
  r.input_embedding = d.at("input_embedding").get<std::vector<double>>();
  r.recurrence = d.at("recurrence").get<std::vector<double>>();
  r.output = d.at("output").get<std::vector<double>>();
  return r;
}

std::vector<proto::TokenEvent> drain(proto::Engine& e, const std::string& id, proto::FinishReason& why) {
  std::vector<proto::TokenEvent> out;
  while (e.wait_events(id, out, why)) {
  }
  return out;
}

// policy documents (policy.hpp:77-82; test_rl_math.cpp:463-474 round trip): the
// drop-in's policy_to_json / policy_from_json on the reference's documents
void test_policy_documents(const json& g) {
  for (const json* d : {&g.at("demo_scenario").at("v0"), &g.at("demo_scenario").at("v1"),
                        &g.at("cross_module").at("checkpoints")[0]}) {
    const Policy p = rlmath::policy_from_json(d->dump());
    const Policy back = rlmath::policy_from_json(rlmath::policy_to_json(p));
    CHECK(json::parse(rlmath::policy_to_json(back)) == json::parse(rlmath::policy_to_json(p)));
    // the wire bytes of the reference client: crc32 over the compact dump
    CHECK(proto::crc32(json::parse(rlmath::policy_to_json(p)).dump()) ==
          proto::crc32(json::parse(rlmath::policy_to_json(policy_of(*d))).dump()));
  }
  check_throws<std::invalid_argument>([] { rlmath::policy_from_json(R"({"schema":"x","type":"tabular"})"); },
                                      "unknown schema");
  check_throws<std::invalid_argument>(
      [] { rlmath::policy_from_json(R"({"schema":"streamrl.policy/1","type":"tabular","vocab_size":0,"context_order":0})"); },
      "invalid policy");
}

// test_protocol.cpp:76-79, 132-144 (engine.cpp:257-291)
void test_crc_and_groups(const json& g) {
  for (const auto& c : g.at("protocol").at("crc32")) CHECK(proto::crc32(c[0].get<std::string>()) == c[1].get<std::uint32_t>());
  CHECK(proto::crc32("123456789") == 0xCBF43926u);
  for (const auto& c : g.at("protocol").at("group_ids"))
    CHECK(proto::process_group_id(c[0].get<std::vector<std::string>>()) == c[1].get<std::string>());
}

// drive_scenario demo_two_streams (test_protocol.cpp:271-287) + version split
// at the pause boundary (test_protocol.cpp:187-208)
void test_demo_scenario(const json& g) {
  const json& d = g.at("demo_scenario");
  proto::Engine e({policy_of(d.at("v0")), false, true});
  const std::string a = e.open_stream("demo", 12, 5, -1), b = e.open_stream("demo", 12, 6, -1);
  CHECK(a == "s0" && b == "s1");
  CHECK(e.advance(5) == 10);
  const auto r = e.apply_weight_update(1, policy_of(d.at("v1")));
  CHECK(r.applied && r.version == 1 && r.error.empty());
  e.advance(7);
  const std::string ids[2] = {a, b};
  for (int s = 0; s < 2; ++s) {
    proto::FinishReason why;
    const auto evs = drain(e, ids[s], why);
    const json& ref = d.at("streams")[s].at("events");
    CHECK(why == proto::FinishReason::Length && evs.size() == ref.size());
    for (std::size_t i = 0; i < evs.size() && i < ref.size(); ++i) {
      CHECK(evs[i].position == ref[i][0].get<int>());
      CHECK(evs[i].token == ref[i][1].get<int>());
      CHECK(rel_close(evs[i].logprob, ref[i][2].get<double>(), 1e-12));
      CHECK(evs[i].weight_version == ref[i][3].get<int>());
      CHECK(evs[i].weight_version == (evs[i].position < 5 ? 0 : 1));
      CHECK(evs[i].stream_id == ids[s]);
    }
  }
}

// test_protocol.cpp:161-185: out-of-order updates rejected without side effects
void test_rejection_safety(const json& g) {
  const json& d = g.at("demo_scenario");
  proto::Engine tainted({policy_of(d.at("v0")), false, true});
  const auto skipped = tainted.apply_weight_update(2, policy_of(d.at("v1")));
  CHECK(!skipped.applied && skipped.error == "version_conflict" && tainted.weight_version() == 0);
  const auto repeated = tainted.apply_weight_update(0, policy_of(d.at("v1")));
  CHECK(!repeated.applied && tainted.weight_version() == 0);
  rlmath::RecurrentToyPolicy wrong;  // different type: policy_mismatch (engine.cpp:96-102)
  wrong.vocab_size = 6;
  wrong.hidden_dim = 2;
  wrong.input_embedding.assign(12, 0.1);
  wrong.recurrence.assign(4, 0.0);
  wrong.output.assign(12, 0.0);
  const auto mism = tainted.apply_weight_update(1, wrong);
  CHECK(!mism.applied && mism.error == "policy_mismatch");
  proto::Engine clean({policy_of(d.at("v0")), false, true});
  const std::string t = tainted.open_stream("demo", 12, 4, -1), c = clean.open_stream("demo", 12, 4, -1);
  tainted.advance(12);
  clean.advance(12);
  proto::FinishReason w1, w2;
  const auto x = drain(tainted, t, w1), y = drain(clean, c, w2);
  CHECK(x.size() == 12 && y.size() == 12);
  for (std::size_t i = 0; i < x.size() && i < y.size(); ++i) {
    CHECK(x[i].token == y[i].token);
    CHECK(x[i].logprob == y[i].logprob);
    CHECK(x[i].weight_version == 0);
  }
}

// test_protocol.cpp:210-229: a stream overlapping two updates carries 0, 1, 2 in order
void test_three_versions(const json& g) {
  const json& d = g.at("demo_scenario");
  proto::Engine e({policy_of(d.at("v0")), false, true});
  const std::string s = e.open_stream("demo", 12, 8, -1);
  e.advance(3);
  CHECK(e.apply_weight_update(1, policy_of(d.at("v1"))).applied);
  e.advance(4);
  CHECK(e.apply_weight_update(2, policy_of(d.at("v0"))).applied);
  e.advance(5);
  proto::FinishReason why;
  const auto evs = drain(e, s, why);
  std::vector<int> bounds;
  for (const auto& ev : evs)
    if (bounds.empty() || bounds.back() != ev.weight_version) bounds.push_back(ev.weight_version);
  CHECK(evs.size() == 12 && (bounds == std::vector<int>{0, 1, 2}));
}

// test_protocol.cpp:231-269 / acceptance.cpp:405-457: engine transcript ==
// mixed_policy_sample seed for seed, stale and recompute
void test_cross_module(const json& g) {
  const json& cm = g.at("cross_module");
  std::vector<Policy> ck;
  for (const auto& d : cm.at("checkpoints")) ck.push_back(policy_of(d));
  const auto seeds = cm.at("seeds").get<std::vector<std::uint64_t>>();
  for (bool recompute : {false, true}) {
    proto::Engine e({ck[0], recompute, true});
    CHECK(e.recompute_state_mode() == recompute);
    std::vector<std::string> ids;
    for (auto s : seeds) ids.push_back(e.open_stream("p", 16, s, -1));
    e.advance(8);
    CHECK(e.apply_weight_update(1, ck[1]).applied);
    e.advance(4);
    CHECK(e.apply_weight_update(2, ck[2]).applied);
    e.advance(4);
    const json& exp = cm.at(recompute ? "recompute" : "stale");
    for (std::size_t i = 0; i < ids.size(); ++i) {
      proto::FinishReason why;
      const auto evs = drain(e, ids[i], why);
      const auto tok = exp[i].at("tokens").get<std::vector<int>>();
      const auto ver = exp[i].at("behavior_versions").get<std::vector<int>>();
      const auto lp = exp[i].at("behavior_logprobs").get<std::vector<double>>();
      CHECK(evs.size() == tok.size());
      for (std::size_t t = 0; t < evs.size() && t < tok.size(); ++t) {
        CHECK(evs[t].token == tok[t]);
        CHECK(evs[t].weight_version == ver[t]);
        // device exp / log / tanh differ from glibc by <= 1 ulp, compounding
        // through the recurrent state: 1e-9 relative
        CHECK(rel_close(evs[t].logprob, lp[t], 1e-9));
      }
    }
  }
}

// engine.cpp:46-48, 63-67, 174-178: the reference's exceptions
void test_engine_errors(const json& g) {
  const json& d = g.at("demo_scenario");
  proto::Engine e({policy_of(d.at("v0")), false, false});
  check_throws<std::invalid_argument>([&] { e.open_stream("demo", 0, 1, -1); }, "max_tokens < 1");
  check_throws<std::invalid_argument>([&] {
    std::vector<proto::TokenEvent> out;
    proto::FinishReason r;
    e.wait_events("s99", out, r);
  }, "unknown stream");
  check_throws<std::logic_error>([&] { e.advance(1); }, "advance on a running engine");
  CHECK(!e.process_group_id().has_value());
  e.set_process_group("pg-1", {"http://a:1"});
  CHECK(e.process_group_id().value() == "pg-1");
  e.pause();
  CHECK(e.advance(0) == 0);
  rlmath::TabularPolicy bad;
  bad.vocab_size = 0;
  check_throws<std::invalid_argument>([&] { proto::Engine x({bad, false, false}); }, "invalid policy");
}

// test_rl_math.cpp:106-183 via the golden cases (rl_math.cpp:128-163)
void test_rlmath(const json& g) {
  for (const auto& c : g.at("logprobs").at("cases")) {
    const auto toks = c.at("tokens").get<std::vector<std::int32_t>>();
    const auto got = rlmath::policy_logprobs(policy_of(c.at("policy")), c.at("prompt"), toks);
    const auto exp = c.at("out").get<std::vector<double>>();
    CHECK(got.size() == exp.size());
    for (std::size_t i = 0; i < got.size() && i < exp.size(); ++i) CHECK(rel_close(got[i], exp[i], 1e-9));
  }
  for (const auto& c : g.at("is_ess").at("truncated"))
    CHECK(rlmath::truncated_is_weight(c[0], c[1], c[2]) == c[3].get<double>());
  for (const auto& c : g.at("is_ess").at("ess"))
    CHECK(rel_close(rlmath::ess(c[0].get<std::vector<double>>()), c[1].get<double>(), 1e-15));
  check_throws<rlmath::EssUndefinedError>([] { rlmath::ess(std::vector<double>{0.0, 0.0}); }, "ess zeros");
  check_throws<std::invalid_argument>([] { rlmath::truncated_is_weight(0.0, 0.0, 0.0); }, "clamp 0");
  // fit_baseline (test_rl_math.cpp:200-215)
  rlmath::Trajectory a{"p", {0, 1, 0}, {-1, -1, -1}, {0, 0, 0}, 0.0};
  rlmath::Trajectory b{"p", {1, 1, 1}, {-1, -1, -1}, {0, 0, 0}, 1.0};
  const auto table = rlmath::fit_baseline(std::vector<rlmath::Trajectory>{a, b});
  for (std::size_t t = 0; t < 3; ++t) CHECK(table.at("p", t) == 0.5);
  check_throws<std::invalid_argument>([] { rlmath::fit_baseline(std::vector<rlmath::Trajectory>{}); }, "no trajs");
}

// The 16 reference gradient cases (rl_math.cpp:211-276) on the device
void test_gradients(const json& g) {
  for (const auto& c : g.at("gradients").at("cases")) {
    const auto pol = std::get<rlmath::TabularPolicy>(policy_of(c.at("policy")));
    std::vector<rlmath::Trajectory> trajs;
    for (const auto& t : c.at("trajectories"))
      trajs.push_back({t.at("prompt_id"), t.at("tokens").get<std::vector<std::int32_t>>(),
                       t.at("behavior_logprobs").get<std::vector<double>>(),
                       t.at("behavior_versions").get<std::vector<std::int32_t>>(), t.at("reward")});
    const auto base = rlmath::fit_baseline(trajs);
    const auto gran = c.at("granularity") == 1 ? rlmath::IsWeightGranularity::PerToken
                                               : rlmath::IsWeightGranularity::Sequence;
    const auto got = c.at("use_is") != 0 ? rlmath::is_reinforce_gradient(pol, trajs, base, c.at("clamp"), gran)
                                         : rlmath::reinforce_gradient(pol, trajs, base);
    rlmath::GradientTable exp;
    for (const auto& r : c.at("grad").at("rows"))
      exp.rows[{r.at("prompt_id"), r.at("context").get<std::vector<std::int32_t>>()}] =
          r.at("grad").get<std::vector<double>>();
    exp.default_row = c.at("grad").at("default_row").get<std::vector<double>>();
    CHECK(got.rows.size() == exp.rows.size());
    CHECK(got.max_abs_diff(exp) <= 1e-12 * std::max(1.0, exp.max_abs()));
  }
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: %s reference_vectors.json\n", argv[0]);
    return 2;
  }
  std::ifstream f(argv[1]);
  const json g = json::parse(f);
  const std::vector<std::pair<const char*, std::function<void(const json&)>>> cases = {
      {"crc_and_groups", test_crc_and_groups}, {"policy_documents", test_policy_documents},
      {"demo_scenario", test_demo_scenario},
      {"rejection_safety", test_rejection_safety}, {"three_versions", test_three_versions},
      {"cross_module", test_cross_module}, {"engine_errors", test_engine_errors},
      {"rlmath", test_rlmath}, {"gradients", test_gradients}};
  for (const auto& [name, fn] : cases) {
    const int before = g_failed;
    try {
      fn(g);
    } catch (const std::exception& e) {
      std::fprintf(stderr, "%s: unexpected exception: %s\n", name, e.what());
      ++g_failed;
    }
    std::printf("[%s] %s\n", g_failed == before ? "ok" : "FAIL", name);
  }
  std::printf("%d checks, %d failed\n", g_checks, g_failed);
  return g_failed == 0 ? 0 : 1;
}
