// ref_shim.cpp -- extern "C" driver over the UNMODIFIED reference streamrl
// sources, compiled by oracle/Makefile into oracle/_ref/libstreamrl_ref.so.
//
// TEST INFRASTRUCTURE ONLY: used to generate/check golden vectors
// (tests/golden/make_golden.py) and as bench.py's reference CPU arm for the
// toy-policy engine.  Nothing in paper_2509_19128_b200/ links or loads it.
//
// All structured data crosses the boundary as JSON text (the reference's own
// policy / trajectory document formats); strings returned by ref_* are
// malloc'd and released with ref_free.
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include <json.hpp>

#include "streamrl/engine.hpp"
#include "streamrl/rl_math.hpp"
#include "streamrl/sim.hpp"
#include "streamrl/throughput.hpp"
#include "streamrl/trajectory.hpp"

using nlohmann::json;
using namespace streamrl;

namespace {

char* dup(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.data(), s.size() + 1);
  return p;
}

char* error_json(const std::exception& e) {
  return dup(json{{"error", e.what()}}.dump());
}

std::vector<rlmath::Policy> policies_from(const json& arr) {
  std::vector<rlmath::Policy> out;
  for (const auto& d : arr) out.push_back(rlmath::policy_from_json(d.dump()));
  return out;
}

json gradient_to_json(const rlmath::GradientTable& g) {
  json rows = json::array();
  for (const auto& [key, row] : g.rows)
    rows.push_back({{"prompt_id", key.prompt_id}, {"context", key.context}, {"grad", row}});
  return {{"rows", rows}, {"default_row", g.default_row}};
}

}  // namespace

extern "C" {

void ref_free(char* p) { std::free(p); }

char* ref_random_recurrent_policy(int vocab, int hidden, double scale, unsigned long long seed) {
  try {
    return dup(rlmath::policy_to_json(rlmath::random_recurrent_policy(vocab, hidden, scale, seed)));
  } catch (const std::exception& e) { return error_json(e); }
}

// keys_json: [["prompt", [ctx...]], ...]
char* ref_random_tabular_policy(int vocab, int order, const char* keys_json, double scale,
                                unsigned long long seed) {
  try {
    std::vector<rlmath::ContextKey> keys;
    for (const auto& k : json::parse(keys_json))
      keys.push_back({k.at(0).get<std::string>(), k.at(1).get<std::vector<std::int32_t>>()});
    return dup(rlmath::policy_to_json(rlmath::random_tabular_policy(vocab, order, keys, scale, seed)));
  } catch (const std::exception& e) { return error_json(e); }
}

char* ref_drift_checkpoints(const char* policy_json, int count, double magnitude,
                            unsigned long long seed) {
  try {
    const auto ck = rlmath::drift_checkpoints(rlmath::policy_from_json(policy_json), count,
                                              magnitude, seed);
    json arr = json::array();
    for (const auto& p : ck) arr.push_back(json::parse(rlmath::policy_to_json(p)));
    return dup(arr.dump());
  } catch (const std::exception& e) { return error_json(e); }
}

// schedule_max_len <= 0: single-policy sample_trajectories.
char* ref_mixed_policy_sample(const char* ckpts_json, int schedule_max_len, int max_lag,
                              int recompute, const char* prompt_id, int count, int max_len,
                              unsigned long long seed, int terminator) {
  try {
    const auto ck = policies_from(json::parse(ckpts_json));
    std::vector<rlmath::Trajectory> trajs;
    json sched = nullptr;
    if (schedule_max_len <= 0) {
      trajs = rlmath::sample_trajectories(ck.at(0), prompt_id, count, max_len, seed, terminator);
    } else {
      const auto s = rlmath::MixedPolicySchedule::make(schedule_max_len, max_lag);
      sched = s.switch_points;
      trajs = rlmath::mixed_policy_sample(ck, s, recompute != 0, prompt_id, count, max_len, seed,
                                          terminator);
    }
    return dup(json{{"switch_points", sched}, {"jsonl", rlmath::trajectories_to_jsonl(trajs)}}.dump());
  } catch (const std::exception& e) { return error_json(e); }
}

int ref_policy_logprobs(const char* policy_json, const char* prompt_id, const int* tokens, int n,
                        double* out) {
  try {
    const auto lp = rlmath::policy_logprobs(rlmath::policy_from_json(policy_json), prompt_id,
                                            std::span<const std::int32_t>(tokens, n));
    for (int i = 0; i < n; ++i) out[i] = lp[i];
    return 0;
  } catch (const std::exception&) { return 1; }
}

int ref_truncated_is_weight(double pi, double mu, double c, double* out) {
  try { *out = rlmath::truncated_is_weight(pi, mu, c); return 0; }
  catch (const std::exception&) { return 1; }
}

int ref_ess(const double* w, int n, double* out) {
  try { *out = rlmath::ess(std::span<const double>(w, n)); return 0; }
  catch (const rlmath::EssUndefinedError&) { return 2; }
  catch (const std::exception&) { return 1; }
}

char* ref_fit_baseline(const char* jsonl) {
  try {
    const auto trajs = rlmath::trajectories_from_jsonl(jsonl);
    const auto table = rlmath::fit_baseline(trajs);
    json cells = json::array();
    for (const auto& [key, v] : table.values) cells.push_back({key.first, key.second, v});
    return dup(cells.dump());
  } catch (const std::exception& e) { return error_json(e); }
}

// baseline_json: [[prompt, t, v], ...] or empty string => fit_baseline(trajs).
char* ref_is_reinforce_gradient(const char* policy_json, const char* jsonl,
                                const char* baseline_json, double clamp, int use_is,
                                int granularity) {
  try {
    const auto pol = rlmath::policy_from_json(policy_json);
    const auto& tab = std::get<rlmath::TabularPolicy>(pol);
    const auto trajs = rlmath::trajectories_from_jsonl(jsonl);
    rlmath::BaselineTable base;
    if (baseline_json == nullptr || baseline_json[0] == '\0') {
      base = rlmath::fit_baseline(trajs);
    } else {
      for (const auto& c : json::parse(baseline_json))
        base.values[{c.at(0).get<std::string>(), c.at(1).get<std::size_t>()}] = c.at(2).get<double>();
    }
    rlmath::GradientTable g =
        use_is ? rlmath::is_reinforce_gradient(
                     tab, trajs, base, clamp,
                     granularity ? rlmath::IsWeightGranularity::PerToken
                                 : rlmath::IsWeightGranularity::Sequence)
               : rlmath::reinforce_gradient(tab, trajs, base);
    return dup(gradient_to_json(g).dump());
  } catch (const std::exception& e) { return error_json(e); }
}

// Drives proto::Engine in-process in lockstep (no HTTP; the survey's
// re-driving of acceptance criteria 9/10).  script:
// {"policy": doc, "recompute": bool,
//  "steps": [{"open": {"prompt_id","max_tokens","seed","terminator"}},
//            {"advance": n}, {"update": {"version": v, "policy": doc}}]}
char* ref_engine_lockstep(const char* script_json) {
  try {
    const json script = json::parse(script_json);
    proto::Engine engine({rlmath::policy_from_json(script.at("policy").dump()),
                          script.value("recompute", false), true});
    std::vector<std::string> ids;
    json updates = json::array();
    json emitted = json::array();
    for (const auto& step : script.at("steps")) {
      if (step.contains("open")) {
        const auto& o = step.at("open");
        ids.push_back(engine.open_stream(o.at("prompt_id").get<std::string>(),
                                         o.at("max_tokens").get<int>(),
                                         o.at("seed").get<std::uint64_t>(),
                                         o.value("terminator", -1)));
      } else if (step.contains("advance")) {
        emitted.push_back(engine.advance(step.at("advance").get<int>()));
      } else if (step.contains("update")) {
        const auto& u = step.at("update");
        const auto r = engine.apply_weight_update(
            u.at("version").get<int>(), rlmath::policy_from_json(u.at("policy").dump()));
        updates.push_back({{"applied", r.applied}, {"version", r.version}, {"error", r.error}});
      }
    }
    // Record which streams were still running, then stop (running streams
    // finish with Shutdown) and drain every buffered event.
    std::vector<int> running_before_stop;
    const long long rounds = engine.rounds_done();
    const int active = engine.active_streams();
    engine.stop();
    json streams = json::array();
    for (const auto& id : ids) {
      std::vector<proto::TokenEvent> evs;
      proto::FinishReason reason = proto::FinishReason::Running;
      for (;;) {
        std::vector<proto::TokenEvent> chunk;
        const bool more = engine.wait_events(id, chunk, reason);
        evs.insert(evs.end(), chunk.begin(), chunk.end());
        if (!more || chunk.empty()) break;
      }
      json ev = json::array();
      for (const auto& e : evs) ev.push_back({e.position, e.token, e.logprob, e.weight_version});
      streams.push_back({{"id", id}, {"events", ev}, {"finish", proto::to_string(reason)}});
    }
    return dup(json{{"streams", streams}, {"updates", updates}, {"emitted", emitted},
                    {"rounds", rounds}, {"active_before_stop", active},
                    {"version", engine.weight_version()}}.dump());
  } catch (const std::exception& e) { return error_json(e); }
}

// Free-running engine throughput probe for bench.py's reference CPU arm:
// one Engine (one scheduler thread) with n_streams streams of max_tokens
// each; returns tokens emitted and wall seconds.
int ref_engine_throughput(const char* policy_json, int n_streams, int max_tokens,
                          unsigned long long seed, long long* tokens, double* seconds) {
  try {
    proto::Engine engine({rlmath::policy_from_json(policy_json), false, true});
    std::vector<std::string> ids;
    for (int i = 0; i < n_streams; ++i)
      ids.push_back(engine.open_stream("p", max_tokens, rng::derive_stream(seed, i), -1));
    const auto t0 = std::chrono::steady_clock::now();
    *tokens = engine.advance(max_tokens);
    const auto t1 = std::chrono::steady_clock::now();
    *seconds = std::chrono::duration<double>(t1 - t0).count();
    engine.stop();
    return 0;
  } catch (const std::exception&) { return 1; }
}

// The same probe on every host core at once: n_threads independent Engines
// (one scheduler thread each, SURVEY 8d "one instance per core"), each with
// n_streams streams; returns the aggregate tokens and the wall seconds of
// the slowest instance.
int ref_engine_throughput_parallel(const char* policy_json, int n_threads, int n_streams,
                                   int max_tokens, unsigned long long seed, long long* tokens,
                                   double* seconds) {
  try {
    const auto pol = rlmath::policy_from_json(policy_json);
    std::vector<long long> tok(n_threads, 0);
    std::vector<double> sec(n_threads, 0.0);
    std::vector<std::thread> th;
    for (int t = 0; t < n_threads; ++t)
      th.emplace_back([&, t] {
        proto::Engine engine({pol, false, true});
        for (int i = 0; i < n_streams; ++i)
          engine.open_stream("p", max_tokens, rng::derive_stream(seed + t, i), -1);
        const auto t0 = std::chrono::steady_clock::now();
        tok[t] = engine.advance(max_tokens);
        sec[t] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        engine.stop();
      });
    for (auto& x : th) x.join();
    *tokens = 0;
    *seconds = 0.0;
    for (int t = 0; t < n_threads; ++t) {
      *tokens += tok[t];
      *seconds = std::max(*seconds, sec[t]);
    }
    return 0;
  } catch (const std::exception&) { return 1; }
}

// The reference's in-flight update pause for one payload (protocol.cpp:147-190
// handler path + engine.cpp:79-117): the trainer serialises the policy
// (policy_to_json), the client checksums the body (crc32), the server parses
// it (policy_from_json) and applies it under the round lock with n_streams
// live streams after `rounds` rounds (stale or recompute state).
// out_ms = {serialize, crc32, parse, apply}; *payload_bytes = JSON body size.
int ref_update_pause(const char* policy_json, const char* new_policy_json, int n_streams,
                     int rounds, int recompute, double* out_ms, long long* payload_bytes) {
  try {
    using clk = std::chrono::steady_clock;
    auto ms = [](clk::time_point a, clk::time_point b) {
      return std::chrono::duration<double, std::milli>(b - a).count();
    };
    proto::Engine engine({rlmath::policy_from_json(policy_json), recompute != 0, true});
    for (int i = 0; i < n_streams; ++i)
      engine.open_stream("p", rounds + 16, rng::derive_stream(7, i), -1);
    engine.advance(rounds);
    const auto next = rlmath::policy_from_json(new_policy_json);
    const auto t0 = clk::now();
    const std::string body = rlmath::policy_to_json(next);
    const auto t1 = clk::now();
    volatile std::uint32_t crc = proto::crc32(body);
    (void)crc;
    const auto t2 = clk::now();
    auto parsed = rlmath::policy_from_json(body);
    const auto t3 = clk::now();
    const auto r = engine.apply_weight_update(1, std::move(parsed));
    const auto t4 = clk::now();
    engine.stop();
    if (!r.applied) return 2;
    out_ms[0] = ms(t0, t1);
    out_ms[1] = ms(t1, t2);
    out_ms[2] = ms(t2, t3);
    out_ms[3] = ms(t3, t4);
    *payload_bytes = (long long)body.size();
    return 0;
  } catch (const std::exception&) { return 1; }
}

char* ref_run_pipeline(const char* sim_config_json) {
  try {
    const auto cfg = sim::SimConfig::from_json(sim_config_json);
    return dup(sim::run_pipeline(cfg).to_json());
  } catch (const std::exception& e) { return error_json(e); }
}

char* ref_run_conventional(const char* sim_config_json) {
  try {
    const auto cfg = sim::SimConfig::from_json(sim_config_json);
    return dup(sim::run_conventional(cfg).to_json());
  } catch (const std::exception& e) { return error_json(e); }
}

long long ref_pipeline_max_lag_steps(long long gen_batch, long long inference_count, double max_len,
                                     double mean_len, long long train_batch) {
  try {
    return throughput::pipeline_max_lag_steps(gen_batch, inference_count, max_len, mean_len,
                                              train_batch);
  } catch (const std::exception&) { return -1; }
}

unsigned int ref_crc32(const char* bytes, size_t n) {
  return proto::crc32(std::string_view(bytes, n));
}

char* ref_process_group_id(const char* members_json) {
  try {
    return dup(proto::process_group_id(json::parse(members_json).get<std::vector<std::string>>()));
  } catch (const std::exception& e) { return error_json(e); }
}

// kl_per_position with a mixed behaviour (schedule_max_len > 0) or single.
char* ref_kl_per_position(const char* behavior_ckpts_json, int schedule_max_len, int max_lag,
                          int recompute, const char* target_json, const char* prompt_id,
                          const char* prefixes_jsonl) {
  try {
    auto ck = policies_from(json::parse(behavior_ckpts_json));
    rlmath::BehaviorSpec spec =
        schedule_max_len > 0
            ? rlmath::BehaviorSpec::mixed(ck, rlmath::MixedPolicySchedule::make(schedule_max_len, max_lag),
                                          recompute != 0)
            : rlmath::BehaviorSpec::single(ck.at(0));
    const auto kl = rlmath::kl_per_position(spec, rlmath::policy_from_json(target_json), prompt_id,
                                            rlmath::trajectories_from_jsonl(prefixes_jsonl));
    return dup(json(kl).dump());
  } catch (const std::exception& e) { return error_json(e); }
}

// The bytes EngineClient::request_weight_update checksums (protocol.cpp:340-356):
// json::parse(policy_to_json(policy)).dump() of the policy the document
// describes, and their crc32.
char* ref_policy_wire(const char* policy_json) {
  try {
    const auto pol = rlmath::policy_from_json(policy_json);
    const std::string bytes = json::parse(rlmath::policy_to_json(pol)).dump();
    return dup(json{{"bytes", bytes}, {"crc32", proto::crc32(bytes)}}.dump());
  } catch (const std::exception& e) { return error_json(e); }
}

// search_configs (throughput.cpp:288-330) on a JSON spec:
// {n, train_batch, curve: [[h, u], ...], padding_window, tau,
//  lengths: {kind: "uniform" | "constant" | "empirical", max_len, values}, cap, use_padding}
char* ref_search_configs(const char* spec_json) {
  try {
    const json s = json::parse(spec_json);
    throughput::UtilizationCurve curve;
    for (const auto& pt : s.at("curve")) curve.samples.push_back({pt[0].get<double>(), pt[1].get<double>()});
    curve.padding_window = s.value("padding_window", 64);
    const json& l = s.at("lengths");
    const std::string kind = l.at("kind");
    const auto lengths = kind == "uniform"    ? throughput::LengthDistribution::uniform(l.at("max_len"))
                         : kind == "constant" ? throughput::LengthDistribution::constant(l.at("max_len"))
                                              : throughput::LengthDistribution::empirical(
                                                    l.at("values").get<std::vector<int>>());
    const auto r = throughput::search_configs(s.at("n"), s.at("train_batch"), curve, s.at("tau"), lengths,
                                              s.at("cap"), s.value("use_padding", false));
    return dup(json{{"feasible", r.feasible}, {"gen_batch", r.gen_batch}, {"inference_count", r.inference_count},
                    {"r_gen", r.report.r_gen}, {"r_train", r.report.r_train}, {"r_total", r.report.r_total},
                    {"max_lag", r.report.max_lag}}
                   .dump());
  } catch (const std::exception& e) { return error_json(e); }
}

}  // extern "C"
