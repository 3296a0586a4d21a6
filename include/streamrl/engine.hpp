// streamrl/engine.hpp -- drop-in for the reference's proto::Engine
// (engine.hpp:22-109) with the same class, signatures, exceptions and
// semantics; the engine is the device engine of libsrl_b200.so (one C++
// scheduler thread per engine, decode rounds on the GPU, token-boundary
// weight swaps under the round lock).  Callers of the reference -- its HTTP
// EngineServer, drive_scenario, tests -- compile against this header
// unchanged.
#pragma once

#include <cstdint>
#include <optional>
#include <string>
#include <string_view>
#include <vector>

#include "streamrl/policy.hpp"
#include "streamrl/rng.hpp"

namespace streamrl::proto {

struct TokenEvent {  // engine.hpp:22-28
  std::string stream_id;
  int position = 0;
  std::int32_t token = 0;
  double logprob = 0.0;
  int weight_version = 0;
};

enum class FinishReason { Running, Length, Terminator, Shutdown };  // engine.hpp:30

inline std::string to_string(FinishReason r) {
  switch (r) {
    case FinishReason::Running: return "running";
    case FinishReason::Length: return "length";
    case FinishReason::Terminator: return "terminator";
    case FinishReason::Shutdown: return "shutdown";
  }
  return "unknown";
}

struct UpdateResult {  // engine.hpp:34-38
  bool applied = false;
  int version = 0;
  std::string error;
};

class Engine {
 public:
  struct Options {
    rlmath::Policy policy;
    bool recompute_state = false;
    bool start_paused = false;
  };

  // engine.cpp:38-42: validates the policy (std::invalid_argument) and starts the scheduler.
  explicit Engine(Options options) : recompute_(options.recompute_state) {
    b200::NativePolicy p(options.policy);
    b200::check(srl_policy_validate(p.get()), "Engine");
    b200::check(srl_engine_create(p.get(), options.recompute_state ? 1 : 0, options.start_paused ? 1 : 0,
                                  nullptr, &e_),
                "Engine");
  }
  ~Engine() {
    if (e_) {
      srl_engine_stop(e_);
      srl_engine_destroy(e_);
    }
  }
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;

  // engine.cpp:46-61: "s<N>"; std::invalid_argument if max_tokens < 1.
  std::string open_stream(const std::string& prompt_id, int max_tokens, std::uint64_t seed,
                          std::int32_t terminator_token) {
    if (max_tokens < 1) throw std::invalid_argument("open_stream: max_tokens must be >= 1");
    std::int64_t id = 0;
    b200::check(srl_engine_open_stream(e_, prompt_id.c_str(), max_tokens, seed, terminator_token, nullptr, 0, &id),
                "open_stream");
    return "s" + std::to_string(id);
  }

  // engine.cpp:63-77: blocks until >= 1 event or the stream finishes, drains;
  // false once finished and drained; unknown id -> std::invalid_argument.
  bool wait_events(const std::string& stream_id, std::vector<TokenEvent>& out, FinishReason& reason) {
    const std::int64_t sid = parse_id(stream_id);
    constexpr std::int32_t kCap = 8192;
    std::vector<srl_token_event> buf(kCap);
    std::int32_t n = 0, fin = 0, more = 0;
    do {  // one native call drains at most kCap events; a full buffer means more are ready
      b200::check(srl_engine_wait_events(e_, sid, buf.data(), kCap, &n, &fin, &more), "wait_events");
      for (int i = 0; i < n; ++i)
        out.push_back({stream_id, buf[i].position, buf[i].token, buf[i].logprob, buf[i].weight_version});
    } while (n == kCap);
    reason = static_cast<FinishReason>(fin);
    return more != 0;
  }

  // engine.cpp:79-117: takes the policy by value; rejected -> state untouched.
  UpdateResult apply_weight_update(int new_version, rlmath::Policy policy) {
    b200::NativePolicy p(policy);
    std::int32_t v = 0;
    const int st = srl_engine_apply_weight_update(e_, new_version, p.get(), &v);
    if (st == SRL_OK) return {true, v, ""};
    if (st == SRL_VERSION_CONFLICT || st == SRL_INVALID_POLICY || st == SRL_POLICY_MISMATCH)
      return {false, weight_version(), srl_status_string(st)};
    b200::check(st, "apply_weight_update");
    return {};
  }

  long long advance(int rounds) {  // engine.cpp:174-187
    if (rounds < 0) throw std::invalid_argument("advance: negative round count");
    std::int64_t emitted = 0;
    b200::check(srl_engine_advance(e_, rounds, &emitted), "advance");
    return emitted;
  }
  void pause() { b200::check(srl_engine_pause(e_), "pause"); }
  void resume() { b200::check(srl_engine_resume(e_), "resume"); }

  int weight_version() const {
    std::int32_t v = 0;
    b200::check(srl_engine_weight_version(e_, &v), "weight_version");
    return v;
  }
  int active_streams() const {
    std::int32_t v = 0;
    b200::check(srl_engine_active_streams(e_, &v), "active_streams");
    return v;
  }
  long long total_streams() const {
    std::int64_t v = 0;
    b200::check(srl_engine_total_streams(e_, &v), "total_streams");
    return v;
  }
  long long rounds_done() const {
    std::int64_t v = 0;
    b200::check(srl_engine_rounds_done(e_, &v), "rounds_done");
    return v;
  }
  bool recompute_state_mode() const { return recompute_; }

  void set_process_group(std::string group_id, std::vector<std::string> members) {
    std::vector<const char*> m;
    for (const auto& s : members) m.push_back(s.c_str());
    b200::check(srl_engine_set_process_group(e_, group_id.c_str(), m.data(), static_cast<std::int32_t>(m.size())),
                "set_process_group");
  }
  std::optional<std::string> process_group_id() const {
    char buf[256];
    std::int32_t has = 0;
    b200::check(srl_engine_process_group_id(e_, buf, sizeof(buf), &has), "process_group_id");
    if (!has) return std::nullopt;
    return std::string(buf);
  }

  void stop() { b200::check(srl_engine_stop(e_), "stop"); }

  // The device handle, for the update channel (srl_comm_recv_weights_*) and
  // the zero-copy begin / commit update path.
  srl_engine* native() const { return e_; }

 private:
  static std::int64_t parse_id(const std::string& id) {
    if (id.size() < 2 || id[0] != 's' || id.find_first_not_of("0123456789", 1) != std::string::npos)
      throw std::invalid_argument("unknown stream id " + id);
    return std::stoll(id.substr(1));
  }
  srl_engine* e_ = nullptr;
  bool recompute_ = false;
};

// engine.cpp:257-274: CRC-32 (IEEE, reflected 0xEDB88320) of the update payload.
inline std::uint32_t crc32(std::string_view bytes) { return srl_crc32(bytes.data(), bytes.size()); }

// engine.cpp:276-291: order-insensitive group id.
inline std::string process_group_id(std::vector<std::string> members) {
  std::vector<const char*> m;
  for (const auto& s : members) m.push_back(s.c_str());
  char buf[64];
  b200::check(srl_process_group_id(m.data(), static_cast<std::int32_t>(m.size()), buf, sizeof(buf)),
              "process_group_id");
  return buf;
}

}  // namespace streamrl::proto
