// runtime.hpp -- host-side C++ runtime behind the C ABI: policy checkpoints,
// the device backends that run decode rounds, and the Engine that mirrors
// streamrl::proto::Engine (reference include/streamrl/engine.hpp:44-109).
#pragma once
#include <condition_variable>
#include <cstdint>
#include <deque>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <string>
#include <thread>
#include <vector>

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "decoder.cuh"
#include "streamrl_b200.h"

namespace srl {

void set_last_error(const std::string& s);

// Status with a detail message recorded for srl_last_error().
inline int fail(int status, const std::string& what) {
  set_last_error(what);
  return status;
}
int cuda_fail(cudaError_t e, const char* where);
#define SRL_CUDA(expr)                                   \
  do {                                                   \
    cudaError_t _e = (expr);                             \
    if (_e != cudaSuccess) return cuda_fail(_e, #expr);  \
  } while (0)

// ------------------------------------------------------------- policies ---
struct TabularRow {
  std::string prompt_id;
  std::vector<int32_t> context;
  std::vector<double> logits;
};
struct TabularHost {  // rlmath::TabularPolicy (policy.hpp:16-47)
  int32_t vocab = 0, order = 0;
  std::vector<double> default_logits;  // empty = uniform fallback
  std::vector<TabularRow> rows;        // sorted like std::map<ContextKey, ...>
};
struct RecurrentHost {  // rlmath::RecurrentToyPolicy (policy.hpp:52-72)
  int32_t vocab = 0, hidden = 0;
  std::vector<double> emb, rec, out;
};
// Decoder weights: one flat bf16 device buffer.
struct DecoderWeights {
  srl_decoder_config cfg{};
  DecoderDims dims{};
  WeightLayout layout{};
  __nv_bfloat16* w = nullptr;
  size_t bytes = 0;
  int device = 0;
  ~DecoderWeights();
};

struct Policy {
  int type = SRL_POLICY_TABULAR;
  TabularHost tab;
  RecurrentHost rec;
  std::shared_ptr<DecoderWeights> dec;
  int32_t vocab() const;
  int validate(std::string* why) const;  // policy.cpp:30-43, 71-82
};

// Make a deep copy of a decoder weight buffer on the same device.
// device < 0: the source's device; otherwise the copy lands on `device`
// (a peer copy when it differs from the source's).
int clone_decoder(const DecoderWeights& src, std::shared_ptr<DecoderWeights>& out, int device = -1);
int create_decoder(const srl_decoder_config& cfg, int device, std::shared_ptr<DecoderWeights>& out);
bool same_decoder_shape(const srl_decoder_config& a, const srl_decoder_config& b);

// --------------------------------------------------------------- events ---
struct SlotEvent {
  int32_t flag;  // 0 none, 1 emitted, 2 emitted + Length, 3 emitted + Terminator
  int32_t token;
  int32_t position;
  int32_t version;
  double logprob;
};

struct StreamSpec {
  int prompt_index = 0;            // interned prompt id
  std::vector<int32_t> prompt;     // decoder prompt tokens (bos prepended by the backend)
  uint64_t seed = 0;
  int32_t max_tokens = 1;
  int32_t terminator = -1;
};

// A device backend runs rounds for `slots()` stream slots.
class Backend {
 public:
  virtual ~Backend() = default;
  virtual int slots() const = 0;
  virtual int open_slot(int slot, const StreamSpec& spec) = 0;
  // open-time validation (the reference's invalid_argument at open_stream):
  // a stream the backend could never seat is refused before it is queued
  virtual int check_stream(const StreamSpec& spec) const { (void)spec; return SRL_OK; }
  virtual void close_slot(int slot) = 0;
  // Launch n rounds, wait, and return n x slots events (row-major by round).
  virtual int run_rounds(int n, std::vector<SlotEvent>& events, double* device_ms) = 0;
  // Compatibility of an incoming policy (type / vocab / shape).
  virtual int check_update(const Policy& p) = 0;
  // Swap in new weights at a token boundary (caller holds the engine lock).
  virtual int apply_update(const Policy& p, bool recompute, int version) = 0;
  // Zero-copy path: standby buffer for a broadcast, then swap.
  virtual int standby(void** ptr, size_t* bytes) { return fail(SRL_INVALID_ARGUMENT, "no standby buffer for this policy type"); }
  virtual int commit_standby(bool recompute, int version) { return fail(SRL_INVALID_ARGUMENT, "no standby buffer"); }
  virtual int slot_history(int slot, std::vector<int32_t>& out) = 0;
  virtual void request_profile() {}
  virtual bool kernel_profile(srl_kernel_profile* out) const { return false; }
  virtual int64_t launches() const { return launches_; }
  virtual void prefill_stats(srl_engine_stats* s) const { (void)s; }
  virtual int prompt_index(const std::string& prompt_id) { return intern(prompt_id); }
  int intern(const std::string& s) {
    auto it = prompts_.find(s);
    if (it != prompts_.end()) return it->second;
    const int id = (int)prompts_.size();
    prompts_.emplace(s, id);
    return id;
  }

 protected:
  std::map<std::string, int> prompts_;
  int64_t launches_ = 0;
};

std::unique_ptr<Backend> make_toy_backend(const Policy& p, const srl_engine_options& o, int* status);
std::unique_ptr<Backend> make_decoder_backend(const Policy& p, const srl_engine_options& o, int* status);

// --------------------------------------------------------------- engine ---
class Engine {
 public:
  Engine(std::unique_ptr<Backend> backend, Policy policy, bool recompute, bool start_paused,
         const srl_engine_options& opts);
  ~Engine();
  int open_stream(const std::string& prompt_id, int max_tokens, uint64_t seed, int32_t terminator,
                  const std::vector<int32_t>& prompt, int64_t* id);
  // block = false: return at once with whatever is queued (srl_engine_poll_events_many)
  int wait_events(int64_t id, std::vector<srl_token_event>& out, int cap, int* reason, int* more,
                  bool block = true);
  int apply_weight_update(int new_version, const Policy& policy, int* version_out);
  int begin_weight_update(int new_version, void** ptr, size_t* bytes);
  int standby_bytes(size_t* bytes);
  int commit_weight_update(int new_version, int* version_out, double* pause_ms);
  int abort_weight_update();
  int advance(int rounds, int64_t* emitted);
  void pause();
  void resume();
  int weight_version() const;
  int active_streams() const;
  int64_t total_streams() const;
  int64_t rounds_done() const;
  bool recompute_state_mode() const { return recompute_; }
  int device() const { return opts_.device; }
  void set_process_group(std::string id, std::vector<std::string> members);
  std::optional<std::string> process_group_id() const;
  void stop();
  int stream_tokens(int64_t id, std::vector<int32_t>& out);
  srl_engine_stats stats() const;
  void profile_next_round();
  bool kernel_profile(srl_kernel_profile* out) const;

 private:
  struct Stream {
    int64_t id = 0;
    StreamSpec spec;
    int slot = -1;
    std::deque<srl_token_event> outbox;
    int finish = SRL_FINISH_RUNNING;
    std::vector<int32_t> history;  // tokens at finish (decoder: full KV history)
  };
  void scheduler_loop();
  int run_rounds_locked(int n, int64_t* emitted);
  void assign_slots_locked();
  Stream* find(int64_t id);

  std::unique_ptr<Backend> backend_;
  Policy policy_;
  bool recompute_ = false;
  srl_engine_options opts_{};
  mutable std::mutex lock_;
  std::condition_variable cv_;
  int version_ = 0;
  int64_t next_stream_ = 0;
  std::vector<std::unique_ptr<Stream>> streams_;
  std::vector<Stream*> slot_owner_;
  std::deque<Stream*> pending_;
  std::optional<std::string> group_id_;
  std::vector<std::string> group_members_;
  bool paused_ = false;
  int64_t budget_ = 0;
  int64_t rounds_done_ = 0;
  bool stopping_ = false;
  int staged_version_ = -1;
  srl_engine_stats stats_{};
  int last_error_ = SRL_OK;
  std::thread scheduler_;
};

}  // namespace srl
