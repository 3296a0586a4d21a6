// engine.cpp -- Engine: the streamrl::proto::Engine contract over a device
// backend.  One std::mutex guards all state and every batch of rounds runs to
// completion on the device under it, so weight swaps land exactly on token
// boundaries (reference src/engine.cpp:103-104).  A background scheduler
// thread runs rounds while streams are live, or only on advance() when
// paused (lockstep mode, engine.cpp:155-187).
#include <algorithm>
#include <chrono>
#include <cstdio>

#include "runtime.hpp"

namespace srl {

int cuda_fail(cudaError_t e, const char* where) {
  set_last_error(std::string(where) + ": " + cudaGetErrorString(e));
  if (e == cudaErrorMemoryAllocation) return SRL_OUT_OF_MEMORY;
  if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) return SRL_NO_DEVICE;
  return SRL_CUDA_ERROR;
}

Engine::Engine(std::unique_ptr<Backend> backend, Policy policy, bool recompute, bool start_paused,
               const srl_engine_options& opts)
    : backend_(std::move(backend)), policy_(std::move(policy)), recompute_(recompute), opts_(opts) {
  paused_ = start_paused;
  slot_owner_.assign(backend_->slots(), nullptr);
  scheduler_ = std::thread([this] { scheduler_loop(); });
}

Engine::~Engine() { stop(); }

Engine::Stream* Engine::find(int64_t id) {
  if (id < 0 || id >= (int64_t)streams_.size()) return nullptr;
  return streams_[id].get();
}

// engine.cpp:46-61
int Engine::open_stream(const std::string& prompt_id, int max_tokens, uint64_t seed,
                        int32_t terminator, const std::vector<int32_t>& prompt, int64_t* id) {
  if (max_tokens < 1) return fail(SRL_INVALID_ARGUMENT, "open_stream: max_tokens must be >= 1");
  std::lock_guard<std::mutex> lk(lock_);
  auto s = std::make_unique<Stream>();
  s->id = next_stream_++;
  s->spec.prompt_index = backend_->prompt_index(prompt_id);
  s->spec.prompt = prompt;
  s->spec.seed = seed;
  s->spec.max_tokens = max_tokens;
  s->spec.terminator = terminator;
  if (policy_.type == SRL_POLICY_DECODER) {
    for (int32_t t : prompt)
      if (t < 0 || t >= policy_.vocab()) {
        --next_stream_;
        return fail(SRL_INVALID_ARGUMENT, "open_stream: prompt token out of vocab");
      }
  }
  if (const int st = backend_->check_stream(s->spec)) {
    --next_stream_;
    return st;
  }
  *id = s->id;
  pending_.push_back(s.get());
  streams_.push_back(std::move(s));
  assign_slots_locked();
  if (stopping_) {
    // engine already stopped: the stream finishes immediately
    streams_.back()->finish = SRL_FINISH_SHUTDOWN;
  }
  cv_.notify_all();
  return SRL_OK;
}

void Engine::assign_slots_locked() {
  for (int slot = 0; slot < (int)slot_owner_.size() && !pending_.empty(); ++slot) {
    if (slot_owner_[slot] != nullptr) continue;
    Stream* s = pending_.front();
    const int st = backend_->open_slot(slot, s->spec);
    if (st != SRL_OK) {
      s->finish = SRL_FINISH_SHUTDOWN;
      pending_.pop_front();
      --slot;
      continue;
    }
    pending_.pop_front();
    s->slot = slot;
    slot_owner_[slot] = s;
  }
}

// engine.cpp:63-77
int Engine::wait_events(int64_t id, std::vector<srl_token_event>& out, int cap, int* reason,
                        int* more, bool block) {
  std::unique_lock<std::mutex> lk(lock_);
  Stream* s = find(id);
  if (s == nullptr) return fail(SRL_UNKNOWN_STREAM, "unknown stream id s" + std::to_string(id));
  if (block) cv_.wait(lk, [&] { return !s->outbox.empty() || s->finish != SRL_FINISH_RUNNING; });
  while (!s->outbox.empty() && (int)out.size() < cap) {
    out.push_back(s->outbox.front());
    s->outbox.pop_front();
  }
  *reason = s->outbox.empty() ? s->finish : SRL_FINISH_RUNNING;
  *more = (!out.empty() || *reason == SRL_FINISH_RUNNING) ? 1 : 0;
  return SRL_OK;
}

// engine.cpp:79-117
int Engine::apply_weight_update(int new_version, const Policy& policy, int* version_out) {
  std::lock_guard<std::mutex> lk(lock_);
  *version_out = version_;
  if (new_version != version_ + 1) return fail(SRL_VERSION_CONFLICT, "version_conflict");
  std::string why;
  if (policy.validate(&why) != SRL_OK) return fail(SRL_INVALID_POLICY, "invalid_policy: " + why);
  if (policy.type != policy_.type || policy.vocab() != policy_.vocab())
    return fail(SRL_POLICY_MISMATCH, "policy_mismatch");
  const int chk = backend_->check_update(policy);
  if (chk != SRL_OK) return chk;
  if (staged_version_ >= 0) return fail(SRL_BUSY, "a staged weight update is pending");
  const auto t0 = std::chrono::steady_clock::now();
  const int st = backend_->apply_update(policy, recompute_, new_version);
  if (st != SRL_OK) return st;
  const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  if (policy.type != SRL_POLICY_DECODER) policy_ = policy;  // decoder weights live in the backend
  version_ = new_version;
  *version_out = version_;
  stats_.updates += 1;
  stats_.last_pause_ms = ms;
  stats_.max_pause_ms = std::max(stats_.max_pause_ms, ms);
  return SRL_OK;
}

int Engine::standby_bytes(size_t* bytes) {
  std::lock_guard<std::mutex> lk(lock_);
  void* p = nullptr;
  return backend_->standby(&p, bytes);
}

int Engine::begin_weight_update(int new_version, void** ptr, size_t* bytes) {
  std::lock_guard<std::mutex> lk(lock_);
  if (new_version != version_ + 1) return fail(SRL_VERSION_CONFLICT, "version_conflict");
  if (staged_version_ >= 0) return fail(SRL_BUSY, "a weight update is already staged");
  const int st = backend_->standby(ptr, bytes);
  if (st != SRL_OK) return st;
  staged_version_ = new_version;
  return SRL_OK;
}

int Engine::commit_weight_update(int new_version, int* version_out, double* pause_ms) {
  const auto t0 = std::chrono::steady_clock::now();
  std::lock_guard<std::mutex> lk(lock_);  // waits for the in-flight rounds: token boundary
  *version_out = version_;
  if (staged_version_ < 0 || new_version != staged_version_ || new_version != version_ + 1)
    return fail(SRL_VERSION_CONFLICT, "version_conflict");
  const auto t1 = std::chrono::steady_clock::now();
  const int st = backend_->commit_standby(recompute_, new_version);
  if (st != SRL_OK) {  // the backend swapped back: version and weights unchanged
    staged_version_ = -1;
    return st;
  }
  const auto t2 = std::chrono::steady_clock::now();
  staged_version_ = -1;
  version_ = new_version;
  *version_out = version_;
  // pause = time the decode loop is blocked by the swap itself (lock held)
  const double ms = std::chrono::duration<double, std::milli>(t2 - t1).count();
  (void)t0;
  if (pause_ms) *pause_ms = ms;
  stats_.updates += 1;
  stats_.last_pause_ms = ms;
  stats_.max_pause_ms = std::max(stats_.max_pause_ms, ms);
  return SRL_OK;
}

int Engine::abort_weight_update() {
  std::lock_guard<std::mutex> lk(lock_);
  staged_version_ = -1;
  return SRL_OK;
}

int Engine::run_rounds_locked(int n, int64_t* emitted) {
  std::vector<SlotEvent> evs;
  double ms = 0.0;
  const int st = backend_->run_rounds(n, evs, &ms);
  if (st != SRL_OK) return -st;
  const int S = backend_->slots();
  int64_t count = 0;
  int64_t rounds_with_events = 0;
  for (int r = 0; r < n; ++r) {
    bool any = false;
    for (int slot = 0; slot < S; ++slot) {
      const SlotEvent& e = evs[(size_t)r * S + slot];
      if (e.flag == 0) continue;
      Stream* s = slot_owner_[slot];
      if (s == nullptr) continue;
      any = true;
      srl_token_event te{};
      te.stream = s->id;
      te.position = e.position;
      te.token = e.token;
      te.logprob = e.logprob;
      te.weight_version = e.version;
      s->outbox.push_back(te);
      ++count;
      if (e.flag >= 2) {
        s->finish = e.flag == 3 ? SRL_FINISH_TERMINATOR : SRL_FINISH_LENGTH;
        backend_->slot_history(slot, s->history);
        backend_->close_slot(slot);
        slot_owner_[slot] = nullptr;
        s->slot = -1;
      }
    }
    if (any) ++rounds_with_events;
  }
  assign_slots_locked();
  stats_.rounds += n;
  stats_.tokens += count;
  stats_.decode_ms += ms;
  if (emitted) *emitted = count;
  return paused_ ? n : (int)rounds_with_events;
}

// engine.cpp:155-172
void Engine::scheduler_loop() {
  for (;;) {
    std::unique_lock<std::mutex> lk(lock_);
    if (stopping_) return;
    bool has_live = false;
    for (Stream* s : slot_owner_)
      if (s != nullptr) { has_live = true; break; }
    const bool runnable = paused_ ? budget_ > 0 : has_live;
    if (!runnable) {
      cv_.wait(lk);
      continue;
    }
    int n = std::max(1, opts_.rounds_per_sync);
    if (paused_) n = (int)std::min<int64_t>(budget_, n);
    const int counted = run_rounds_locked(n, nullptr);
    if (counted < 0) {
      // device failure: fail loudly -- every running stream ends with Shutdown
      last_error_ = -counted;
      std::fprintf(stderr, "srl engine: round failed (%d): %s\n", last_error_, srl_last_error());
      stopping_ = true;
      for (auto& s : streams_)
        if (s->finish == SRL_FINISH_RUNNING) s->finish = SRL_FINISH_SHUTDOWN;
      cv_.notify_all();
      return;
    }
    if (paused_) budget_ -= n;
    rounds_done_ += paused_ ? n : std::max(counted, 0);
    cv_.notify_all();
  }
}

// engine.cpp:174-187
int Engine::advance(int rounds, int64_t* emitted) {
  if (rounds < 0) return fail(SRL_INVALID_ARGUMENT, "advance: negative round count");
  std::unique_lock<std::mutex> lk(lock_);
  if (!paused_) return fail(SRL_LOGIC_ERROR, "advance requires a paused engine");
  int64_t before = stats_.tokens;
  const int64_t target = rounds_done_ + rounds;
  budget_ += rounds;
  cv_.notify_all();
  cv_.wait(lk, [&] { return rounds_done_ >= target || stopping_; });
  if (emitted) *emitted = stats_.tokens - before;
  if (last_error_ != SRL_OK) return fail(last_error_, "engine stopped after a device failure");
  return SRL_OK;
}

void Engine::pause() {
  std::lock_guard<std::mutex> lk(lock_);
  paused_ = true;
}

void Engine::resume() {
  std::lock_guard<std::mutex> lk(lock_);
  paused_ = false;
  budget_ = 0;
  cv_.notify_all();
}

int Engine::weight_version() const {
  std::lock_guard<std::mutex> lk(lock_);
  return version_;
}

int Engine::active_streams() const {
  std::lock_guard<std::mutex> lk(lock_);
  int n = 0;
  for (const auto& s : streams_)
    if (s->finish == SRL_FINISH_RUNNING) ++n;
  return n;
}

int64_t Engine::total_streams() const {
  std::lock_guard<std::mutex> lk(lock_);
  return next_stream_;
}

int64_t Engine::rounds_done() const {
  std::lock_guard<std::mutex> lk(lock_);
  return rounds_done_;
}

void Engine::set_process_group(std::string id, std::vector<std::string> members) {
  std::lock_guard<std::mutex> lk(lock_);
  group_id_ = std::move(id);
  group_members_ = std::move(members);
}

std::optional<std::string> Engine::process_group_id() const {
  std::lock_guard<std::mutex> lk(lock_);
  return group_id_;
}

// engine.cpp:240-253
void Engine::stop() {
  {
    std::lock_guard<std::mutex> lk(lock_);
    if (!stopping_) {
      stopping_ = true;
      for (auto& s : streams_)
        if (s->finish == SRL_FINISH_RUNNING) {
          s->finish = SRL_FINISH_SHUTDOWN;
          if (s->slot >= 0) {
            backend_->slot_history(s->slot, s->history);
            backend_->close_slot(s->slot);
            slot_owner_[s->slot] = nullptr;
            s->slot = -1;
          }
        }
      pending_.clear();
    }
    cv_.notify_all();
  }
  if (scheduler_.joinable()) scheduler_.join();
}

int Engine::stream_tokens(int64_t id, std::vector<int32_t>& out) {
  std::lock_guard<std::mutex> lk(lock_);
  Stream* s = find(id);
  if (s == nullptr) return fail(SRL_UNKNOWN_STREAM, "unknown stream id");
  if (s->slot >= 0) return backend_->slot_history(s->slot, out);
  out = s->history;
  return SRL_OK;
}

srl_engine_stats Engine::stats() const {
  std::lock_guard<std::mutex> lk(lock_);
  srl_engine_stats s = stats_;
  s.launches = backend_->launches();
  backend_->prefill_stats(&s);
  return s;
}

void Engine::profile_next_round() {
  std::lock_guard<std::mutex> lk(lock_);
  backend_->request_profile();
}

bool Engine::kernel_profile(srl_kernel_profile* out) const {
  std::lock_guard<std::mutex> lk(lock_);
  return backend_->kernel_profile(out);
}

}  // namespace srl
