// decoder_engine.hpp -- DecoderRunner (device buffers + varlen forward) and
// DecoderBackend (the Engine backend for decoder policies).
#pragma once
#include <memory>
#include <vector>

#include "decode_mk.cuh"
#include "gemm.cuh"
#include "runtime.hpp"

namespace srl {

struct WeightMaps {  // TMA descriptors of one flat weight buffer
  std::vector<CUtensorMap> qkv, o, gate_up, down;
  CUtensorMap lm_head;
};
WeightMaps build_weight_maps(const DecoderDims& d, const WeightLayout& lay, const __nv_bfloat16* w);

// CUDA-event timer around individual launches (profiled rounds only).
struct KernelTimer {
  std::vector<cudaEvent_t> pool;
  std::vector<int> kinds;
  size_t used = 0;
  cudaStream_t st = nullptr;
  void begin(int kind);
  void end();
  void reset() { used = 0; kinds.clear(); }
  void collect(srl_kernel_profile* out);
  ~KernelTimer();
};

// Activations for up to M_max rows, a paged KV cache for S slots x max_seq
// tokens, and the split-K / split-KV workspaces.
struct DecoderRunner {
  DecoderDims d{};
  WeightLayout lay{};
  int S = 0, max_seq = 0, pages_per_seq = 0, M_max = 0, logits_rows = 0, dev = 0, sms = 148;
  size_t kv_layer_elems = 0;
  float* x = nullptr;             // [M_max x H] fp32 residual stream
  __nv_bfloat16* xg = nullptr;    // [M_max x H] bf16(x * next RMSNorm gain)
  float* ssq = nullptr;           // [M_max x ceil(H/128)] partial sums of x^2
  float* qkv = nullptr;           // [M_max x (nq+2nkv)hd]
  __nv_bfloat16* q = nullptr;     // [M_max x nq hd] (RoPE applied)
  __nv_bfloat16* attn = nullptr;  // [M_max x nq hd]
  __nv_bfloat16* act = nullptr;   // [M_max x I]
  __nv_bfloat16* xg_last = nullptr;
  float* ssq_last = nullptr;
  float* logits = nullptr;        // [logits_rows x V]
  float* lse_max = nullptr;       // [logits_rows x ceil(V/128)] per-tile max
  double* lse_sum = nullptr;      // [logits_rows x ceil(V/128)] per-tile fp64 sum exp(x - max)
  __nv_bfloat16 *kc = nullptr, *vc = nullptr;  // [L][pages][nkv][64][hd]
  int32_t* block_table = nullptr;
  float* cos_sin = nullptr;
  RoundPlan plan{}, next{};
  GemmWorkspace gws{};
  float* attn_ws = nullptr;
  int* attn_counters = nullptr;
  size_t attn_ws_floats = 0;
  CUtensorMap xg_map[2], attn_map[2], act_map[2], last_map[2];
  // Prompt / recompute segments of the next forward (tensor-core attention):
  // rows [0, n_single) attend one query each (per-row kernel); segment y covers
  // rows seg[y] .. + seg[S + y] at positions seg[2S + y] .. of slot seg[3S + y].
  int32_t* seg = nullptr;         // device [4][slots]
  int n_seg = 0, n_single = 0, seg_max_rows = 0;
  KernelTimer* timer = nullptr;  // set for a profiled round
  bool unfused_qkv = false;
  bool precise = false;  // split (hi + lo) activations between the GEMMs
  int sp = 1;            // 2 when precise: the split buffers are twice as wide
  void tb(int kind) { if (timer) timer->begin(kind); }
  void te() { if (timer) timer->end(); }

  ~DecoderRunner();
  int init(const DecoderDims& dims, const WeightLayout& layout, int slots, int max_seq, int m_max,
           int logits_rows, int device, cudaStream_t st, bool precise_mode = false);
  int forward(int M, const __nv_bfloat16* w, const WeightMaps& wm);
  int lm_head(int rows, const WeightMaps& wm, bool gathered);
  int gemm(const CUtensorMap& tw, const CUtensorMap* tx, int M, int N, int K, const EpiParams& e);
  cudaStream_t stream() const { return st_; }

 private:
  cudaStream_t st_ = nullptr;
  // a prefill round's single-row attention runs beside the segment attention
  cudaStream_t side_ = nullptr;
  cudaEvent_t fork_ = nullptr, join_ = nullptr;
  std::vector<void*> allocs_;
};

class DecoderBackend final : public Backend {
 public:
  DecoderBackend(const Policy& p, const srl_engine_options& o);
  ~DecoderBackend() override;
  int init(const Policy& p);
  int slots() const override { return S_; }
  int open_slot(int slot, const StreamSpec& spec) override;
  void close_slot(int slot) override;
  int run_rounds(int n, std::vector<SlotEvent>& events, double* device_ms) override;
  void prefill_stats(srl_engine_stats* s) const override {
    s->prefill_rounds = prefill_rounds_;
    s->prefill_rows = prefill_rows_;
    s->prefill_ms = prefill_ms_;
  }
  int check_update(const Policy& p) override;
  int apply_update(const Policy& p, bool recompute, int version) override;
  int check_stream(const StreamSpec& spec) const override;
  int standby(void** ptr, size_t* bytes) override;
  int commit_standby(bool recompute, int version) override;
  int slot_history(int slot, std::vector<int32_t>& out) override;
  void request_profile() override { profile_next_ = true; }
  bool kernel_profile(srl_kernel_profile* out) const override {
    *out = profile_;
    return profile_.valid != 0;
  }

 private:
  struct HostSlot {
    bool live = false, pending = false;
    int fed = 0;                  // tokens already in the KV cache
    std::vector<int32_t> tokens;  // bos + prompt + generated
  };
  int decode_round_eager(int b);
  int capture(int b);
  // persistent megakernel decode rounds (decode_mk.cu)
  int mega_init();
  int mega_round(int b, bool profile);
  int prefill_round(int b, std::vector<int>& prefilled);
  int swap_and_recompute(bool recompute, int version);
  int recompute_kv();

  srl_engine_options opts_;
  DecoderDims d_{};
  int S_ = 1, max_seq_ = 2, R_ = 1, prefill_budget_ = 1;
  std::shared_ptr<DecoderWeights> buf_[2];
  WeightMaps maps_[2];
  int active_ = 0;
  std::unique_ptr<DecoderRunner> runner_;
  cudaStream_t st_ = nullptr;
  cudaGraphExec_t exec_[2] = {nullptr, nullptr};
  cudaEvent_t ev_start_ = nullptr, ev_stop_ = nullptr;
  cudaEvent_t ev_prof_[2] = {nullptr, nullptr};  // around a profiled megakernel launch
  cudaEvent_t ev_pf_[2] = {nullptr, nullptr};    // around a prefill round
  int32_t* slot_stage_ = nullptr;  // pinned [slots x max_seq] prompt staging (open_slot)
  int64_t prefill_rounds_ = 0, prefill_rows_ = 0;
  double prefill_ms_ = 0.0;
  int last_prefill_rows_ = 0;
  void* dev_state_ = nullptr;
  void* pinned_ = nullptr;
  size_t pinned_bytes_ = 0;
  SlotState ss_{};
  EventRing ring_{};
  int32_t* version_dev_ = nullptr;
  int32_t* round_ctr_dev_ = nullptr;
  int64_t round_ctr_host_ = 0;
  std::vector<HostSlot> host_;
  bool any_pending_ = false;
  bool profile_next_ = false;
  srl_kernel_profile profile_{};
  KernelTimer timer_;
  struct Mega {
    bool on = false;
    int grid = 0, n_phases = 0;
    std::vector<MkPhase> phases;         // host copy (profile class mapping)
    MkParams params[2]{};                // per weight buffer
    CUtensorMap* wmaps[2] = {nullptr, nullptr};
    void* mem = nullptr;                 // phases, layers, xmaps, counters, stamps
    float* ws = nullptr;
    float* qkv_part = nullptr;
    unsigned long long* stamps = nullptr;
    unsigned long long* stamps_host = nullptr;
    unsigned long long* trace = nullptr;  // SRL_MK_TRACE=<file>: per-CTA phase timestamps
  } mk_;
};

}  // namespace srl
