// trainer.hpp -- DecoderTrainer: IS-REINFORCE gradient of the decoder policy
// on the device (see trainer.cpp).
#pragma once
#include <memory>
#include <vector>

#include "gemm.cuh"
#include "runtime.hpp"

namespace srl {

// A packed batch of sequences: rows (seq, pos) with input and target token.
struct TrainBatch {
  int rows = 0;
  int n_trajectories = 1;  // m of rl_math.cpp:219 (1/m normalisation)
  double clamp = 5.0;
  int granularity = 0;     // 0 Sequence, 1 PerToken (rl_math.hpp:52)
  int n_loss_rows = 0;
  std::vector<int32_t> seq_start, seq_len, loss_begin;  // per sequence (rows)
  std::vector<int32_t> row_slot, row_pos, row_token, row_target;
  std::vector<double> row_mu, row_adv;  // behaviour log-prob and advantage of each row's target
};

class DecoderTrainer {
 public:
  ~DecoderTrainer();
  int init(const DecoderWeights& w, const srl_trainer_options& o);
  int step(const TrainBatch& b, srl_trainer_stats* stats);
  int apply_adam(float lr, float beta1, float beta2, float eps);
  float* gradient() const { return grad_; }
  cudaStream_t stream() const { return st_; }
  int device() const { return dev_; }
  size_t elements() const { return n_; }
  DecoderWeights& weights() { return *weights_; }
  const std::vector<double>& last_logprobs() const { return lp_host_; }

 private:
  struct LayerActs {
    float *x_in = nullptr, *rstd1 = nullptr, *lse = nullptr, *x_mid = nullptr, *rstd2 = nullptr;
    __nv_bfloat16 *xg1 = nullptr, *q = nullptr, *attn = nullptr, *xg2 = nullptr, *act = nullptr,
                  *gu = nullptr;  // rstd-scaled gate | up pre-activations (bf16, 64-row interleave,
                                      // token-blocked: gemm.cuh gu_index)
    float* gu32 = nullptr;        // the same in fp32 (precise mode)
  };
  // Split operands of the precise mode (EpiParams::seg_kb): up to 3 segments
  // of the K concatenation with per-segment X / W offsets, and the column
  // counts of the X / W buffers (0: the logical width).
  struct Seg {
    int n = 1;
    int x_off[3] = {0, 0, 0}, w_off[3] = {0, 0, 0};
    int x_cols = 0, w_cols = 0;
  };
  // (hi + lo) . W: X rows [hi (w) | lo (w)], W exact
  static Seg seg_x(int w) {
    Seg s;
    s.n = 2; s.x_off[1] = w; s.x_cols = 2 * w;
    return s;
  }
  // (dh + dl)^T (uh + ul) ~ dh uh + dh ul + dl uh: X rows [dh | dl] (width xw),
  // W rows [uh | ul] (width ww), both MN-major
  static Seg seg_xw(int xw, int ww) {
    Seg s;
    s.n = 3; s.x_off[2] = xw; s.w_off[1] = ww; s.x_cols = 2 * xw; s.w_cols = 2 * ww;
    return s;
  }
  template <typename T>
  int alloc(T** p, size_t n);
  int gemm(const __nv_bfloat16* X, int x_rows_alloc, int M, const __nv_bfloat16* W, int N, int K,
           const EpiParams& e);
  int gemm_store(const __nv_bfloat16* X, int M, const __nv_bfloat16* W, int N, int K, float* out);
  int gemm_accum(const __nv_bfloat16* X, int M, const __nv_bfloat16* W, int N, int K, float* out);
  int gemm_mn(const __nv_bfloat16* X, bool x_kmajor, int M, const __nv_bfloat16* W, int N, int k_rows,
              float* out, bool accumulate, const Seg* seg = nullptr);
  int gemm_swiglu_bwd(const __nv_bfloat16* dY, int M, const __nv_bfloat16* W, int I, int k_rows,
                      const __nv_bfloat16* gu, __nv_bfloat16* dgu, const LayerActs* a = nullptr);
  static void apply_seg(EpiParams& e, const Seg* seg, int K);

  srl_trainer_options opts_{};
  DecoderDims d_{};
  WeightLayout lay_{};
  std::shared_ptr<DecoderWeights> weights_;
  size_t n_ = 0;
  int dev_ = 0, T_max_ = 64, sms_ = 148, adam_t_ = 0;
  bool precise_ = true;  // split (hi + lo) activations and backward operands
  int sp_ = 2;           // 2 when precise (split buffers are twice as wide), else 1
  cudaStream_t st_ = nullptr;
  std::vector<void*> allocs_;
  float *master_ = nullptr, *grad_ = nullptr, *adam_m_ = nullptr, *adam_v_ = nullptr;
  int* tile_flags_ = nullptr;  // ordered split-K counters of gemm_mn (self-resetting)
  std::vector<LayerActs> acts_;
  int chunk_ = 512;  // LM-head rows per pass (trainer.cpp, kLogitChunkMax)
  float *x_ = nullptr, *rstdF_ = nullptr, *ssq_ = nullptr, *pmax_ = nullptr;
  double* psum_ = nullptr;
  __nv_bfloat16 *xgF_ = nullptr, *dlogits_ = nullptr, *dbig_bf_ = nullptr, *xn_ = nullptr,
                *dgu_ = nullptr;
  float *dx_ = nullptr, *dz_ = nullptr, *dbig_ = nullptr, *ones_ = nullptr, *coef_ = nullptr,
        *cos_sin_ = nullptr;
  double* lp_ = nullptr;
  double* lse_ = nullptr;       // per row, from pass 1 (reused by the pass-2 dlogits epilogue)
  float* tgt_logit_ = nullptr;  // per row: the target's logit (pass 1)
  int32_t *row_slot_ = nullptr, *row_pos_ = nullptr, *row_tok_ = nullptr, *row_tgt_ = nullptr;
  __nv_bfloat16 *kc_ = nullptr, *vc_ = nullptr;
  size_t kv_cap_ = 0;
  float* ws_ = nullptr;  // split-K partials
  size_t ws_floats_ = 0;
  std::vector<double> lp_host_;
};

}  // namespace srl
