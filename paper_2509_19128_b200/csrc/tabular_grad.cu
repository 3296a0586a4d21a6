// tabular_grad.cu -- is_reinforce_gradient / reinforce_gradient for the
// reference's TabularPolicy on the device (rl_math.cpp:211-276).
//
// The reference walks trajectories in order and, per position t with a
// non-zero scale = (1/m) * w * (R - b(prompt, t)), adds
// scale * (onehot(y_t) - softmax(row)) into the gradient row of the context
// that produced y_t (a policy row, or the default row).  Here:
//   * per-token log pi(y_t) come from the device policy (toy.cu, fp64, the
//     reference's log-softmax order);
//   * the host forms the IS weights (truncated_is_weight, scalar per
//     sequence or per token) and each token's row -- context_at / find_row,
//     a std::map lookup -- and lays the contributions out by row in the
//     reference's visiting order (CSR);
//   * one CTA per gradient row: softmax of the row in numeric.hpp's order,
//     then thread k accumulates its column over the row's contributions in
//     that same order, mul and add rounded separately (no FMA contraction,
//     as the reference's x86-64 build).  Results equal the reference's up to
//     the last-ulp differences of the device exp/log from glibc's.
#include <algorithm>
#include <cmath>
#include <map>
#include <numeric>

#include "runtime.hpp"

namespace srl {

int toy_policy_logprobs(const Policy& p, const std::string& prompt_id, const std::vector<int32_t>& tokens,
                        std::vector<double>& out, int device);

namespace {

__global__ void tabular_grad_kernel(const double* __restrict__ row_logits, const double* __restrict__ default_logits,
                                    int has_default, int n_rows, int V, const int64_t* __restrict__ row_ptr,
                                    const int32_t* __restrict__ tok, const double* __restrict__ scale,
                                    double* __restrict__ grad) {
  extern __shared__ double s_prob[];
  __shared__ double s_lse;
  const int r = blockIdx.x;  // n_rows = the default row
  const int64_t b = row_ptr[r], e = row_ptr[r + 1];
  if (b == e) return;
  const double* logits = r < n_rows ? row_logits + (size_t)r * V : (has_default ? default_logits : nullptr);
  if (logits == nullptr) {  // uniform fallback (policy.cpp:62-64)
    for (int k = threadIdx.x; k < V; k += blockDim.x) s_prob[k] = 1.0 / V;
    __syncthreads();
  } else {
    if (threadIdx.x == 0) {  // numeric::log_sum_exp, sequential
      double m = -INFINITY;
      for (int k = 0; k < V; ++k) m = logits[k] > m ? logits[k] : m;
      double lse = m;
      if (isfinite(m)) {
        double s = 0.0;
        for (int k = 0; k < V; ++k) s = __dadd_rn(s, exp(__dadd_rn(logits[k], -m)));
        lse = __dadd_rn(m, log(s));
      }
      s_lse = lse;
    }
    __syncthreads();
    for (int k = threadIdx.x; k < V; k += blockDim.x) s_prob[k] = exp(__dadd_rn(logits[k], -s_lse));
    __syncthreads();
  }
  for (int k = threadIdx.x; k < V; k += blockDim.x) {
    double acc = 0.0;
    const double pk = s_prob[k];
    for (int64_t j = b; j < e; ++j) {
      const double ind = tok[j] == k ? 1.0 : 0.0;
      acc = __dadd_rn(acc, __dmul_rn(scale[j], __dadd_rn(ind, -pk)));
    }
    grad[(size_t)r * V + k] = acc;
  }
}

int find_row(const TabularHost& t, const std::string& prompt, const int32_t* tokens, int position) {
  // context_at (policy.cpp:46-52): the last min(order, position) tokens
  const int window = std::min(t.order, position);
  for (size_t r = 0; r < t.rows.size(); ++r) {
    const TabularRow& row = t.rows[r];
    if (row.prompt_id != prompt || (int)row.context.size() != window) continue;
    if (std::equal(row.context.begin(), row.context.end(), tokens + (position - window))) return (int)r;
  }
  return -1;
}

}  // namespace

int tabular_is_reinforce_gradient(const Policy& p, int n_traj, const char* const* prompt_ids,
                                  const int32_t* tokens, const int64_t* offsets, const double* mu,
                                  const double* rewards, const double* baseline, bool use_is, double clamp,
                                  int granularity, double* grad_out, int32_t* touched_out, int device) {
  if (p.type != SRL_POLICY_TABULAR) return fail(SRL_INVALID_ARGUMENT, "gradient: needs a tabular policy");
  if (n_traj < 1) return fail(SRL_INVALID_ARGUMENT, "reinforce_gradient: no trajectories");
  if (use_is && (clamp <= 0.0 || !std::isfinite(clamp)))
    return fail(SRL_INVALID_ARGUMENT, "truncated_is_weight: clamp must be positive");
  const TabularHost& t = p.tab;
  const int V = t.vocab, R = (int)t.rows.size();
  const double inv_m = 1.0 / (double)n_traj;
  std::vector<std::vector<std::pair<int32_t, double>>> per_row(R + 1);
  for (int q = 0; q < n_traj; ++q) {
    const int64_t o = offsets[q], n = offsets[q + 1] - o;
    if (n < 1) return fail(SRL_INVALID_ARGUMENT, "Trajectory: empty token sequence");
    for (int64_t i = 0; i < n; ++i)
      if (tokens[o + i] < 0 || tokens[o + i] >= V)
        return fail(SRL_INVALID_ARGUMENT, "token " + std::to_string(tokens[o + i]) + " out of vocab range");
    const std::string prompt = prompt_ids[q] ? prompt_ids[q] : "";
    std::vector<double> lp;
    int st = toy_policy_logprobs(p, prompt, std::vector<int32_t>(tokens + o, tokens + o + n), lp, device);
    if (st != SRL_OK) return st;
    double seq_w = 1.0;
    if (use_is && granularity == 0) {  // truncated_is_weight of the sums (rl_math.cpp:226-229)
      const double pi = std::accumulate(lp.begin(), lp.end(), 0.0);
      const double mus = std::accumulate(mu + o, mu + o + n, 0.0);
      if (!std::isfinite(pi) || !std::isfinite(mus))
        return fail(SRL_INVALID_ARGUMENT, "truncated_is_weight: non-finite log-probability");
      seq_w = std::min(clamp, std::exp(pi - mus));
    }
    for (int64_t i = 0; i < n; ++i) {
      const double adv = rewards[q] - baseline[o + i];
      double w = seq_w;
      if (use_is && granularity == 1) {
        if (!std::isfinite(lp[i]) || !std::isfinite(mu[o + i]))
          return fail(SRL_INVALID_ARGUMENT, "truncated_is_weight: non-finite log-probability");
        w = std::min(clamp, std::exp(lp[i] - mu[o + i]));
      }
      const double scale = inv_m * w * adv;
      if (scale == 0.0) continue;  // rl_math.cpp:237
      int r = find_row(t, prompt, tokens + o, (int)i);
      if (r < 0) r = R;  // the default row
      per_row[r].emplace_back(tokens[o + i], scale);
    }
  }
  std::vector<int64_t> row_ptr(R + 2, 0);
  std::vector<int32_t> tok;
  std::vector<double> sc;
  for (int r = 0; r <= R; ++r) {
    for (auto& [k, s] : per_row[r]) {
      tok.push_back(k);
      sc.push_back(s);
    }
    row_ptr[r + 1] = (int64_t)tok.size();
    touched_out[r] = per_row[r].empty() ? 0 : 1;
  }
  std::fill(grad_out, grad_out + (size_t)(R + 1) * V, 0.0);
  if (tok.empty()) return SRL_OK;
  SRL_CUDA(cudaSetDevice(device));
  std::vector<double> lg;
  for (const TabularRow& row : t.rows) lg.insert(lg.end(), row.logits.begin(), row.logits.end());
  double *d_lg = nullptr, *d_def = nullptr, *d_sc = nullptr, *d_grad = nullptr;
  int64_t* d_ptr = nullptr;
  int32_t* d_tok = nullptr;
  auto cleanup = [&] {
    for (void* q : {(void*)d_lg, (void*)d_def, (void*)d_sc, (void*)d_grad, (void*)d_ptr, (void*)d_tok})
      if (q) cudaFree(q);
  };
  cudaError_t err = cudaSuccess;
  auto up = [&](auto** dst, const auto& src) {
    if (err != cudaSuccess || src.empty()) return;
    const size_t bytes = src.size() * sizeof(src[0]);
    if ((err = cudaMalloc(dst, bytes)) == cudaSuccess)
      err = cudaMemcpy(*dst, src.data(), bytes, cudaMemcpyHostToDevice);
  };
  up(&d_lg, lg);
  up(&d_def, t.default_logits);
  up(&d_sc, sc);
  up(&d_ptr, row_ptr);
  up(&d_tok, tok);
  if (err == cudaSuccess) err = cudaMalloc(&d_grad, sizeof(double) * (size_t)(R + 1) * V);
  if (err == cudaSuccess) err = cudaMemset(d_grad, 0, sizeof(double) * (size_t)(R + 1) * V);
  if (err == cudaSuccess) {
    tabular_grad_kernel<<<R + 1, 128, sizeof(double) * (size_t)V>>>(d_lg, d_def, t.default_logits.empty() ? 0 : 1,
                                                                   R, V, d_ptr, d_tok, d_sc, d_grad);
    err = cudaGetLastError();
  }
  if (err == cudaSuccess)
    err = cudaMemcpy(grad_out, d_grad, sizeof(double) * (size_t)(R + 1) * V, cudaMemcpyDeviceToHost);
  cleanup();
  if (err != cudaSuccess) return cuda_fail(err, "tabular gradient");
  return SRL_OK;
}

}  // namespace srl
