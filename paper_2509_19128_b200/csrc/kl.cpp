// kl.cpp -- kl_per_position (rl_math.cpp:336-372) for the decoder policy on
// the device: mean exact categorical KL(behaviour || target) per position
// over teacher-forced prefixes, the behaviour being the mixed checkpoint
// chain of a MixedPolicySchedule (rl_math.cpp:286-310) walked as
// PolicyWalker walks it (rl_math.cpp:27-82) and as the engine serves it:
//   * position t is computed under checkpoint segment_at(t) (clamped to the
//     last checkpoint): the forward of input row t (bos, then prefix[t-1])
//     writes that row's K/V and attends to the cache of rows [0, t);
//   * stale (PipelineRL): the cache keeps the rows earlier checkpoints wrote;
//   * recompute: at a switch to checkpoint g at position s the cache rows
//     [0, s) are rebuilt under g first (engine.cpp:107-113).
// The target walks the prefix under one policy.  Both sides run the
// DecoderRunner's chunked forward + LM head; row_kl_kernel forms the KL of
// the two [rows x V] logits blocks in fp64; the per-position means are
// accumulated on the host in the reference's order (prefixes in order).
#include <algorithm>
#include <cmath>

#include "decoder_engine.hpp"

namespace srl {

int decoder_kl_per_position(const std::vector<const DecoderWeights*>& ck, const std::vector<int>& switch_points,
                            bool recompute, const DecoderWeights& target,
                            const std::vector<std::vector<int32_t>>& prefixes, std::vector<double>& out) {
  if (ck.empty()) return fail(SRL_INVALID_ARGUMENT, "kl: empty behavior spec");
  for (const DecoderWeights* w : ck)
    if (!same_decoder_shape(w->cfg, target.cfg) || w->device != target.device)
      return fail(SRL_INVALID_ARGUMENT, "kl: checkpoints and target differ in shape or device");
  for (size_t i = 1; i < switch_points.size(); ++i)
    if (switch_points[i] <= switch_points[i - 1]) return fail(SRL_INVALID_ARGUMENT, "kl: switch points not increasing");
  size_t max_pos = 0;
  for (const auto& p : prefixes) {
    if (p.empty()) return fail(SRL_INVALID_ARGUMENT, "Trajectory: empty token sequence");
    for (int32_t t : p)
      if (t < 0 || t >= target.dims.V)
        return fail(SRL_INVALID_ARGUMENT, "token " + std::to_string(t) + " out of vocab range");
    max_pos = std::max(max_pos, p.size());
  }
  out.assign(max_pos, 0.0);
  if (prefixes.empty()) return SRL_OK;
  if ((int)max_pos + 1 > target.dims.max_pos) return fail(SRL_INVALID_ARGUMENT, "prefix longer than max_positions");
  const int dev = target.device;
  SRL_CUDA(cudaSetDevice(dev));
  cudaStream_t st = nullptr;
  SRL_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  const int chunk = (int)std::min<size_t>(max_pos, 512);
  DecoderRunner rb, rt;  // behaviour and target, one slot each, the same stream
  int status = rb.init(target.dims, target.layout, 1, (int)max_pos + 1, chunk, chunk, dev, st);
  if (status == SRL_OK) status = rt.init(target.dims, target.layout, 1, (int)max_pos + 1, chunk, chunk, dev, st);
  std::vector<WeightMaps> maps;
  for (const DecoderWeights* w : ck) maps.push_back(build_weight_maps(w->dims, w->layout, w->w));
  const WeightMaps tmaps = build_weight_maps(target.dims, target.layout, target.w);
  double* dkl = nullptr;
  if (status == SRL_OK && cudaMalloc(&dkl, sizeof(double) * chunk) != cudaSuccess)
    status = cuda_fail(cudaGetLastError(), "kl alloc");
  std::vector<int32_t> rs(chunk, 0), rp(chunk), rtok(chunk);
  std::vector<double> kl(chunk);
  std::vector<long long> counts(max_pos, 0);
  auto segment = [&](int pos) {
    int g = 0;
    for (int s : switch_points) {
      if (pos >= s) ++g;
      else break;
    }
    return std::min<int>(g, (int)ck.size() - 1);
  };
  // forward rows [c0, c1) of `prefix` on runner r with weights w (input row p = bos, then prefix[p-1])
  auto run = [&](DecoderRunner& r, const DecoderWeights& w, const WeightMaps& wm, const std::vector<int32_t>& prefix,
                 int c0, int c1, bool logits) -> int {
    const int M = c1 - c0;
    for (int i = 0; i < M; ++i) {
      rp[i] = c0 + i;
      rtok[i] = c0 + i == 0 ? w.dims.bos : prefix[c0 + i - 1];
    }
    cudaMemcpyAsync(r.plan.row_slot, rs.data(), 4 * (size_t)M, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(r.plan.row_pos, rp.data(), 4 * (size_t)M, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(r.plan.row_token, rtok.data(), 4 * (size_t)M, cudaMemcpyHostToDevice, st);
    int s2 = r.forward(M, w.w, wm);
    if (s2 == SRL_OK && logits) s2 = r.lm_head(M, wm, false);
    // the plan buffers are reused by the next call: finish this one first
    if (s2 == SRL_OK && cudaStreamSynchronize(st) != cudaSuccess) s2 = cuda_fail(cudaGetLastError(), "kl forward");
    return s2;
  };
  for (size_t q = 0; q < prefixes.size() && status == SRL_OK; ++q) {
    const auto& pre = prefixes[q];
    const int n = (int)pre.size();
    int cur = 0;
    for (int c0 = 0; c0 < n && status == SRL_OK;) {
      const int g = segment(c0);
      int c1 = std::min(n, c0 + chunk);
      for (int s : switch_points)
        if (s > c0 && s < c1) { c1 = s; break; }  // a chunk never spans a switch
      if (recompute && g != cur) {  // rebuild rows [0, c0) under checkpoint g
        for (int r0 = 0; r0 < c0 && status == SRL_OK; r0 += chunk)
          status = run(rb, *ck[g], maps[g], pre, r0, std::min(c0, r0 + chunk), false);
      }
      cur = g;
      if (status == SRL_OK) status = run(rb, *ck[g], maps[g], pre, c0, c1, true);
      if (status == SRL_OK) status = run(rt, target, tmaps, pre, c0, c1, true);
      if (status != SRL_OK) break;
      launch_row_kl(rb.logits, rt.logits, target.dims.V, c1 - c0, dkl, st);
      if (cudaMemcpyAsync(kl.data(), dkl, sizeof(double) * (c1 - c0), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
          cudaStreamSynchronize(st) != cudaSuccess) {
        status = cuda_fail(cudaGetLastError(), "kl");
        break;
      }
      for (int i = 0; i < c1 - c0; ++i) {
        out[c0 + i] += kl[i];
        counts[c0 + i] += 1;
      }
      c0 = c1;
    }
  }
  for (size_t t = 0; t < max_pos; ++t)
    if (counts[t] > 0) out[t] /= (double)counts[t];
  if (dkl) cudaFree(dkl);
  cudaStreamDestroy(st);
  return status;
}

}  // namespace srl
