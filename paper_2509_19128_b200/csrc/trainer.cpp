// trainer.cpp -- trainer-side device computations of the decoder policy:
// per-token current-policy log-prob recompute (rl_math.cpp:128-142) as a
// chunked varlen forward over the sequence with the LM head on every row.
#include <algorithm>
#include <cstring>

#include "decoder_engine.hpp"

namespace srl {

int decoder_policy_logprobs(const DecoderWeights& w, const std::vector<int32_t>& tokens,
                            std::vector<double>& out) {
  const int n = (int)tokens.size();
  out.assign(n, 0.0);
  if (n == 0) return SRL_OK;
  if (n + 1 > w.dims.max_pos) return fail(SRL_INVALID_ARGUMENT, "sequence longer than max_positions");
  SRL_CUDA(cudaSetDevice(w.device));
  cudaStream_t st = nullptr;
  SRL_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  const int chunk = std::min(n, 512);
  DecoderRunner r;
  int status = r.init(w.dims, w.layout, 1, n + 1, chunk, chunk, w.device, st);
  if (status != SRL_OK) { cudaStreamDestroy(st); return status; }
  const WeightMaps maps = build_weight_maps(w.dims, w.layout, w.w);
  int32_t* dtarget = nullptr;
  double* dout = nullptr;
  SRL_CUDA(cudaMalloc(&dtarget, 4 * (size_t)n));
  SRL_CUDA(cudaMalloc(&dout, 8 * (size_t)n));
  SRL_CUDA(cudaMemcpy(dtarget, tokens.data(), 4 * (size_t)n, cudaMemcpyHostToDevice));
  std::vector<int32_t> rs(chunk, 0), rp(chunk), rt(chunk);
  for (int c0 = 0; c0 < n && status == SRL_OK; c0 += chunk) {
    const int M = std::min(chunk, n - c0);
    for (int i = 0; i < M; ++i) {
      const int p = c0 + i;
      rp[i] = p;
      rt[i] = p == 0 ? w.dims.bos : tokens[p - 1];  // input at position p predicts tokens[p]
    }
    cudaMemcpyAsync(r.plan.row_slot, rs.data(), 4 * (size_t)M, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(r.plan.row_pos, rp.data(), 4 * (size_t)M, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(r.plan.row_token, rt.data(), 4 * (size_t)M, cudaMemcpyHostToDevice, st);
    if ((status = r.forward(M, w.w, maps)) != SRL_OK) break;
    if ((status = r.lm_head(M, maps, false)) != SRL_OK) break;
    launch_row_logprobs(r.logits, w.dims.V, M, dtarget + c0, dout + c0, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) status = cuda_fail(cudaGetLastError(), "logprobs");
  }
  if (status == SRL_OK) {
    if (cudaMemcpy(out.data(), dout, 8 * (size_t)n, cudaMemcpyDeviceToHost) != cudaSuccess)
      status = cuda_fail(cudaGetLastError(), "logprobs copy");
  }
  cudaFree(dtarget);
  cudaFree(dout);
  cudaStreamDestroy(st);
  return status;
}

}  // namespace srl
