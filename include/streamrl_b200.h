/*
 * streamrl_b200.h -- C ABI of the B200-native PipelineRL hot path.
 *
 * This is the drop-in boundary for the reference streamrl toolkit
 * (/root/reference/proj, C++20).  Each entry point replaces one reference
 * interface, cited as file:line under proj/core.  Plain pointers and sizes
 * only; device pointers are marked "device".  Every function returns an
 * srl_status; the non-zero codes map 1:1 to the reference's error strings
 * and exception types.  The library fails loudly (SRL_NO_DEVICE) when no
 * CUDA device is present -- there is no CPU fallback.
 */
#ifndef STREAMRL_B200_H
#define STREAMRL_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------- status --- */
typedef enum {
  SRL_OK = 0,
  SRL_VERSION_CONFLICT = 1,  /* "version_conflict"  include/streamrl/engine.hpp:34-38, src/engine.cpp:82-87 */
  SRL_INVALID_POLICY = 2,    /* "invalid_policy"    src/engine.cpp:88-95 */
  SRL_POLICY_MISMATCH = 3,   /* "policy_mismatch"   src/engine.cpp:96-102 */
  SRL_CHECKSUM_MISMATCH = 4, /* "checksum_mismatch" src/protocol.cpp:163-172 */
  SRL_INVALID_ARGUMENT = 5,  /* std::invalid_argument */
  SRL_LOGIC_ERROR = 6,       /* std::logic_error (e.g. advance() on a running engine, engine.cpp:178) */
  SRL_UNKNOWN_STREAM = 7,    /* "unknown stream id" engine.cpp:67 */
  SRL_ESS_UNDEFINED = 8,     /* EssUndefinedError include/streamrl/rl_math.hpp:30-32 */
  SRL_CUDA_ERROR = 9,
  SRL_NO_DEVICE = 10,
  SRL_OUT_OF_MEMORY = 11,
  SRL_BUSY = 12,             /* a weight update is already staged */
  SRL_NCCL_ERROR = 13
} srl_status;

/* Reference error string for a status ("version_conflict", ...). */
const char* srl_status_string(int status);
/* Thread-local human-readable detail of the last failure in this thread. */
const char* srl_last_error(void);

/* ------------------------------------------------ kernel entry points --- */
/* Single-kernel entry points over device pointers, used by the parity tests
 * and bench.py.  `stream` is a cudaStream_t (NULL = legacy default). */

/* tcgen05 GEMM: Y = epilogue(X[M x K] . W[N x K]^T), bf16 in, fp32 accumulate.
 * epi_kind: 0 store fp32 (out = rstd*acc + bias), 1 residual (resid += acc,
 * xg = bf16(resid * gain), ssq_out partials), 2 SwiGLU (out bf16 [M x N/2]),
 * 3 store bf16.  splits <= 0 picks a split-K factor automatically. */
int srl_kernel_gemm_bf16(const void* w, const void* x, int32_t M, int32_t N, int32_t K,
                         int32_t splits, int32_t epi_kind, const void* bias,
                         const float* ssq_in, int32_t ssq_parts, float inv_dim, float eps,
                         void* out, float* resid, const void* gain, void* xg, float* ssq_out,
                         void* stream);

#ifdef __cplusplus
}
#endif
#endif /* STREAMRL_B200_H */
