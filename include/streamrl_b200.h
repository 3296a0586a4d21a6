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

/* ------------------------------------------------------- policies --- */
/* A policy checkpoint (the reference `rlmath::Policy` variant,
 * include/streamrl/policy.hpp:16-82).  Tabular and recurrent policies keep
 * the reference's fp64 semantics on the device; the decoder policy is the
 * Qwen2.5-shaped bf16 transformer this framework adds as a third variant of
 * the same "streamrl.policy/1" document schema (type "decoder"). */
typedef struct srl_policy srl_policy;

enum { SRL_POLICY_TABULAR = 0, SRL_POLICY_RECURRENT = 1, SRL_POLICY_DECODER = 2 };

/* TabularPolicy (policy.hpp:16-47).  Rows are (prompt id, context window)
 * keys; row_contexts is [n_rows x context_order], only the first
 * row_context_lens[r] entries of a row are meaningful.  default_logits may be
 * NULL (uniform fallback, policy.cpp:62-64). */
int srl_policy_tabular_create(int32_t vocab_size, int32_t context_order,
                              const double* default_logits, int32_t n_rows,
                              const char* const* row_prompt_ids, const int32_t* row_context_lens,
                              const int32_t* row_contexts, const double* row_logits,
                              srl_policy** out);
/* RecurrentToyPolicy (policy.hpp:52-72): row-major fp64 matrices
 * input_embedding [V x D], recurrence [D x D], output [D x V]. */
int srl_policy_recurrent_create(int32_t vocab_size, int32_t hidden_dim,
                                const double* input_embedding, const double* recurrence,
                                const double* output, srl_policy** out);

/* Decoder policy shape (Qwen2.5 family: RMSNorm, RoPE, GQA, SwiGLU, QKV bias). */
typedef struct {
  int32_t vocab_size;
  int32_t hidden;
  int32_t layers;
  int32_t q_heads;
  int32_t kv_heads;
  int32_t head_dim;       /* 64 or 128 */
  int32_t intermediate;
  int32_t tie_embeddings; /* LM head = embedding matrix */
  int32_t bos_token;      /* prepended to every stream's prompt */
  int32_t max_positions;  /* RoPE table length = max KV length per stream */
  double rope_theta;
  double rms_eps;
} srl_decoder_config;

/* Random-init decoder weights on `device` (counter-based SplitMix64
 * Box-Muller, scale * N(0,1); norm gains 1).  Weights live in one flat bf16
 * buffer (layout: DESIGN.md "Data layout"). */
int srl_policy_decoder_create(const srl_decoder_config* cfg, uint64_t init_seed,
                              double init_scale, int32_t device, srl_policy** out);
/* Decoder policy from an existing flat bf16 buffer (host or device), copied. */
int srl_policy_decoder_from_buffer(const srl_decoder_config* cfg, const void* weights,
                                   size_t nbytes, int32_t weights_on_device, int32_t device,
                                   srl_policy** out);
/* Size in bytes of the flat bf16 weight buffer for cfg. */
size_t srl_decoder_weight_bytes(const srl_decoder_config* cfg);
/* Device pointer + size of a decoder policy's flat weights (owned by it). */
int srl_policy_decoder_weights(const srl_policy* p, void** device_ptr, size_t* nbytes);
/* CUDA device index the decoder policy's weights live on. */
int srl_policy_decoder_device(const srl_policy* p, int32_t* device);
/* Element offset (bf16 elements) of a named tensor: "embed", "final_norm",
 * "lm_head", or "<layer>.<ln1|qkv_w|qkv_b|o_w|ln2|gate_up_w|down_w>". */
int srl_policy_decoder_offset(const srl_policy* p, const char* name, size_t* offset);
/* In-place drift w += magnitude * N(0,1) (a stand-in trainer step for
 * benchmarks; the real trainer path is srl_trainer_*). */
int srl_policy_decoder_perturb(srl_policy* p, uint64_t seed, double magnitude);
int srl_policy_type(const srl_policy* p);
int32_t srl_policy_vocab_size(const srl_policy* p);
/* validate() (policy.cpp:30-43, 71-82); SRL_INVALID_POLICY with detail. */
int srl_policy_validate(const srl_policy* p);
void srl_policy_destroy(srl_policy* p);

/* -------------------------------------------------- generator engine --- */
/* proto::Engine (include/streamrl/engine.hpp:44-109, src/engine.cpp). */
typedef struct srl_engine srl_engine;

typedef struct {
  int32_t max_streams;     /* device stream slots = constant generation batch H */
  int32_t max_seq_len;     /* KV capacity per stream (bos + prompt + generated) */
  int32_t greedy;          /* 1: argmax decoding (lowest index on ties) */
  int32_t rounds_per_sync; /* free-running rounds launched per host sync (>= 1) */
  int32_t use_graphs;      /* capture decode rounds in CUDA graphs */
  int32_t device;
  int32_t event_ring;      /* device event ring depth in rounds (>= rounds_per_sync) */
  int32_t prefill_budget;  /* max prompt tokens prefilled per round */
  int32_t precise;         /* decoder: 1 = activations between the GEMMs as bf16 hi + lo pairs
                              (only q / k / v and the K/V cache bf16; the multi-kernel round) --
                              log-probs within 1e-3 of the fp64 oracle at every shape */
} srl_engine_options;

/* TokenEvent (engine.hpp:22-28); stream id "s<N>" is numeric N here. */
typedef struct {
  int64_t stream;
  int32_t position;
  int32_t token;
  double logprob;
  int32_t weight_version;
  int32_t reserved;
} srl_token_event;

/* FinishReason (engine.hpp:30) */
enum { SRL_FINISH_RUNNING = 0, SRL_FINISH_LENGTH = 1, SRL_FINISH_TERMINATOR = 2,
       SRL_FINISH_SHUTDOWN = 3 };

/* Engine(Options{policy, recompute_state, start_paused}) (engine.cpp:38-42).
 * The engine copies the policy; opts may be NULL for defaults. */
int srl_engine_create(const srl_policy* policy, int32_t recompute_state, int32_t start_paused,
                      const srl_engine_options* opts, srl_engine** out);
void srl_engine_destroy(srl_engine* e);
/* open_stream (engine.cpp:46-61): prompt tokens are used by decoder policies
 * (bos is prepended); SRL_INVALID_ARGUMENT if max_tokens < 1. */
int srl_engine_open_stream(srl_engine* e, const char* prompt_id, int32_t max_tokens,
                           uint64_t seed, int32_t terminator_token, const int32_t* prompt_tokens,
                           int32_t n_prompt, int64_t* stream_out);
/* wait_events (engine.cpp:63-77): blocks until >= 1 event or finish, drains
 * up to cap events; *more = the reference's return value. */
int srl_engine_wait_events(srl_engine* e, int64_t stream, srl_token_event* buf, int32_t cap,
                           int32_t* n_out, int32_t* finish_reason, int32_t* more);
/* One wait_events per listed stream in one call (the actor's per-step drain):
 * stream i's events follow stream i-1's in buf, counts[i] of them (cap shared;
 * a stream whose events do not fit gets more[i] = 1 and keeps the rest). */
int srl_engine_wait_events_many(srl_engine* e, const int64_t* streams, int32_t n_streams,
                                srl_token_event* buf, int32_t cap, int32_t* counts,
                                int32_t* finish_reasons, int32_t* more);
/* The same without blocking: each stream returns whatever is queued (possibly
 * nothing; more = 1 while it is running) -- an actor polling a paused
 * engine whose streams may not have emitted yet. */
int srl_engine_poll_events_many(srl_engine* e, const int64_t* streams, int32_t n_streams,
                                srl_token_event* buf, int32_t cap, int32_t* counts,
                                int32_t* finish_reasons, int32_t* more);
/* apply_weight_update (engine.cpp:79-117).  Returns SRL_VERSION_CONFLICT /
 * SRL_INVALID_POLICY / SRL_POLICY_MISMATCH without side effects. */
int srl_engine_apply_weight_update(srl_engine* e, int32_t new_version, const srl_policy* policy,
                                   int32_t* version_out);
/* Device-resident update path (decoder): stage new_version, get the standby
 * weight buffer to receive the broadcast into, then commit (pointer swap at
 * the next token boundary) or abort.  pause_ms = time the decode stream was
 * blocked by the swap. */
int srl_engine_begin_weight_update(srl_engine* e, int32_t new_version, void** standby_device_ptr,
                                   size_t* nbytes);
int srl_engine_commit_weight_update(srl_engine* e, int32_t new_version, int32_t* version_out,
                                    double* pause_ms);
int srl_engine_abort_weight_update(srl_engine* e);
/* Size of the weight payload an update of this engine carries (the standby
 * buffer's size), without staging anything. */
int srl_engine_standby_bytes(srl_engine* e, size_t* nbytes);
/* advance (engine.cpp:174-187): paused engines only (SRL_LOGIC_ERROR). */
int srl_engine_advance(srl_engine* e, int32_t rounds, int64_t* emitted);
int srl_engine_pause(srl_engine* e);
int srl_engine_resume(srl_engine* e);
int srl_engine_weight_version(const srl_engine* e, int32_t* out);
int srl_engine_active_streams(const srl_engine* e, int32_t* out);
int srl_engine_total_streams(const srl_engine* e, int64_t* out);
int srl_engine_rounds_done(const srl_engine* e, int64_t* out);
int srl_engine_recompute_state_mode(const srl_engine* e, int32_t* out);
int srl_engine_set_process_group(srl_engine* e, const char* group_id, const char* const* members,
                                 int32_t n_members);
/* *has_group = 0 when no group is set (std::optional empty). */
int srl_engine_process_group_id(const srl_engine* e, char* buf, size_t cap, int32_t* has_group);
int srl_engine_stop(srl_engine* e);
/* Token history of a stream as fed to the KV cache (bos, prompt, generated). */
int srl_engine_stream_tokens(srl_engine* e, int64_t stream, int32_t* buf, int32_t cap,
                             int32_t* n_out);
/* Counters since creation: rounds, tokens, device decode ms, swap pause ms. */
typedef struct {
  int64_t rounds;
  int64_t tokens;
  int64_t updates;
  double decode_ms;      /* device time of all rounds (CUDA events on the engine stream) */
  double last_pause_ms;
  double max_pause_ms;
  int64_t launches;      /* kernels launched by the engine (graph nodes counted) */
  int64_t prefill_rounds; /* rounds that prefilled newly opened streams */
  int64_t prefill_rows;   /* token rows those rounds ran (prompts + running decode rows) */
  double prefill_ms;      /* their device time (CUDA events), included in decode_ms */
} srl_engine_stats;
int srl_engine_stats_get(const srl_engine* e, srl_engine_stats* out);

/* Per-kernel-class device time of one decode round, recorded with CUDA events
 * around every launch of the round after srl_engine_profile_next_round()
 * (the round runs eagerly instead of from its CUDA graph; it is a real round
 * and emits events).  Classes: 0 plan, 1 embed, 2 qkv_gemm, 3 rope_kv_append,
 * 4 attention, 5 o_gemm, 6 gate_up_gemm, 7 down_gemm, 8 lm_head_gemm,
 * 9 sample. */
enum { SRL_KERNEL_CLASSES = 10 };
typedef struct {
  double ms[SRL_KERNEL_CLASSES];
  int32_t launches[SRL_KERNEL_CLASSES];
  int32_t valid;
  int32_t rows;
  /* 1 when the round ran as the persistent megakernel: ms[] then holds the
   * grid-wide phase durations (globaltimer stamps) per class and fused_ms the
   * CUDA-event time of the one launch. */
  int32_t fused;
  double fused_ms;
} srl_kernel_profile;
int srl_engine_profile_next_round(srl_engine* e);
int srl_engine_kernel_profile(const srl_engine* e, srl_kernel_profile* out);

/* ------------------------------------------------------ trainer math --- */
/* rlmath free functions (include/streamrl/rl_math.hpp:20-121). */

/* policy_logprobs (rl_math.cpp:128-142), computed on the device. */
int srl_policy_logprobs(const srl_policy* p, const char* prompt_id, const int32_t* tokens,
                        int32_t n, double* out);
/* truncated_is_weight (rl_math.cpp:144-150). */
int srl_truncated_is_weight(double pi_logprob_sum, double mu_logprob_sum, double clamp,
                            double* out);
/* ess (rl_math.cpp:152-163): SRL_ESS_UNDEFINED when all weights are zero. */
int srl_ess(const double* weights, int32_t n, double* out);
/* is_reinforce_gradient / reinforce_gradient for a TabularPolicy
 * (rl_math.cpp:211-276, GradientTable rl_math.hpp:39-46) on the device.
 * Trajectories packed: tokens[offsets[n_traj]], prompt_ids[n_traj],
 * behavior_logprobs packed like tokens, rewards[n_traj]; baseline packed like
 * tokens (b(prompt, t) -- the caller's BaselineTable::at lookups, which throw
 * on a missing cell in the reference).  use_is = 0: reinforce_gradient (clamp
 * and granularity ignored); granularity 0 = Sequence, 1 = PerToken.
 * Output: grad_rows [(n_rows + 1) x V] -- the policy's rows in ContextKey
 * order (std::map order, as srl_policy_tabular_create stores them), then the
 * default row -- and row_touched[n_rows + 1]: 1 where the
 * reference would have created the row (a non-zero contribution landed). */
int srl_tabular_is_reinforce_gradient(const srl_policy* p, int32_t n_traj, const char* const* prompt_ids,
                                      const int32_t* tokens, const int64_t* offsets,
                                      const double* behavior_logprobs, const double* rewards,
                                      const double* baseline, int32_t use_is, double clamp,
                                      int32_t granularity, double* grad_rows, int32_t* row_touched);


/* kl_per_position (rl_math.cpp:336-372) for the decoder policy, on the device:
 * mean exact KL(behaviour || target) per position over teacher-forced
 * prefixes (packed tokens[offsets[n_prefix]]).  Behaviour = the checkpoint
 * chain switching at switch_points (MixedPolicySchedule::switch_points,
 * rl_math.cpp:286-310; n_switch = 0 for a single policy), its KV cache stale
 * across a switch (PipelineRL) or rebuilt under the new checkpoint
 * (recompute_state = 1), as the engine serves it.  kl_out[cap] receives
 * max prefix length values. */
int srl_decoder_kl_per_position(const srl_policy* const* checkpoints, int32_t n_checkpoints,
                                const int32_t* switch_points, int32_t n_switch, int32_t recompute_state,
                                const srl_policy* target, const int32_t* tokens, const int64_t* offsets,
                                int32_t n_prefix, double* kl_out, int32_t cap);

/* ------------------------------------------------ decoder trainer step --- */
/* IS-REINFORCE for the decoder policy: the reference's
 * is_reinforce_gradient (rl_math.cpp:211-276) generalised from tabular logits
 * to every decoder parameter.  Gradient = ascent direction of
 * J = (1/m) sum_traj sum_t w * A_t * log pi(y_t), stop-gradient on the
 * truncated IS weight w (sequence level by default, or per token). */
typedef struct srl_trainer srl_trainer;
typedef struct {
  int32_t max_tokens;  /* packed rows per step (sum of sequence lengths - 1) */
  int32_t device;      /* the trainer's device (weights are peer-copied there); < 0 = the policy's */
  int32_t fast_bf16;   /* 0 (default): precise -- activations and backward operands carried as
                          bf16 hi + lo pairs (fp32-class, the 1e-3 parity bar); 1: single bf16
                          operands (faster, ~1e-2 gradient agreement) */
  int32_t logit_chunk; /* LM-head rows per pass (0 = 16384) */
} srl_trainer_options;
typedef struct {
  double objective;    /* J at the current weights */
  double ess;          /* ESS of the IS weights used (rl_math.cpp:152-163) */
  int32_t clamped;     /* weights truncated at c */
  int32_t tokens;      /* rows processed */
  double forward_ms;   /* device time: forward + log-prob recompute */
  double step_ms;      /* device time: whole step incl. backward */
} srl_trainer_stats;
int srl_trainer_create(const srl_policy* decoder_policy, const srl_trainer_options* opts,
                       srl_trainer** out);
void srl_trainer_destroy(srl_trainer* t);
/* tokens: packed sequences (bos + prompt + generated), offsets[n_seq + 1];
 * loss_begin[q]: index (within the sequence) of the first scored token, >= 1;
 * behavior_logprobs / advantages: one per token, same packing (entries before
 * loss_begin ignored); n_trajectories: m.  logprobs_out (optional, packed like
 * tokens): log pi of every token under the current weights (0 at index 0). */
int srl_trainer_step(srl_trainer* t, const int32_t* tokens, const int64_t* offsets, int32_t n_seq,
                     const int32_t* loss_begin, const double* behavior_logprobs,
                     const double* advantages, int32_t n_trajectories, double clamp,
                     int32_t granularity, double* logprobs_out, srl_trainer_stats* stats);
/* fp32 gradient buffer (device, same element layout as the flat weights). */
int srl_trainer_gradient(srl_trainer* t, void** device_ptr, size_t* n_elems);
/* Adam ascent step on fp32 master weights; refreshes the bf16 weights. */
int srl_trainer_apply_adam(srl_trainer* t, double lr, double beta1, double beta2, double eps);
/* bf16 flat weights (device) -- the payload broadcast to the generators. */
int srl_trainer_weights(srl_trainer* t, void** device_ptr, size_t* nbytes);

/* ------------------------------------------------------- comm (NCCL) --- */
/* The weight-transfer channel and the trainer's gradient all-reduce over
 * NCCL on NVLink / NVSwitch, drivable from C++ (csrc/comm.cpp).  Replaces the
 * reference's group weight push -- init_process_group (protocol.cpp:378-395,
 * engine.cpp:276-291) and request_group_weight_update (protocol.cpp:397-406:
 * the policy JSON POSTed to each member in turn) -- with one broadcast of the
 * flat bf16 buffer from the trainer root into every generator's standby
 * buffer, overlapped with decode, then the swap at a token boundary.
 * NCCL is loaded at run time; without it every call returns SRL_NCCL_ERROR.
 * A generator/trainer partition uses two communicators: the trainer group
 * (gradient all-reduce) and the broadcast group (trainer root + generators),
 * each from its own unique id (srl_comm_unique_id on the group's first rank,
 * distributed out of band). */
typedef struct srl_comm srl_comm;
int srl_comm_unique_id(uint8_t* id_out /* 128 bytes */);
int srl_comm_init(const uint8_t* id, int32_t world, int32_t rank, int32_t device, srl_comm** out);
void srl_comm_destroy(srl_comm* c);
int srl_comm_size(const srl_comm* c, int32_t* world, int32_t* rank);
/* In-place broadcast of a device buffer from root (synchronous). */
int srl_comm_broadcast_bytes(srl_comm* c, int32_t root, void* device_buf, size_t nbytes);
/* Root: broadcast the trainer's bf16 weights (ordered after its queued work;
 * its next Adam step waits for the send).  Asynchronous: srl_comm_wait. */
int srl_comm_send_weights(srl_comm* c, srl_trainer* t);
/* Generator: stage new_version and enqueue the receive into the engine's
 * standby buffer on the transfer stream; returns at once (decode continues).
 * *staged = 0 when the engine rejected the version (version_conflict): the
 * rank still receives (into scratch) so the collective completes on every
 * rank, and keeps serving at its old version. */
int srl_comm_recv_weights_begin(srl_comm* c, int32_t root, srl_engine* e, int32_t new_version,
                                int32_t* staged);
/* Generator: wait for the transfer, then commit (swap at the next token
 * boundary).  transfer_ms = device time of the broadcast; pause_ms = time
 * the decode loop was blocked by the swap. */
int srl_comm_recv_weights_finish(srl_comm* c, srl_engine* e, int32_t new_version, int32_t* applied,
                                 int32_t* version_out, double* transfer_ms, double* pause_ms);
/* Wait for the in-flight broadcast (root side); transfer_ms as above. */
int srl_comm_wait(srl_comm* c, double* transfer_ms);
/* Trainer group: in-place SUM of the fp32 gradient, on the trainer's stream
 * between its backward and its Adam step. */
int srl_comm_allreduce_gradient(srl_comm* c, srl_trainer* t);

/* ---------------------------------------------------------------- lag --- */
/* Per consumed batch lag statistics on the device (sim.cpp:63-110):
 * lag = version_before - token_version; hist must hold hist_cap counters.
 * versions are packed per sequence (device pointers); seq_offsets has
 * n_seq + 1 entries.  totals = {tokens, lag_sum, max_lag}. */
int srl_lag_stats(const int32_t* versions, const int64_t* seq_offsets, int32_t n_seq,
                  int32_t version_before, int64_t* hist, int32_t hist_cap, int64_t* seq_lag_sums,
                  int64_t* totals, void* stream);

/* --------------------------------------------------------- protocol --- */
/* crc32 (engine.cpp:257-274) and process_group_id (engine.cpp:276-291). */
uint32_t srl_crc32(const void* bytes, size_t n);
int srl_process_group_id(const char* const* members, int32_t n_members, char* buf, size_t cap);

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

/* tcgen05 GEMM with an MN-major W operand (the trainer's weight gradients
 * and input gradients without transposes): out[m, n] (+)= scale * sum_k
 * X(m, k) w[k, n]; w is [k_rows x N] row-major bf16; X is x[k, m] ([k_rows x
 * M], x_kmajor = 0) or x[m, k] ([M x k_rows], x_kmajor = 1, k_rows % 64 == 0).
 * K = k_rows rounded up to 64 (rows past k_rows read as zero).  accumulate
 * != 0 adds into out (fp32 [M x N]); splits <= 0 plans the K slicing, which
 * stays deterministic (ordered slices). */
int srl_kernel_gemm_mn(const void* w, const void* x, int32_t M, int32_t N, int32_t k_rows,
                       int32_t x_kmajor, int32_t splits, int32_t accumulate, float scale, float* out,
                       void* stream);

/* The decode sampler on raw fp32 logits rows (device pointers): row r uses
 * draw #draw_index[r] of SplitMix64(seeds[r]) (rng.hpp:18-28) and the
 * inverse CDF of exp(log_softmax) in fp64 (rng.hpp:61-69, engine.cpp:130-138);
 * greedy = argmax, lowest index on ties.  Writes token and log-prob. */
/* Single-query paged GQA attention of the multi-kernel round (decoder.cu
 * attention_kernel): q [rows x nq x hd], caches [pages][nkv][64][hd] (bf16),
 * block_table [slots x pages_per_seq], keys 0..row_pos[r] of slot row_slot[r];
 * out [rows x nq x hd] bf16.  hd 64 or 128. */
int srl_kernel_attention_decode(const void* q, const void* kc, const void* vc, const int32_t* block_table,
                                int32_t pages_per_seq, const int32_t* row_slot, const int32_t* row_pos,
                                int32_t rows, int32_t nq, int32_t nkv, int32_t hd, int32_t max_ctx, void* out,
                                void* stream);
/* Causal paged GQA attention over packed query segments (train_attn.cu
 * attn_fwd_mma: the trainer's forward, a prefill round's prompt rows).
 * Segment y: query rows seq_start[y] .. + seq_len[y] of q [T x nq x hd] at
 * positions seg_pos0[y] .. (0 when null) of slot seg_slot[y] (y when null),
 * attending to keys 0 .. its position from the slot's pages (caches
 * [pages][nkv][64][hd] bf16, block_table [slots x pages_per_seq]); max_rows
 * >= every seq_len.  out [T x (nq hd + out_lo)] bf16 (out_lo > 0: the
 * rounding residual at + out_lo), lse [T x nq] (natural log of the scaled
 * scores' partition sum; may be null).  hd 64 or 128. */
int srl_kernel_attention_prefill(const void* q, const void* kc, const void* vc, const int32_t* block_table,
                                 int32_t pages_per_seq, const int32_t* seq_start, const int32_t* seq_len,
                                 const int32_t* seg_pos0, const int32_t* seg_slot, int32_t n_seg,
                                 int32_t max_rows, int32_t nq, int32_t nkv, int32_t hd, void* out, float* lse,
                                 int32_t out_lo, void* stream);
/* Device-to-device cudaMemcpyAsync on the given stream, e.g. a one-GPU
 * update into the standby buffer on a side stream while decode runs. */
int srl_device_copy_async(void* dst, const void* src, size_t nbytes, void* stream);
int srl_kernel_sample_logits(const float* logits, int32_t vocab, int32_t rows,
                             const uint64_t* seeds, const int32_t* draw_index, int32_t greedy,
                             int32_t* tokens_out, double* logprobs_out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* STREAMRL_B200_H */
