/*
 * streamrl_oracle.c -- CPU restatement of the reference streamrl hot-path
 * algorithms.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker: it is linked
 * by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg, and by
 * nothing in the product path (paper_2509_19128_b200/ never loads it).
 *
 * Every function restates one reference routine in plain C with fp64
 * arithmetic in the same operation order as the reference (sequential sums,
 * no FMA contraction: build with -ffp-contract=off), so that on x86-64 its
 * results are bit-identical to the reference build under oracle/_ref.
 * References are to /root/reference/proj (read-only, not vendored).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_EINVAL 1
#define ORC_EUNDEFINED 2

/* ------------------------------------------------------------------ rng --- */

/* SplitMix64 step -- core/include/streamrl/rng.hpp:18-23 */
uint64_t orc_splitmix_next(uint64_t *state) {
  uint64_t z = (*state += 0x9E3779B97F4A7C15ULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

/* 53-bit uniform in [0,1) -- rng.hpp:26-28 */
double orc_next_double(uint64_t *state) {
  return (double)(orc_splitmix_next(state) >> 11) * 0x1.0p-53;
}

/* Box-Muller normal, two uniforms per draw -- rng.hpp:39-43 */
double orc_next_gaussian(uint64_t *state) {
  const double u1 = 1.0 - orc_next_double(state);
  const double u2 = orc_next_double(state);
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586476925286766559 * u2);
}

/* Substream seed -- rng.hpp:54-57 */
uint64_t orc_derive_stream(uint64_t seed, uint64_t index) {
  uint64_t s = seed ^ (0x9E3779B97F4A7C15ULL * (index + 1));
  return orc_splitmix_next(&s);
}

/* Inverse-CDF draw with fallback to the last index -- rng.hpp:61-69 */
int orc_sample_categorical(uint64_t *state, const double *probs, int n) {
  const double u = orc_next_double(state);
  double cum = 0.0;
  for (int k = 0; k < n; ++k) {
    cum += probs[k];
    if (u < cum) return k;
  }
  return n - 1;
}

/* Same draw with the uniform supplied by the caller (used to check the GPU
 * sampler against dumped logits). */
int orc_sample_categorical_u(double u, const double *probs, int n) {
  double cum = 0.0;
  for (int k = 0; k < n; ++k) {
    cum += probs[k];
    if (u < cum) return k;
  }
  return n - 1;
}

/* -------------------------------------------------------------- numeric --- */

/* numeric.hpp:13-20 */
double orc_log_sum_exp(const double *x, int n) {
  double m = -INFINITY;
  for (int i = 0; i < n; ++i) m = x[i] > m ? x[i] : m;
  if (!isfinite(m)) return m;
  double s = 0.0;
  for (int i = 0; i < n; ++i) s += exp(x[i] - m);
  return m + log(s);
}

/* numeric.hpp:22-27 */
void orc_log_softmax(const double *x, int n, double *out) {
  const double lse = orc_log_sum_exp(x, n);
  for (int i = 0; i < n; ++i) out[i] = x[i] - lse;
}

/* Sampling step of Engine::run_round_locked (engine.cpp:130-132) applied to
 * a raw logits row: log-softmax, probs = exp(lp), inverse CDF with the
 * caller's uniform.  Writes lp[token] to *logprob.  Used by the
 * "sampler bit-exact given dumped logits" parity tests. */
int orc_sample_from_logits(const double *logits, int n, double u, double *logprob,
                           double *scratch /* 2n */) {
  double *lp = scratch, *p = scratch + n;
  orc_log_softmax(logits, n, lp);
  for (int k = 0; k < n; ++k) p[k] = exp(lp[k]);
  const int tok = orc_sample_categorical_u(u, p, n);
  *logprob = lp[tok];
  return tok;
}

/* Greedy rule (documented in DESIGN.md): argmax, lowest index on ties. */
int orc_argmax(const double *x, int n) {
  int best = 0;
  for (int k = 1; k < n; ++k)
    if (x[k] > x[best]) best = k;
  return best;
}

/* --------------------------------------------------------------- policy --- */

/* A policy checkpoint.  type 0 = TabularPolicy (policy.hpp:16-47),
 * type 1 = RecurrentToyPolicy (policy.hpp:52-72).  Tabular rows are keyed by
 * (prompt index, context window); the caller interns prompt ids to ints. */
typedef struct {
  int type;
  int vocab;
  /* recurrent */
  int hidden;
  const double *emb; /* vocab x hidden   */
  const double *rec; /* hidden x hidden  */
  const double *out; /* hidden x vocab   */
  /* tabular */
  int order;
  int n_rows;
  const int *row_prompt;    /* n_rows            */
  const int *row_ctx_len;   /* n_rows            */
  const int *row_ctx;       /* n_rows x order    */
  const double *row_logits; /* n_rows x vocab    */
  const double *default_logits; /* vocab or NULL */
} orc_policy;

/* RecurrentToyPolicy::advance_state -- policy.cpp:84-95 */
void orc_rec_advance(const orc_policy *p, double *state, int token, double *scratch) {
  const int D = p->hidden;
  for (int i = 0; i < D; ++i) {
    double acc = p->emb[(size_t)token * D + i];
    const double *w = p->rec + (size_t)i * D;
    for (int j = 0; j < D; ++j) acc += w[j] * state[j];
    scratch[i] = tanh(acc);
  }
  memcpy(state, scratch, sizeof(double) * (size_t)D);
}

/* RecurrentToyPolicy::next_token_logprobs -- policy.cpp:104-113 */
void orc_rec_next_logprobs(const orc_policy *p, const double *state, double *lp,
                           double *scratch /* vocab */) {
  const int V = p->vocab, D = p->hidden;
  for (int k = 0; k < V; ++k) scratch[k] = 0.0;
  for (int i = 0; i < D; ++i) {
    const double s = state[i];
    const double *w = p->out + (size_t)i * V;
    for (int k = 0; k < V; ++k) scratch[k] += s * w[k];
  }
  orc_log_softmax(scratch, V, lp);
}

/* TabularPolicy::context_at + find_row -- policy.cpp:44-57.  Returns the row
 * index or -1 for the default row. */
int orc_tab_find_row(const orc_policy *p, int prompt, const int *prefix, int n) {
  const int window = p->order < n ? p->order : n;
  const int *ctx = prefix + (n - window);
  for (int r = 0; r < p->n_rows; ++r) {
    if (p->row_prompt[r] != prompt || p->row_ctx_len[r] != window) continue;
    const int *rc = p->row_ctx + (size_t)r * p->order;
    int same = 1;
    for (int j = 0; j < window; ++j)
      if (rc[j] != ctx[j]) { same = 0; break; }
    if (same) return r;
  }
  return -1;
}

/* TabularPolicy::next_token_logprobs -- policy.cpp:59-69 */
void orc_tab_next_logprobs(const orc_policy *p, int prompt, const int *prefix, int n,
                           double *lp, double *scratch /* vocab */) {
  const int r = orc_tab_find_row(p, prompt, prefix, n);
  const double *row;
  if (r >= 0) {
    row = p->row_logits + (size_t)r * p->vocab;
  } else if (p->default_logits) {
    row = p->default_logits;
  } else {
    for (int k = 0; k < p->vocab; ++k) scratch[k] = 0.0;
    row = scratch;
  }
  orc_log_softmax(row, p->vocab, lp);
}

/* ------------------------------------------------------- policy walker --- */

/* PolicyWalker -- rl_math.cpp:27-82.  One sequence walked position by
 * position under a checkpoint chain with stale or recomputed state. */
typedef struct {
  const orc_policy *ckpts;
  int n_ckpt;
  const int *switch_points;
  int n_switch;
  int recompute;
  int prompt;
  int current;
  int *prefix;
  int len;
  double *state;
  double *scratch;
} orc_walker;

static int walker_segment(const orc_walker *w, int pos) {
  int g = 0;
  for (int i = 0; i < w->n_switch; ++i) {
    if (pos >= w->switch_points[i]) ++g;
    else break;
  }
  return g; /* MixedPolicySchedule::segment_at, rl_math.cpp:303-310 */
}

static void walker_state_for_prefix(const orc_policy *p, const int *prefix, int n,
                                    double *state, double *scratch) {
  for (int i = 0; i < p->hidden; ++i) state[i] = 0.0; /* initial_state, policy.hpp:62 */
  for (int t = 0; t < n; ++t) orc_rec_advance(p, state, prefix[t], scratch);
}

static void walker_next(orc_walker *w, int pos, double *lp) {
  int target = walker_segment(w, pos);
  if (target > w->n_ckpt - 1) target = w->n_ckpt - 1;
  if (target != w->current) { /* maybe_switch, rl_math.cpp:64-73 */
    w->current = target;
    if (w->recompute && w->ckpts[target].type == 1)
      walker_state_for_prefix(&w->ckpts[target], w->prefix, w->len, w->state, w->scratch);
  }
  const orc_policy *p = &w->ckpts[w->current];
  if (p->type == 0)
    orc_tab_next_logprobs(p, w->prompt, w->prefix, w->len, lp, w->scratch);
  else
    orc_rec_next_logprobs(p, w->state, lp, w->scratch);
}

static void walker_push(orc_walker *w, int token) {
  const orc_policy *p = &w->ckpts[w->current];
  if (p->type == 1) orc_rec_advance(p, w->state, token, w->scratch);
  w->prefix[w->len++] = token;
}

static int max_dim(const orc_policy *c, int n) {
  int m = 1;
  for (int i = 0; i < n; ++i) {
    if (c[i].vocab > m) m = c[i].vocab;
    if (c[i].type == 1 && c[i].hidden > m) m = c[i].hidden;
  }
  return m;
}

/* sample_with_walker -- rl_math.cpp:84-124 (mixed_policy_sample :312-319 and
 * sample_trajectories :278-284 are the n_switch / n_ckpt special cases).
 * Outputs are [count x max_len] row-major with per-trajectory lengths. */
int orc_mixed_sample(const orc_policy *ckpts, int n_ckpt, const int *switch_points, int n_switch,
                     int recompute, int prompt, int count, int max_len, uint64_t seed,
                     int terminator, int32_t *tokens, double *logprobs, int32_t *versions,
                     int32_t *lengths) {
  if (count < 1 || max_len < 1 || n_ckpt < 1) return ORC_EINVAL;
  const int V = ckpts[0].vocab;
  for (int i = 0; i < n_ckpt; ++i)
    if (ckpts[i].vocab != V) return ORC_EINVAL;
  if (n_ckpt < n_switch + 1 && n_switch > 0) return ORC_EINVAL;
  const int dim = max_dim(ckpts, n_ckpt);
  double *lp = malloc(sizeof(double) * (size_t)V);
  double *pr = malloc(sizeof(double) * (size_t)V);
  double *state = calloc((size_t)dim, sizeof(double));
  double *scratch = malloc(sizeof(double) * (size_t)dim);
  int *prefix = malloc(sizeof(int) * (size_t)max_len);
  for (int i = 0; i < count; ++i) {
    uint64_t gen = orc_derive_stream(seed, (uint64_t)i);
    orc_walker w = {ckpts, n_ckpt, switch_points, n_switch, recompute, prompt, 0,
                    prefix, 0, state, scratch};
    memset(state, 0, sizeof(double) * (size_t)dim);
    int len = 0;
    for (int t = 0; t < max_len; ++t) {
      walker_next(&w, t, lp);
      for (int k = 0; k < V; ++k) pr[k] = exp(lp[k]);
      const int tok = orc_sample_categorical(&gen, pr, V);
      tokens[(size_t)i * max_len + t] = tok;
      logprobs[(size_t)i * max_len + t] = lp[tok];
      versions[(size_t)i * max_len + t] = w.current;
      walker_push(&w, tok);
      len = t + 1;
      if (tok == terminator) break;
    }
    lengths[i] = len;
  }
  free(lp); free(pr); free(state); free(scratch); free(prefix);
  return ORC_OK;
}

/* policy_logprobs -- rl_math.cpp:128-142 */
int orc_policy_logprobs(const orc_policy *p, int prompt, const int32_t *tokens, int n,
                        double *out) {
  for (int t = 0; t < n; ++t)
    if (tokens[t] < 0 || tokens[t] >= p->vocab) return ORC_EINVAL;
  const int dim = max_dim(p, 1);
  double *lp = malloc(sizeof(double) * (size_t)p->vocab);
  double *state = calloc((size_t)dim, sizeof(double));
  double *scratch = malloc(sizeof(double) * (size_t)dim);
  int *prefix = malloc(sizeof(int) * (size_t)(n > 0 ? n : 1));
  orc_walker w = {p, 1, NULL, 0, 0, prompt, 0, prefix, 0, state, scratch};
  for (int t = 0; t < n; ++t) {
    walker_next(&w, t, lp);
    out[t] = lp[tokens[t]];
    walker_push(&w, tokens[t]);
  }
  free(lp); free(state); free(scratch); free(prefix);
  return ORC_OK;
}

/* ------------------------------------------------------- engine rounds --- */

/* Lockstep restatement of proto::Engine: open_stream (engine.cpp:46-61),
 * run_round_locked (:119-153) and apply_weight_update (:79-117).  Stream i
 * opens after open_after[i] rounds; update j (to checkpoint j+1, version
 * j+1) lands after upd_after[j] rounds.  Streams are seeded with their seed
 * directly (engine.cpp:35).  Events are written [stream x max_events]. */
int orc_engine_lockstep(const orc_policy *ckpts, int n_ckpt, const int *upd_after, int n_upd,
                        int recompute, int n_streams, const int *prompt, const uint64_t *seeds,
                        const int *max_tokens, const int *terminators, const int *open_after,
                        int total_rounds, int max_events, int32_t *ev_token, double *ev_logprob,
                        int32_t *ev_version, int32_t *ev_count, int32_t *finish) {
  if (n_ckpt < n_upd + 1) return ORC_EINVAL;
  const int V = ckpts[0].vocab;
  const int dim = max_dim(ckpts, n_ckpt);
  double *lp = malloc(sizeof(double) * (size_t)V);
  double *pr = malloc(sizeof(double) * (size_t)V);
  double *scratch = malloc(sizeof(double) * (size_t)dim);
  double *states = calloc((size_t)n_streams * (size_t)dim, sizeof(double));
  int *prefix = malloc(sizeof(int) * (size_t)n_streams * (size_t)max_events);
  uint64_t *gen = malloc(sizeof(uint64_t) * (size_t)n_streams);
  int *opened = calloc((size_t)n_streams, sizeof(int));
  int version = 0;
  for (int s = 0; s < n_streams; ++s) {
    ev_count[s] = 0;
    finish[s] = 0; /* Running */
    gen[s] = seeds[s];
  }
  int next_upd = 0;
  for (int round = 0; round <= total_rounds; ++round) {
    /* boundary "after `round` rounds": updates first in the order given,
     * then stream opens (callers order them that way). */
    while (next_upd < n_upd && upd_after[next_upd] == round) {
      version += 1;
      const orc_policy *np = &ckpts[version];
      if (recompute && np->type == 1) {
        for (int s = 0; s < n_streams; ++s)
          if (opened[s] && finish[s] == 0)
            walker_state_for_prefix(np, prefix + (size_t)s * max_events, ev_count[s],
                                    states + (size_t)s * dim, scratch);
      }
      ++next_upd;
    }
    for (int s = 0; s < n_streams; ++s)
      if (!opened[s] && open_after[s] == round) opened[s] = 1;
    if (round == total_rounds) break;
    const orc_policy *p = &ckpts[version];
    for (int s = 0; s < n_streams; ++s) {
      if (!opened[s] || finish[s] != 0) continue;
      int *pre = prefix + (size_t)s * max_events;
      double *st = states + (size_t)s * dim;
      const int n = ev_count[s];
      if (n >= max_events) return ORC_EINVAL;
      if (p->type == 0) orc_tab_next_logprobs(p, prompt[s], pre, n, lp, scratch);
      else orc_rec_next_logprobs(p, st, lp, scratch);
      for (int k = 0; k < V; ++k) pr[k] = exp(lp[k]);
      const int tok = orc_sample_categorical(&gen[s], pr, V);
      ev_token[(size_t)s * max_events + n] = tok;
      ev_logprob[(size_t)s * max_events + n] = lp[tok];
      ev_version[(size_t)s * max_events + n] = version;
      if (p->type == 1) orc_rec_advance(p, st, tok, scratch);
      pre[n] = tok;
      ev_count[s] = n + 1;
      if (tok == terminators[s]) finish[s] = 2;             /* Terminator */
      else if (n + 1 >= max_tokens[s]) finish[s] = 1;        /* Length */
    }
  }
  free(lp); free(pr); free(scratch); free(states); free(prefix); free(gen); free(opened);
  return ORC_OK;
}

/* ----------------------------------------------------------- trainer math --- */

/* truncated_is_weight -- rl_math.cpp:144-150 */
int orc_truncated_is_weight(double pi_sum, double mu_sum, double clamp, double *out) {
  if (clamp <= 0.0 || !isfinite(clamp)) return ORC_EINVAL;
  if (!isfinite(pi_sum) || !isfinite(mu_sum)) return ORC_EINVAL;
  const double r = exp(pi_sum - mu_sum);
  *out = r < clamp ? r : clamp;
  return ORC_OK;
}

/* ess -- rl_math.cpp:152-163 */
int orc_ess(const double *w, int n, double *out) {
  if (n < 1) return ORC_EINVAL;
  double sum = 0.0, sq = 0.0;
  for (int i = 0; i < n; ++i) {
    if (!isfinite(w[i]) || w[i] < 0.0) return ORC_EINVAL;
    sum += w[i];
    sq += w[i] * w[i];
  }
  if (sq == 0.0) return ORC_EUNDEFINED;
  *out = (sum * sum) / ((double)n * sq);
  return ORC_OK;
}

/* fit_baseline -- rl_math.cpp:165-179.  Dense table [n_prompt x max_len];
 * count[c] == 0 marks a missing cell (BaselineTable::at throws). */
int orc_fit_baseline(int n_traj, const int *prompt, const int32_t *lengths,
                     const double *reward, int n_prompt, int max_len, double *table,
                     int64_t *count) {
  if (n_traj < 1) return ORC_EINVAL;
  const size_t cells = (size_t)n_prompt * (size_t)max_len;
  double *sum = calloc(cells, sizeof(double));
  for (size_t c = 0; c < cells; ++c) count[c] = 0;
  /* the reference accumulates per cell in trajectory order */
  for (int j = 0; j < n_traj; ++j)
    for (int t = 0; t < lengths[j]; ++t) {
      const size_t c = (size_t)prompt[j] * max_len + t;
      sum[c] += reward[j];
      count[c] += 1;
    }
  for (size_t c = 0; c < cells; ++c) table[c] = count[c] ? sum[c] / (double)count[c] : 0.0;
  free(sum);
  return ORC_OK;
}

/* weighted_reinforce_gradient for a tabular policy -- rl_math.cpp:211-260.
 * Trajectories are packed: tokens/behavior_lp at offsets[j]..offsets[j]+len.
 * grad is dense [(n_rows + 1) x vocab]: row r for policy row r, the last row
 * for the default row.  touched[r] marks rows the reference would create.
 * use_is = 0 reproduces reinforce_gradient (:264-269). granularity 0 =
 * Sequence, 1 = PerToken (rl_math.hpp:52). */
int orc_reinforce_gradient_tab(const orc_policy *p, int n_traj, const int *prompt,
                               const int32_t *lengths, const int64_t *offsets,
                               const int32_t *tokens, const double *behavior_lp,
                               const double *reward, const double *baseline, const int64_t *bcount,
                               int baseline_max_len, double clamp, int use_is, int granularity,
                               double *grad, int *touched) {
  if (n_traj < 1 || p->type != 0) return ORC_EINVAL;
  const int V = p->vocab;
  const double inv_m = 1.0 / (double)n_traj;
  memset(grad, 0, sizeof(double) * (size_t)(p->n_rows + 1) * V);
  memset(touched, 0, sizeof(int) * (size_t)(p->n_rows + 1));
  int max_n = 1;
  for (int j = 0; j < n_traj; ++j) max_n = lengths[j] > max_n ? lengths[j] : max_n;
  double *lps = malloc(sizeof(double) * (size_t)max_n);
  double *probs = malloc(sizeof(double) * (size_t)V);
  double *lsm = malloc(sizeof(double) * (size_t)V);
  int status = ORC_OK;
  for (int j = 0; j < n_traj && status == ORC_OK; ++j) {
    const int32_t *tk = tokens + offsets[j];
    const double *mu = behavior_lp + offsets[j];
    const int n = lengths[j];
    if (orc_policy_logprobs(p, prompt[j], tk, n, lps) != ORC_OK) { status = ORC_EINVAL; break; }
    double seq_w = 1.0;
    if (use_is && granularity == 0) {
      double pi_sum = 0.0, mu_sum = 0.0;
      for (int t = 0; t < n; ++t) pi_sum += lps[t];
      for (int t = 0; t < n; ++t) mu_sum += mu[t];
      if (orc_truncated_is_weight(pi_sum, mu_sum, clamp, &seq_w) != ORC_OK) { status = ORC_EINVAL; break; }
    }
    for (int t = 0; t < n; ++t) {
      if (t >= baseline_max_len || bcount[(size_t)prompt[j] * baseline_max_len + t] == 0) {
        status = ORC_EINVAL; /* BaselineTable::at missing cell, trajectory.cpp:35-41 */
        break;
      }
      const double adv = reward[j] - baseline[(size_t)prompt[j] * baseline_max_len + t];
      double w = seq_w;
      if (use_is && granularity == 1)
        if (orc_truncated_is_weight(lps[t], mu[t], clamp, &w) != ORC_OK) { status = ORC_EINVAL; break; }
      const double scale = inv_m * w * adv;
      if (scale == 0.0) continue;
      const int r = orc_tab_find_row(p, prompt[j], tk, t);
      const double *row;
      int target;
      if (r >= 0) {
        row = p->row_logits + (size_t)r * V;
        target = r;
        orc_log_softmax(row, V, lsm);
        for (int k = 0; k < V; ++k) probs[k] = exp(lsm[k]);
      } else {
        target = p->n_rows;
        if (p->default_logits) {
          orc_log_softmax(p->default_logits, V, lsm);
          for (int k = 0; k < V; ++k) probs[k] = exp(lsm[k]);
        } else {
          for (int k = 0; k < V; ++k) probs[k] = 1.0 / V;
        }
      }
      touched[target] = 1;
      double *g = grad + (size_t)target * V;
      for (int k = 0; k < V; ++k) {
        const double ind = (k == tk[t]) ? 1.0 : 0.0;
        g[k] += scale * (ind - probs[k]);
      }
    }
  }
  free(lps); free(probs); free(lsm);
  return status;
}

/* ------------------------------------------------------------------- lag --- */

/* Per consumed batch lag statistics: make_step_record (sim.cpp:63-87),
 * batch_ess (:49-60, clamp 5), fill_sample_lags (:89-104) and
 * batch_post_warmup (:106-110).  Versions are packed per sequence.
 * consumed_at_emit may be NULL (sample lags then left at zero).  hist must
 * hold hist_cap counters indexed by lag (lag >= 0 assumed; a negative or
 * too-large lag returns ORC_EINVAL). */
int orc_lag_stats(int version_before, int n_seq, const int32_t *lengths,
                  const int32_t *versions, const int64_t *consumed_at_emit,
                  int64_t consumed_before, double drift_magnitude, int64_t *hist, int hist_cap,
                  int64_t *tokens_out, int64_t *max_lag, double *mean_lag,
                  int64_t *seq_lag_sums, double *ess_out, int64_t *max_lag_samples,
                  double *mean_lag_samples, int *post_warmup) {
  for (int i = 0; i < hist_cap; ++i) hist[i] = 0;
  int64_t tokens = 0, lag_sum = 0, mx = 0;
  size_t off = 0;
  int warm = 1;
  for (int s = 0; s < n_seq; ++s) {
    int64_t seq_sum = 0;
    for (int t = 0; t < lengths[s]; ++t) {
      const int64_t lag = (int64_t)version_before - versions[off + t];
      if (lag < 0 || lag >= hist_cap) return ORC_EINVAL;
      hist[lag] += 1;
      if (lag > mx) mx = lag;
      lag_sum += lag;
      seq_sum += lag;
    }
    if (lengths[s] == 0 || versions[off] < 1) warm = 0;
    tokens += lengths[s];
    seq_lag_sums[s] = seq_sum;
    off += (size_t)lengths[s];
  }
  *tokens_out = tokens;
  *max_lag = mx;
  *mean_lag = tokens > 0 ? (double)lag_sum / (double)tokens : 0.0;
  *post_warmup = warm;
  /* batch_ess */
  if (n_seq <= 0) {
    *ess_out = 1.0;
  } else {
    double *w = malloc(sizeof(double) * (size_t)n_seq);
    for (int s = 0; s < n_seq; ++s) {
      const double e = exp(-drift_magnitude * (double)seq_lag_sums[s]);
      w[s] = e < 5.0 ? e : 5.0;
    }
    double v = 0.0;
    const int st = orc_ess(w, n_seq, &v);
    *ess_out = st == ORC_OK ? v : 0.0;
    free(w);
  }
  /* fill_sample_lags */
  int64_t smax = 0, ssum = 0, scount = 0;
  if (consumed_at_emit) {
    int64_t index = consumed_before;
    off = 0;
    for (int s = 0; s < n_seq; ++s) {
      for (int t = 0; t < lengths[s]; ++t) {
        const int64_t lag = index - consumed_at_emit[off + t];
        if (lag > smax) smax = lag;
        ssum += lag;
        ++scount;
      }
      off += (size_t)lengths[s];
      ++index;
    }
  }
  *max_lag_samples = smax;
  *mean_lag_samples = scount > 0 ? (double)ssum / (double)scount : 0.0;
  return ORC_OK;
}

/* pipeline_max_lag_steps -- throughput.cpp:260-269 restated:
 * g_max = ceil(H * I * L / (mean_len * B)). */
int64_t orc_pipeline_max_lag_steps(double gen_batch, double inference_units, double max_len,
                                   double mean_len, double train_batch) {
  return (int64_t)ceil(gen_batch * inference_units * max_len / (mean_len * train_batch));
}

/* ------------------------------------------------------------ protocol --- */

/* crc32 (IEEE, reflected 0xEDB88320) -- engine.cpp:257-274 */
uint32_t orc_crc32(const unsigned char *bytes, size_t n) {
  uint32_t table[256];
  for (uint32_t i = 0; i < 256; ++i) {
    uint32_t c = i;
    for (int k = 0; k < 8; ++k) c = (c & 1) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
    table[i] = c;
  }
  uint32_t c = 0xFFFFFFFFu;
  for (size_t i = 0; i < n; ++i) c = table[(c ^ bytes[i]) & 0xFFu] ^ (c >> 8);
  return c ^ 0xFFFFFFFFu;
}

/* MixedPolicySchedule::make -- rl_math.cpp:286-301.  Returns the number of
 * switch points written (<= max_lag), or -1 on invalid input. */
int orc_schedule_make(int max_len, int max_lag, int *switch_points) {
  if (max_len < 1 || max_lag < 1) return -1;
  const int first = (2 * max_len) / max_lag, step = max_len / max_lag;
  int n = 0;
  for (int t = first; t < max_len && n < max_lag;) {
    switch_points[n++] = t;
    if (step == 0) break;
    t += step;
  }
  return n;
}
