// decode_mk.cuh -- the persistent decode-round megakernel (one CTA per SM).
//
// A decode round is a fixed sequence of phases: [plan+embed] then per layer
// [QKV GEMM, attention, O GEMM, gate/up GEMM, down GEMM], then [LM head,
// sample].  Instead of ~150 dependent kernel launches, one cooperative launch
// runs every phase; phases are separated by grid-wide arrival counters
// (monotonic across rounds, target = (epoch + 1) * gridDim.x).  Each CTA is
// warp-specialised:
//   warp 0   TMA producer: weight tiles of its next GEMM item are issued as
//            soon as ring slots free up -- across phase boundaries -- and only
//            the activation tiles wait for the previous phase's counter;
//   warp 1   tcgen05.mma issuer, double-buffered TMEM accumulators;
//   warps 4-7 compute: TMEM drain + fused epilogues, attention, embedding,
//            sampling (named barrier 1, 128 threads).
// Split-K tiles are reduced by the last-arriving split (L2 partials, split
// order: deterministic).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "decoder.cuh"

namespace srl {

constexpr int kMkAttnChunk = 4096;  // keys per attention item (longer contexts split)
constexpr int kMkMaxAttnItems = 4096;  // items of one attention phase (the order's scratch)

enum MkKind : int { MK_EMBED = 0, MK_QKV = 1, MK_ATTN = 2, MK_O = 3, MK_GU = 4, MK_DOWN = 5,
                    MK_LM = 6, MK_SAMPLE = 7 };

struct MkPhase {
  int kind;
  int layer;
  int n_items;  // work items (GEMM: n_tiles * cs)
  int cs;       // split-K factor (GEMM); ATTN: the QKV phase's split-K factor
  int N, K;     // GEMM shape
  int wmap;     // weight tensor-map index
  int xmap;     // activation tensor-map index: 0 xg, 1 attn, 2 act
  int ctr_base; // first split-K counter of this phase
  int rot;      // item -> CTA rotation
  long long colv;  // O / DOWN: offset of the next RMSNorm gain (epilogue column constant);
                   // ATTN: offset of the layer's qkv bias; else -1
  // Dataflow dependency (QKV after DOWN, DOWN after gate/up): instead of the
  // grid barrier, the producer waits per k-block for the producing tile's
  // done counter tile_ctr[flow_ctr + (kb * 64) / flow_cols] to reach
  // flow_target per round; -1: grid barrier.
  int flow_ctr, flow_cols, flow_target;
  int done_ctr;  // this phase's items signal tile_ctr[done_ctr + tile] after their epilogue (-1: no)
};

struct MkLayer {
  size_t ln1, qkv_b, ln2;
};

struct MkParams {
  int S, H, I, V, L, nq, nkv, hd, qkv, parts, pps, attn_splits, attn_chunk, greedy;
  float eps, inv_h, scale;
  const __nv_bfloat16* w;       // flat weights (active buffer)
  const CUtensorMap* wmaps;     // [4 * L + 1]: per layer qkv, o, gate_up, down; then lm_head
  const CUtensorMap* xmaps;     // [3]: xg, attn, act (box 64 rows)
  const MkLayer* layers;        // [L]
  size_t off_embed, off_final_norm;
  float* x;
  __nv_bfloat16* xg;
  float* ssq;
  __nv_bfloat16* q;
  __nv_bfloat16* attn;
  __nv_bfloat16* act;
  float* logits;
  float* lse_max;
  double* lse_sum;
  __nv_bfloat16 *kc, *vc;
  size_t kv_layer_elems;
  const int32_t* block_table;
  const float* cos_sin;
  RoundPlan plan, next;
  SlotState ss;
  EventRing ring;
  int32_t* round_ctr;
  const int32_t* version;
  unsigned* phase_done;         // [n_phases][8] monotonic arrival counters
  unsigned* epoch;              // rounds completed by this kernel (device scalar)
  unsigned* tile_ctr;           // split-K / split-KV arrival counters (monotonic)
  int32_t* attn_order;          // this round's attention items, longest first (built in the embed phase)
  float* ws;                    // split-K and split-KV partials
  float* qkv_part;              // QKV split partials [S][nkv][cs][(G+2) hd] (reduced by attention)
  const MkPhase* phases;
  int n_phases;
  unsigned long long* stamps;   // profiling: [n_phases + 1] globaltimer (ns) or nullptr
  int dbg;                      // experiments
  int trace_item;               // SRL_MK_TRACE_ITEM: which attention item of a CTA the trace stamps (0: first)
  int l2_prefetch;              // GEMM phases: the first item's remaining weight boxes to L2 early
  int pairs;                    // launched as CTA pairs (cluster 2): QKV and O reduce split-K
                                // through DSMEM; attention reads finished q / K / V
  unsigned long long* trace;    // debugging: [n_phases][grid][8] per-CTA timestamps or nullptr
};

// Host: can this config run the megakernel (rows <= 64, supported G/HD)?
bool megakernel_supported(const DecoderDims& d, int slots);
// Split-K factor of a GEMM phase on `grid` CTAs (one wave unless cs = 1).
int megakernel_splits(int N, int K, int grid);
// QKV split-K factor (capped by the attention items' partial staging).
int megakernel_qkv_splits(const DecoderDims& d, int grid);
// Floats of split partials a phase needs.
size_t megakernel_ws_floats(int n_items, int cs, int rows);
size_t megakernel_smem_bytes(const DecoderDims& d);
// Co-resident clusters of two megakernel CTAs (pair mode needs grid / 2).
int megakernel_pair_clusters(const DecoderDims& d);
// CTAs of the megakernel resident per SM (0: cannot launch).
int megakernel_occupancy(const DecoderDims& d);
cudaError_t launch_megakernel(const MkParams& p, const DecoderDims& d, int grid, cudaStream_t st);

}  // namespace srl
