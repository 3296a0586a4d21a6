// gemm_epi.cuh -- the fused GEMM epilogues (EpiKind), shared by the
// one-tile-per-CTA decode GEMM (gemm.cu) and the persistent large-M GEMM
// (gemm_big.cu).
//
// Both kernels stage a block of the fp32 accumulator tile in shared memory as
// tile[j * pitch + c]: j = token row of the block (global row t0 + j), c = one
// of the tile's 128 output columns (global column n0 + c).  `tid`/`nthr` are
// the cooperating threads (a multiple of 32, >= 64); `sync()` is their barrier.
#pragma once
#include <cuda_bf16.h>
#include <stdint.h>

#include "gemm.cuh"

namespace srl::gemm_detail {

__device__ __forceinline__ float epi_bf2f(__nv_bfloat16 v) { return __bfloat162float(v); }
__device__ __forceinline__ float epi_warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double epi_warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float epi_warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Sum of a row's x^2 partials (one per 128 columns) in index order -- the
// loads of a batch of 8 are issued together (a dependent load-add chain costs
// one L2 round trip per part).
__device__ __forceinline__ float ssq_row_sum(const float* row, int parts) {
  float s = 0.f;
  for (int p0 = 0; p0 < parts; p0 += 8) {
    float v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = p0 + u < parts ? row[p0 + u] : 0.f;
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (p0 + u < parts) s += v[u];
  }
  return s;
}

// The epilogue kind: a compile-time constant when the kernel is specialised
// (EK >= 0; dead variants drop out of the instruction stream), else runtime.
template <int EK>
__device__ __forceinline__ int epi_kind(const EpiParams& e) { return EK >= 0 ? EK : e.kind; }

// Per-row inputs of rows [r0, r1): the deferred-RMSNorm rstd and (EPI_QKV)
// the row's KV-cache coordinates (slot, pos, page, offset in page).
template <int EK = -1>
__device__ __forceinline__ void epi_row_meta(const EpiParams& epi, int r0, int r1, int t0, int M,
                                             float* s_rstd, int4* s_row, int tid, int nthr) {
  const int kind = epi_kind<EK>(epi);
  for (int j = r0 + tid; j < r1; j += nthr) {
    float r = 1.f;
    const int m = t0 + j;
    if (epi.ssq_in != nullptr && m < M) {
      const float s = ssq_row_sum(epi.ssq_in + (size_t)m * epi.ssq_in_parts, epi.ssq_in_parts);
      r = rsqrtf(s * epi.inv_dim + epi.eps);
    }
    s_rstd[j] = r;
    if ((kind == EPI_LOGITS || kind == EPI_DLOGITS) && epi.tgt_row != nullptr)
      s_row[j] = make_int4(m < M ? epi.tgt_row[m] : -1, 0, 0, 0);
    if (kind == EPI_QKV) {
      int4 rc = make_int4(-1, 0, 0, 0);
      if (m < M) {
        rc.x = epi.row_slot[m];
        rc.y = epi.row_pos[m];
        if (rc.x >= 0) {
          rc.z = epi.block_table[(size_t)rc.x * epi.pages_per_seq + rc.y / 64];
          rc.w = rc.y % 64;
        }
      }
      s_row[j] = rc;
    }
  }
}

// The epilogue over rows [r0, r1) of the staged block.  n_tile / n_tiles
// index the per-(row, 128-column tile) outputs (EPI_LOGITS, EPI_RESID ssq).
template <int EK = -1, class Sync>
__device__ __forceinline__ void epi_apply(const EpiParams& epi, float* tile, int pitch, int r0, int r1,
                                          int t0, int n0, int n_tile, int n_tiles, int M, int N,
                                          const float* s_rstd, const int4* s_row, int tid, int nthr,
                                          Sync sync) {
  const int rows = r1 - r0;
  const int warp = tid >> 5, lane = tid & 31, nwarps = nthr >> 5;
  const int kind = epi_kind<EK>(epi);
  if (kind == EPI_STORE_F32 || kind == EPI_STORE_BF16) {
#pragma unroll 4
    for (int idx = tid; idx < rows * 128; idx += nthr) {
      const int j = r0 + (idx >> 7), c = idx & 127;
      const int m = t0 + j, n = n0 + c;
      if (m >= M || n >= N) continue;
      float v = tile[j * pitch + c] * s_rstd[j];
      if (epi.bias) v += epi_bf2f(epi.bias[n]);
      if (kind == EPI_STORE_F32)
        epi.out_f32[(size_t)m * epi.ld_out + n] = v;
      else
        epi.out_bf16[(size_t)m * epi.ld_bf16 + n] = __float2bfloat16(v);
    }
  } else if (kind == EPI_ACCUM_F32) {
    for (int idx = tid; idx < rows * 128; idx += nthr) {
      const int j = r0 + (idx >> 7), c = idx & 127;
      const int m = t0 + j, n = n0 + c;
      if (m >= M || n >= N) continue;
      epi.out_f32[(size_t)m * epi.ld_out + n] += epi.scale * tile[j * pitch + c];
    }
  } else if (kind == EPI_SWIGLU) {
#pragma unroll 4
    for (int idx = tid; idx < rows * 64; idx += nthr) {
      const int j = r0 + (idx >> 6), c = idx & 63;
      const int m = t0 + j;
      if (m >= M || n0 + c >= N) continue;
      const float g = tile[j * pitch + c] * s_rstd[j];
      const float u = tile[j * pitch + 64 + c] * s_rstd[j];
      const float a = g / (1.f + expf(-g)) * u;
      epi.out_bf16[(size_t)m * epi.ld_bf16 + (n0 >> 1) + c] = __float2bfloat16(a);
      if (epi.out2_bf16) {
        epi.out2_bf16[gu_index(m, n0 + c, N)] = __float2bfloat16(g);
        epi.out2_bf16[gu_index(m, n0 + 64 + c, N)] = __float2bfloat16(u);
      }
    }
  } else if (kind == EPI_QKV && (nthr & 127) == 0) {
    // thread = one column c for rows r0 + (tid >> 7) + k * (nthr / 128): the
    // bias is loaded once, the RoPE cos/sin of 8 rows are in flight together
    const int c = tid & 127, rstep = nthr >> 7, n = n0 + c;
    const bool colok = n < N;
    const float bias = colok ? epi_bf2f(epi.bias[n]) : 0.f;
    for (int j = r0 + (tid >> 7); j < r1; j += rstep) {
      float v = 0.f;
      if (t0 + j < M && colok) v = tile[j * pitch + c] * s_rstd[j] + bias;
      tile[j * pitch + c] = v;
    }
    sync();
    const int hd = epi.hd, half = hd >> 1;
    const int qend = epi.nq * hd, kend = (epi.nq + epi.nkv) * hd;
    const int jj = n % hd, i = jj < half ? jj : jj - half;
    const bool rot = n < kend;
    for (int jb = r0 + (tid >> 7); jb < r1; jb += 8 * rstep) {
      float co[8], si[8];
      int4 rc[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int j = jb + u * rstep;
        rc[u] = j < r1 ? s_row[j] : make_int4(-1, 0, 0, 0);
        co[u] = 1.f;
        si[u] = 0.f;
        if (rot && colok && rc[u].x >= 0 && t0 + j < M) {
          co[u] = epi.cos_sin[(size_t)rc[u].y * hd + i];
          si[u] = epi.cos_sin[(size_t)rc[u].y * hd + half + i];
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int j = jb + u * rstep, m = t0 + j;
        if (j >= r1 || m >= M || !colok || rc[u].x < 0) continue;
        const float* row = &tile[j * pitch + (c - jj)];  // this head's hd values
        float y;
        if (rot) {  // RoPE (rotate pairs (i, i + hd/2)) on q and k
          const float x1 = row[i], x2 = row[i + half];
          y = jj < half ? x1 * co[u] - x2 * si[u] : x2 * co[u] + x1 * si[u];
        } else {
          y = row[jj];
        }
        const __nv_bfloat16 b = __float2bfloat16(y);
        if (n < qend) {
          epi.q_out[(size_t)m * qend + n] = b;
        } else {
          const int kv = n < kend ? n - qend : n - kend;
          const size_t at = (((size_t)rc[u].z * epi.nkv + kv / hd) * 64 + rc[u].w) * hd + jj;
          if (n < kend) epi.kc[at] = b;
          else epi.vc[at] = b;
        }
      }
    }
  } else if (kind == EPI_QKV) {
    for (int idx = tid; idx < rows * 128; idx += nthr) {
      const int j = r0 + (idx >> 7), c = idx & 127;
      const int n = n0 + c;
      float v = 0.f;
      if (t0 + j < M && n < N) v = tile[j * pitch + c] * s_rstd[j] + epi_bf2f(epi.bias[n]);
      tile[j * pitch + c] = v;
    }
    sync();
    const int hd = epi.hd, half = hd >> 1;
    const int qend = epi.nq * hd, kend = (epi.nq + epi.nkv) * hd;
    for (int idx = tid; idx < rows * 128; idx += nthr) {
      const int j = r0 + (idx >> 7), c = idx & 127;
      const int m = t0 + j, n = n0 + c;
      const int4 rc = s_row[j];
      if (m >= M || n >= N || rc.x < 0) continue;
      const int jj = n % hd;
      const float* row = &tile[j * pitch + (c - jj)];
      float y;
      if (n < kend) {
        const int i = jj < half ? jj : jj - half;
        const float co = epi.cos_sin[(size_t)rc.y * hd + i];
        const float si = epi.cos_sin[(size_t)rc.y * hd + half + i];
        const float x1 = row[i], x2 = row[i + half];
        y = jj < half ? x1 * co - x2 * si : x2 * co + x1 * si;
      } else {
        y = row[jj];
      }
      const __nv_bfloat16 b = __float2bfloat16(y);
      if (n < qend) {
        epi.q_out[(size_t)m * qend + n] = b;
      } else {
        const int kv = n < kend ? n - qend : n - kend;
        const size_t at = (((size_t)rc.z * epi.nkv + kv / hd) * 64 + rc.w) * hd + jj;
        if (n < kend) epi.kc[at] = b;
        else epi.vc[at] = b;
      }
    }
  } else if (kind == EPI_LOGITS) {
    for (int idx = tid; idx < rows * 128; idx += nthr) {
      const int j = r0 + (idx >> 7), c = idx & 127;
      const int m = t0 + j, n = n0 + c;
      float v = -INFINITY;
      if (m < M && n < N) {
        v = tile[j * pitch + c] * s_rstd[j];
        if (epi.out_f32) epi.out_f32[(size_t)m * epi.ld_out + n] = v;
        if (epi.tgt_out && n == s_row[j].x) epi.tgt_out[m] = v;
      }
      tile[j * pitch + c] = v;
    }
    sync();
    for (int j = r0 + warp; j < r1; j += nwarps) {
      const float4 x = *reinterpret_cast<const float4*>(&tile[j * pitch + lane * 4]);
      const float mx = epi_warp_max(fmaxf(fmaxf(x.x, x.y), fmaxf(x.z, x.w)));
      double s = 0.0;
      if (mx != -INFINITY) {
        const double md = (double)mx;
        s = exp((double)x.x - md) + exp((double)x.y - md) + exp((double)x.z - md) +
            exp((double)x.w - md);
      }
      s = epi_warp_sum_d(s);
      const int m = t0 + j;
      if (lane == 0 && m < M) {
        epi.part_max[(size_t)m * n_tiles + n_tile] = mx;
        epi.part_sum[(size_t)m * n_tiles + n_tile] = s;
      }
    }
  } else if (kind == EPI_DLOGITS) {
    for (int idx = tid; idx < rows * 128; idx += nthr) {
      const int j = r0 + (idx >> 7), c = idx & 127;
      const int m = t0 + j, n = n0 + c;
      if (m >= M || n >= N) continue;
      const float x = tile[j * pitch + c] * s_rstd[j];
      const float p = __expf(x - (float)epi.lse_in[m]);
      const __nv_bfloat16 d = __float2bfloat16(epi.row_coef[m] * ((n == s_row[j].x ? 1.f : 0.f) - p));
      epi.out_bf16[(size_t)m * epi.ld_bf16 + n] = d;
      if (epi.outT_bf16) epi.outT_bf16[(size_t)n * epi.ldT + m] = d;
    }
  } else if (kind == EPI_RESID && (nthr & 127) == 0) {
    // thread = one column; the residual loads of 8 rows are in flight together
    const int c = tid & 127, rstep = nthr >> 7, n = n0 + c;
    const bool colok = n < N;
    const float gain = colok ? epi_bf2f(epi.gain[n]) : 0.f;
    for (int jb = r0 + (tid >> 7); jb < r1; jb += 8 * rstep) {
      float xr[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int j = jb + u * rstep;
        xr[u] = (j < r1 && t0 + j < M && colok) ? epi.resid[(size_t)(t0 + j) * N + n] : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int j = jb + u * rstep;
        if (j >= r1) break;
        float x = 0.f;
        if (t0 + j < M && colok) {
          const size_t o = (size_t)(t0 + j) * N + n;
          x = xr[u] + tile[j * pitch + c];
          epi.resid[o] = x;
          epi.xg[o] = __float2bfloat16(x * gain);
        }
        tile[j * pitch + c] = x;
      }
    }
    sync();
    for (int j = r0 + warp; j < r1; j += nwarps) {
      float s = 0.f;
      for (int cc = lane; cc < 128; cc += 32) {
        const float x = tile[j * pitch + cc];
        s += x * x;
      }
      s = epi_warp_sum(s);
      if (lane == 0 && t0 + j < M) epi.ssq_out[(size_t)(t0 + j) * n_tiles + n_tile] = s;
    }
  } else if (kind == EPI_RESID) {
#pragma unroll 4
    for (int idx = tid; idx < rows * 128; idx += nthr) {
      const int j = r0 + (idx >> 7), c = idx & 127;
      const int m = t0 + j, n = n0 + c;
      float x = 0.f;
      if (m < M && n < N) {
        const size_t o = (size_t)m * N + n;
        x = epi.resid[o] + tile[j * pitch + c];
        epi.resid[o] = x;
        epi.xg[o] = __float2bfloat16(x * epi_bf2f(epi.gain[n]));
      }
      tile[j * pitch + c] = x;
    }
    sync();
    for (int j = r0 + warp; j < r1; j += nwarps) {
      float s = 0.f;
      for (int c = lane; c < 128; c += 32) {
        const float x = tile[j * pitch + c];
        s += x * x;
      }
      s = epi_warp_sum(s);
      if (lane == 0 && t0 + j < M) epi.ssq_out[(size_t)(t0 + j) * n_tiles + n_tile] = s;
    }
  }
}

}  // namespace srl::gemm_detail
