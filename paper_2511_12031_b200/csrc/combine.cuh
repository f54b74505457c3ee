// combine.cuh -- split-K merge of partial attention records,
// shared by the CUDA-core and the tcgen05 attention kernels.
//
// A unit (batch row, kv head) whose tiles were spread over CTAs c_lo..c_hi has
// one record per CTA: o[M][D] (unnormalised, relative to that CTA's running
// max), m[M] (log2-domain max), l[M] (sum of exp2(s - m)).  The last CTA to
// finish the unit merges them:
//     mu = max_c m_c,  w_c = 2^(m_c - mu),  O = (sum_c w_c o_c) / (sum_c w_c l_c).
// Segments that saw only masked keys have m = -inf, l = 0, o = 0: weight 0.
// Both variants issue the record loads of several segments before using
// them, so a merge costs a few L2 round trips rather than M*nseg dependent
// ones.
#pragma once
#include <cuda_runtime.h>
#include <math.h>

namespace bmc {

__device__ __forceinline__ float cmb_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Record of CTA c for a unit whose first global tile is `ufirst`: slot 0 when
// the unit is the CTA's first segment, 1 otherwise.
__device__ __forceinline__ const float* cmb_record(const float* ws, int c, long long ufirst,
                                                   long long NT, int C, size_t rec) {
  const long long tb = (long long)c * NT / C;
  return ws + ((size_t)c * 2 + (tb >= ufirst ? 0 : 1)) * rec;
}

// Per-row merge weights' normalisers: mu (max) and 1/L for row r.  The
// records' scalars are loaded 8 segments at a time so a merge costs ~2 L2
// round trips per 8 segments instead of 2 per segment.
__device__ __forceinline__ void cmb_row_stats(const float* ws, size_t rec, int c_lo, int c_hi,
                                              long long ufirst, long long NT, int C, int M,
                                              int D, int r, float* mu_out, float* invl_out) {
  constexpr int BT = 8;
  float mu = -INFINITY, L = 0.f;
  for (int c0 = c_lo; c0 <= c_hi; c0 += BT) {
    float mv[BT], lv[BT];
#pragma unroll
    for (int s = 0; s < BT; ++s) {
      mv[s] = -INFINITY;
      lv[s] = 0.f;
      if (c0 + s <= c_hi) {
        const float* rr = cmb_record(ws, c0 + s, ufirst, NT, C, rec) + (size_t)M * D + r;
        mv[s] = __ldcg(rr);
        lv[s] = __ldcg(rr + M);
      }
    }
    float mb = mv[0];
#pragma unroll
    for (int s = 1; s < BT; ++s) mb = fmaxf(mb, mv[s]);
    if (mb > mu) {                       // rescale the running sum to the new max
      L = (mu == -INFINITY) ? 0.f : L * cmb_exp2(mu - mb);
      mu = mb;
    }
#pragma unroll
    for (int s = 0; s < BT; ++s)
      if (mv[s] != -INFINITY) L += lv[s] * cmb_exp2(mv[s] - mu);
  }
  *mu_out = mu;
  *invl_out = 1.f / L;
}

// Cooperative merge by `nthr` threads (tid in [0, nthr)) parallel over output
// elements, kCmbSeg segments per pass.  `wsm`: shared scratch of
// (kCmbSeg + 2) * M floats; `sync`: a barrier over the participating threads.
// D multiple of 4.
template <int kCmbSeg, typename Sync>
__device__ void combine_unit(const float* ws, size_t rec, int c_lo, int c_hi, long long ufirst,
                             long long NT, int C, int M, int D, float* out, float* wsm, int tid,
                             int nthr, Sync sync) {
  float* wgt = wsm;                     // [kCmbSeg][M]
  float* mus = wsm + kCmbSeg * M;       // [M]
  float* invl = mus + M;                // [M]
  for (int r = tid; r < M; r += nthr)
    cmb_row_stats(ws, rec, c_lo, c_hi, ufirst, NT, C, M, D, r, &mus[r], &invl[r]);
  sync();
  const int nv = M * D / 4;
  for (int c0 = c_lo; c0 <= c_hi; c0 += kCmbSeg) {
    const int ns = min(kCmbSeg, c_hi - c0 + 1);
    for (int x = tid; x < ns * M; x += nthr) {
      const int s = x / M, r = x % M;
      const float mk = __ldcg(cmb_record(ws, c0 + s, ufirst, NT, C, rec) + (size_t)M * D + r);
      wgt[s * M + r] = (mk == -INFINITY) ? 0.f : cmb_exp2(mk - mus[r]) * invl[r];
    }
    sync();
    for (int v = tid; v < nv; v += nthr) {
      const int r = (v * 4) / D;
      float4 acc = (c0 == c_lo) ? make_float4(0.f, 0.f, 0.f, 0.f)
                                : reinterpret_cast<const float4*>(out)[v];
      float4 x[kCmbSeg];
#pragma unroll
      for (int s = 0; s < kCmbSeg; ++s)
        if (s < ns)
          x[s] = __ldcg(reinterpret_cast<const float4*>(
                            cmb_record(ws, c0 + s, ufirst, NT, C, rec)) + v);
#pragma unroll
      for (int s = 0; s < kCmbSeg; ++s) {
        if (s < ns) {
          const float ww = wgt[s * M + r];
          acc.x += ww * x[s].x;
          acc.y += ww * x[s].y;
          acc.z += ww * x[s].z;
          acc.w += ww * x[s].w;
        }
      }
      reinterpret_cast<float4*>(out)[v] = acc;
    }
    sync();
  }
}

// Merge of columns [col0, col0 + ncol) of row r by one thread (the tcgen05
// epilogue has threads per query row and no spare shared memory).
// out_row: the row's D floats.  ncol multiple of 32.
__device__ inline void combine_row(const float* ws, size_t rec, int c_lo, int c_hi,
                                   long long ufirst, long long NT, int C, int M, int D, int r,
                                   float* out_row, int col0, int ncol) {
  float mu, invl;
  cmb_row_stats(ws, rec, c_lo, c_hi, ufirst, NT, C, M, D, r, &mu, &invl);
  constexpr int CH = 8;                     // float4 columns per chunk
  for (int v0 = col0 / 4; v0 < (col0 + ncol) / 4; v0 += CH) {
    float4 acc[CH];
#pragma unroll
    for (int q = 0; q < CH; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int c = c_lo; c <= c_hi; ++c) {
      const float* rr = cmb_record(ws, c, ufirst, NT, C, rec);
      const float mk = __ldcg(rr + (size_t)M * D + r);
      const float w = (mk == -INFINITY) ? 0.f : cmb_exp2(mk - mu) * invl;
      const float4* src = reinterpret_cast<const float4*>(rr + (size_t)r * D) + v0;
      float4 x[CH];
#pragma unroll
      for (int q = 0; q < CH; ++q) x[q] = __ldcg(src + q);
#pragma unroll
      for (int q = 0; q < CH; ++q) {
        acc[q].x += w * x[q].x;
        acc[q].y += w * x[q].y;
        acc[q].z += w * x[q].z;
        acc[q].w += w * x[q].w;
      }
    }
#pragma unroll
    for (int q = 0; q < CH; ++q) reinterpret_cast<float4*>(out_row)[v0 + q] = acc[q];
  }
}

// Merge by `nthr` threads parallel over 16-byte chunks of the unit's M x D
// output (no shared memory): each thread recomputes the stats of the rows it
// touches (2*nseg L2-resident scalars) and loads its chunk of every record
// before combining.  out: the unit's M*D floats.
template <int SEG>
__device__ void combine_chunks(const float* ws, size_t rec, int c_lo, int c_hi, long long ufirst,
                               long long NT, int C, int M, int D, float* out, int tid, int nthr) {
  const int nv = M * D / 4;
  for (int v = tid; v < nv; v += nthr) {
    const int r = (v * 4) / D;
    float mu, invl;
    cmb_row_stats(ws, rec, c_lo, c_hi, ufirst, NT, C, M, D, r, &mu, &invl);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int c0 = c_lo; c0 <= c_hi; c0 += SEG) {
      float4 x[SEG];
      float w[SEG];
#pragma unroll
      for (int s = 0; s < SEG; ++s) {
        if (c0 + s <= c_hi) {
          const float* rr = cmb_record(ws, c0 + s, ufirst, NT, C, rec);
          x[s] = __ldcg(reinterpret_cast<const float4*>(rr) + v);
          const float mk = __ldcg(rr + (size_t)M * D + r);
          w[s] = (mk == -INFINITY) ? 0.f : cmb_exp2(mk - mu) * invl;
        }
      }
#pragma unroll
      for (int s = 0; s < SEG; ++s) {
        if (c0 + s <= c_hi) {
          acc.x += w[s] * x[s].x;
          acc.y += w[s] * x[s].y;
          acc.z += w[s] * x[s].z;
          acc.w += w[s] * x[s].w;
        }
      }
    }
    reinterpret_cast<float4*>(out)[v] = acc;
  }
}

}  // namespace bmc
