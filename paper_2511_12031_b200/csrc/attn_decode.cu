// attn_decode.cu -- fused masked decode / small-M verify attention over the
// padded BMC cache, CUDA cores, sm_100a.
//
// What it computes (mask P:L846-853, GQA P:L834-844,
// SD query block P:L444-448): for every (batch b, kv head g) unit and each of
// its M = G*t query rows (query head h = g*G + m/t, chain position tau = m%t)
//     o = softmax(q K^T / sqrt(D) + bias) V,  bias_j = 0 if j < valid_b + tau
//                                             else masked,
// over ALL cap rows of the unit's slab.  Padded rows are read from HBM (the
// method's contract: they cost bandwidth) but get probability exactly 0.
//
// Design:
//  * The whole launch is one stream of 16 KiB tiles: tile i covers rows
//    [j*TR, j*TR+TR) of unit u, i = u*TPU + j.  Each CTA (one per SM,
//    persistent) takes a contiguous, equal share of that stream (split-K
//    across the sequence AND across units), so every SM streams the same
//    number of bytes regardless of B*H_kv or cap.
//  * Thread 0 also acts as the producer: it moves K and V tiles into a
//    4-stage shared-memory ring with cp.async.bulk (TMA bulk copies; each
//    tile is a contiguous slab range) completing on mbarriers, refilling a
//    stage as soon as all 8 warps released it.  No warp touches HBM for K/V
//    through registers.
//  * 8 consumer warps each own TR/8 rows of every tile and keep their own
//    online-softmax state (running max, per-lane partial sums and outputs) in
//    fp32 registers; q is held pre-scaled by log2(e)/sqrt(D) and scores use
//    exp2.  Dot products use packed FFMA2; the per-row reduction uses warp
//    shuffles over the lanes that split the row.
//  * Copy-on-read growth (SURVEY NEXT-1, P:L676-678 fused with P:L853): at a
//    growth step the tiles are read from the OLD buffer (rows < cap_old) and
//    from an L2-resident zero page (rows >= cap_old), and every staged tile
//    (after the appended row is patched in) is written to the NEW buffer with
//    a bulk shared->global copy.  That is the realloc copy + zero fill + row
//    write of the growth without a separate kernel and without reading the
//    new buffer back: cap_old rows read + cap_new rows written instead of
//    cap_old + cap_new (copy) + cap_new (attention).
//  * At a unit boundary the warps merge in shared memory.  A unit covered by
//    one CTA writes O directly; otherwise each CTA writes a partial
//    (max, sum, o) record and the last CTA to finish the unit (atomic
//    arrival counter) merges the records and writes O (split-K combine).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "bmc_internal.h"
#include "combine.cuh"

namespace bmc {
namespace attn {

constexpr int kStageBytes = 16384;  // per operand (K or V) per stage
constexpr int kConsumerWarps = 8;
constexpr int kThreads = kConsumerWarps * 32;  // 2 warps per SMSP -> 255-register budget
constexpr float kLog2e = 1.4426950408889634f;

// ------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read() {   // smem sources of my bulk stores are read
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_g2s_plain(void* dst, const void* src, uint32_t bytes,
                                               uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ void consumer_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(kConsumerWarps * 32) : "memory");
}

// 16-byte chunk -> float pairs (exact widening)
template <typename T>
struct Chunk;
template <>
struct Chunk<__nv_bfloat16> {
  static constexpr int EPC = 8;  // elements per 16-byte chunk
  __device__ static __forceinline__ void load(const uint4 c, float2* f) {
    const uint32_t w[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
    for (int i = 0; i < 4; ++i)
      f[i] = make_float2(__uint_as_float(w[i] << 16), __uint_as_float(w[i] & 0xffff0000u));
  }
};
template <>
struct Chunk<float> {
  static constexpr int EPC = 4;
  __device__ static __forceinline__ void load(const uint4 c, float2* f) {
    f[0] = make_float2(__uint_as_float(c.x), __uint_as_float(c.y));
    f[1] = make_float2(__uint_as_float(c.z), __uint_as_float(c.w));
  }
};

// Zeros for the rows a copy-on-read growth adds (static device memory is
// zero-initialised; the page stays L2-resident, so it costs no HBM reads).
__device__ __align__(128) uint8_t g_zero_page[kStageBytes];

// One layer of a launch (host fills it; kernel parameter space).
struct LayerDesc {
  const uint8_t* K;      // cache [U][cap][D]
  const uint8_t* V;
  const uint8_t* Ksrc;   // copy-on-read growth: old buffer [U][cap_src][D] (else null);
  const uint8_t* Vsrc;   //   K / V above are then the new buffer the tiles are written to
  long long cap_src;     // old row stride
  long long rows_src;    // rows [0, rows_src) come from the old buffer, the rest are zero
  const uint8_t* Q;      // [B][H_q][t][D]
  float* O;              // [B][H_q][t][D]
  const uint8_t* Knew;   // pending appended row per unit [B][H_kv][D] (n_app == 1)
  const uint8_t* Vnew;
  const uint8_t* Kd;     // pending drafts [B][H_kv][kd_stride][D] (n_draft rows)
  const uint8_t* Vd;
  float* ws;             // partial records of this layer's split units
  int* counters;         // [U] arrival counters, zero between launches
  long long cap;         // rows per unit slab (row stride)
  long long scan;        // rows streamed per unit (= cap; less only in the length-aware ablation)
  long long tile0;       // first tile of this layer in the launch's tile stream
  int tpu;               // tiles per unit
  int n_app, n_draft, kd_stride;
};

template <int MAXL>
struct Params {
  long long total_tiles;
  int L, U, H_kv, H_q, G, t;
  int M;                  // query rows per unit handled by this launch (<= MAXM)
  int m0;                 // first query row of the unit handled by this launch
  int ctas;
  float qscale;           // log2(e) / sqrt(D)
  int tree;               // staged rows form a token tree (else a chain)
  uint32_t anc[32];       // tree: bit j of anc[i] = node j is node i or its ancestor
  int valid[BMC_MAX_B];   // committed rows per batch row (incl. a pending append)
  LayerDesc layer[MAXL];
};

template <typename T, int D, int MAXM, int CPL, int CTAS>
struct Cfg {
  static constexpr int ROWB = D * (int)sizeof(T);
  static constexpr int CH = ROWB / 16;          // chunks per row
  static constexpr int LPR = CH / CPL;          // lanes per row
  static constexpr int RPP = 32 / LPR;          // rows per warp pass
  static constexpr int TR = kStageBytes / ROWB; // rows per tile
  static constexpr int RPW = TR / kConsumerWarps;
  static constexpr int PASSES = RPW / RPP;
  static constexpr int EPC = Chunk<T>::EPC;
  static constexpr int EL2 = CPL * EPC / 2;     // float2 per lane per row
  static constexpr int STAGES = CTAS == 2 ? 3 : 4;
  static_assert(LPR >= 1 && LPR <= 32 && RPW % RPP == 0 && PASSES >= 1, "bad tiling");
  static_assert(CPL == 1 || CPL == 2, "CPL");
  static constexpr size_t kRing = (size_t)STAGES * 2 * kStageBytes;
  static constexpr size_t kMerge = (size_t)kConsumerWarps * D * 4;          // one query at a time
  static constexpr size_t kSmall = (size_t)kConsumerWarps * MAXM * 2 * 4 + 64;
  static constexpr size_t kBars = 2 * STAGES * 8;
  static constexpr size_t kSmem = kRing + kMerge + kSmall + kBars + 128;
};

// CTA owning global tile x in the equal partition t0(c) = floor(c*NT/C).
__device__ __forceinline__ int cta_of_tile(long long x, long long NT, int C) {
  return (int)(((x + 1) * C + NT - 1) / NT) - 1;
}
__device__ __forceinline__ long long tile_begin(int c, long long NT, int C) {
  return (long long)c * NT / C;
}

// Position in the tile stream: layer l, unit u (= b*H_kv + g), tile j of u.
struct Cursor {
  int l, b, g, j;
  long long u;
};

template <int MAXL>
__device__ __forceinline__ Cursor locate(const Params<MAXL>& p, long long tile) {
  int l = 0;
  while (l + 1 < p.L && p.layer[l + 1].tile0 <= tile) ++l;
  const long long local = tile - p.layer[l].tile0;
  const int tpu = p.layer[l].tpu;
  Cursor c;
  c.l = l;
  c.u = local / tpu;
  c.j = (int)(local - c.u * tpu);
  c.b = (int)(c.u / p.H_kv);
  c.g = (int)(c.u - (long long)c.b * p.H_kv);
  return c;
}

template <int MAXL>
__device__ __forceinline__ void advance(const Params<MAXL>& p, Cursor& c) {
  if (++c.j == p.layer[c.l].tpu) {
    c.j = 0;
    ++c.u;
    if (++c.g == p.H_kv) { c.g = 0; ++c.b; }
    if (c.u == p.U) { c.u = 0; c.b = 0; c.g = 0; ++c.l; }
  }
}

template <typename T, int D, int MAXM, int CPL, int CTAS, int MAXL>
__global__ void __launch_bounds__(kThreads, CTAS) attn_step_kernel(const __grid_constant__ Params<MAXL> p) {
  using C = Cfg<T, D, MAXM, CPL, CTAS>;
  constexpr int S = C::STAGES;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* ring = smem;                                             // [stage][K|V][16 KiB]
  float* sm_o = reinterpret_cast<float*>(smem + C::kRing);          // [warp][D]
  float* sm_m = sm_o + (size_t)kConsumerWarps * D;                  // [warp][MAXM]
  float* sm_l = sm_m + kConsumerWarps * MAXM;                       // [warp][MAXM]
  int* sm_flag = reinterpret_cast<int*>(sm_l + kConsumerWarps * MAXM);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::kRing + C::kMerge + C::kSmall);
  uint64_t* empty = full + S;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int tid = threadIdx.x;
  const int cta = blockIdx.x;
  const long long NT = p.total_tiles;
  const long long t_begin = tile_begin(cta, NT, p.ctas);
  const long long t_end = tile_begin(cta + 1, NT, p.ctas);

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // ---- producer state (thread 0 only): tiles are issued in order
  uint64_t pol = 0;
  long long pi = t_begin;
  Cursor pc = locate(p, t_begin);
  int ps_stage = 0;
  auto issue = [&]() {
    const LayerDesc& ld = p.layer[pc.l];
    const long long row0 = (long long)pc.j * C::TR;
    const long long rows = min((long long)C::TR, ld.scan - row0);
    const uint32_t bytes = (uint32_t)(rows * C::ROWB);
    const size_t off = (size_t)(pc.u * ld.cap + row0) * C::ROWB;
    uint8_t* dk = ring + (size_t)ps_stage * 2 * kStageBytes;
    mbar_expect_tx(&full[ps_stage], 2 * bytes);
    if (ld.Ksrc == nullptr) {
      bulk_g2s(dk, ld.K + off, bytes, &full[ps_stage], pol);
      bulk_g2s(dk + kStageBytes, ld.V + off, bytes, &full[ps_stage], pol);
    } else {   // copy-on-read growth: old rows, then zero rows
      const long long nold = max(0LL, min(rows, ld.rows_src - row0));
      const uint32_t bo = (uint32_t)(nold * C::ROWB);
      if (bo) {
        const size_t so = (size_t)(pc.u * ld.cap_src + row0) * C::ROWB;
        bulk_g2s(dk, ld.Ksrc + so, bo, &full[ps_stage], pol);
        bulk_g2s(dk + kStageBytes, ld.Vsrc + so, bo, &full[ps_stage], pol);
      }
      if (bytes > bo) {
        bulk_g2s_plain(dk + bo, g_zero_page, bytes - bo, &full[ps_stage]);
        bulk_g2s_plain(dk + kStageBytes + bo, g_zero_page, bytes - bo, &full[ps_stage]);
      }
    }
    ++pi;
    advance(p, pc);
    if (++ps_stage == S) ps_stage = 0;
  };
  if (tid == 0) {
    pol = evict_first_policy();
    while (pi < t_end && pi < t_begin + S) issue();
  }

  // ---- consumers (all 8 warps)
  const int rip = lane / C::LPR;   // row within a pass
  const int cl = lane % C::LPR;    // lane within the row
  int chunk[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) chunk[c] = cl + C::LPR * ((c + rip) % CPL);

  float2 q2[MAXM][C::EL2];
  float2 o2[MAXM][C::EL2];
  float mw[MAXM], lsum[MAXM];
  int nvis[MAXM];
  uint32_t qmask[MAXM];            // tree: visible staged rows (bit j = row valid_b + j)
  int max_vis = 0;
  bool seg_first = true;
  bool seg_start = true;
  long long seg_tile0 = t_begin;   // first global tile of the current unit

  Cursor cc = locate(p, t_begin);
  int stage = 0;
  uint32_t phase = 0;

  for (long long i = t_begin; i < t_end; ++i) {
    const LayerDesc& ld = p.layer[cc.l];
    const long long row0 = (long long)cc.j * C::TR;
    const int rows_in_tile = (int)min((long long)C::TR, ld.scan - row0);
    const int vb = p.valid[cc.b];

    if (seg_start) {
      // new segment: load this unit's query rows, reset the softmax state
      seg_start = false;
      seg_tile0 = i - cc.j;
      const uint8_t* qbase =
          ld.Q + ((size_t)((size_t)cc.b * p.H_q + (size_t)cc.g * p.G) * p.t + p.m0) * C::ROWB;
      max_vis = 0;
#pragma unroll
      for (int m = 0; m < MAXM; ++m) {
        mw[m] = -INFINITY;
        lsum[m] = 0.f;
        nvis[m] = 0;
        qmask[m] = 0;
#pragma unroll
        for (int e = 0; e < C::EL2; ++e) {
          o2[m][e] = make_float2(0.f, 0.f);
          q2[m][e] = make_float2(0.f, 0.f);
        }
        if (m < p.M) {
          // chain (reading R7): rows [0, valid_b + tau); token tree:
          // the committed rows plus the node's ancestors and itself
          const int tau = (p.m0 + m) % p.t;
          nvis[m] = p.tree ? vb : vb + tau;
          qmask[m] = (p.tree && tau > 0) ? p.anc[tau - 1] : 0u;
          max_vis = max(max_vis, vb + tau);
#pragma unroll
          for (int c = 0; c < CPL; ++c) {
            const uint4 raw =
                *reinterpret_cast<const uint4*>(qbase + (size_t)m * C::ROWB + chunk[c] * 16);
            float2 f[C::EPC / 2];
            Chunk<T>::load(raw, f);
#pragma unroll
            for (int e = 0; e < C::EPC / 2; ++e)
              q2[m][c * (C::EPC / 2) + e] = make_float2(f[e].x * p.qscale, f[e].y * p.qscale);
          }
        }
      }
    }

    mbar_wait(&full[stage], phase);
    uint8_t* sk = ring + (size_t)stage * 2 * kStageBytes;
    uint8_t* sv = sk + kStageBytes;

    // ---- fused KV-cache update: rows appended / drafted since the last
    // launch are written into the cache here (P:L609 in-place update) and
    // patched into the staged tile, so no separate write kernel runs.
    {
      const int a_row = ld.n_app ? vb - 1 : -1;              // appended row
      const int d_lo = vb, d_hi = vb + ld.n_draft;           // drafts
      const long long t_lo = row0, t_hi = row0 + rows_in_tile;
      const bool has_app = ld.n_app && a_row >= t_lo && a_row < t_hi;
      const int pd_lo = (int)max((long long)d_lo, t_lo), pd_hi = (int)min((long long)d_hi, t_hi);
      const int npd = ld.n_draft ? max(0, pd_hi - pd_lo) : 0;
      if (has_app || npd > 0) {
        consumer_sync();                       // every warp has seen the TMA bytes land
        const int nrows = (has_app ? 1 : 0) + npd;
        constexpr int CHR = C::ROWB / 16;      // 16-byte chunks per row
        for (int x = tid; x < nrows * 2 * CHR; x += kThreads) {
          const int ck = x % CHR;
          const int tensor = (x / CHR) & 1;
          const int ri = x / (2 * CHR);
          int row;
          const uint8_t* src;
          if (has_app && ri == 0) {
            row = a_row;
            src = (tensor ? ld.Vnew : ld.Knew) + (size_t)cc.u * C::ROWB;
          } else {
            const int di = pd_lo - d_lo + ri - (has_app ? 1 : 0);
            row = d_lo + di;
            src = (tensor ? ld.Vd : ld.Kd) + ((size_t)cc.u * ld.kd_stride + di) * C::ROWB;
          }
          const uint4 v = *reinterpret_cast<const uint4*>(src + ck * 16);
          *reinterpret_cast<uint4*>((tensor ? sv : sk) + (size_t)(row - row0) * C::ROWB + ck * 16) = v;
          uint8_t* dst = const_cast<uint8_t*>(tensor ? ld.V : ld.K) +
                         ((size_t)cc.u * ld.cap + row) * C::ROWB + ck * 16;
          *reinterpret_cast<uint4*>(dst) = v;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        consumer_sync();
      }
    }
    if (ld.Ksrc != nullptr && tid == 0) {
      // copy-on-read growth: the staged tile (old rows, zero rows, patched
      // appended row) is the new buffer's content for these rows
      const size_t off = (size_t)(cc.u * ld.cap + row0) * C::ROWB;
      const uint32_t bytes = (uint32_t)(rows_in_tile * C::ROWB);
      bulk_s2g(const_cast<uint8_t*>(ld.K) + off, sk, bytes);
      bulk_s2g(const_cast<uint8_t*>(ld.V) + off, sv, bytes);
      bulk_commit();
    }

    if (row0 < max_vis) {  // tiles with no visible row for any query are only streamed
      // K rows of all passes first (independent loads, then independent FMA chains)
      float2 kf[C::PASSES][C::EL2];
#pragma unroll
      for (int ps = 0; ps < C::PASSES; ++ps) {
        const int row = warp * C::RPW + ps * C::RPP + rip;
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
          const uint4 raw = *reinterpret_cast<const uint4*>(sk + row * C::ROWB + chunk[c] * 16);
          Chunk<T>::load(raw, kf[ps] + c * (C::EPC / 2));
        }
      }
      float sc[C::PASSES][MAXM];
#pragma unroll
      for (int m = 0; m < MAXM; ++m) {
        if (m < p.M) {
#pragma unroll
          for (int ps = 0; ps < C::PASSES; ++ps) {
            float2 a0 = make_float2(0.f, 0.f), a1 = make_float2(0.f, 0.f);
#pragma unroll
            for (int e = 0; e < C::EL2; e += 2) {
              a0 = __ffma2_rn(q2[m][e], kf[ps][e], a0);
              if (e + 1 < C::EL2) a1 = __ffma2_rn(q2[m][e + 1], kf[ps][e + 1], a1);
            }
            sc[ps][m] = (a0.x + a1.x) + (a0.y + a1.y);
          }
        }
      }
#pragma unroll
      for (int off = 1; off < C::LPR; off <<= 1) {
#pragma unroll
        for (int m = 0; m < MAXM; ++m) {
          if (m < p.M) {
#pragma unroll
            for (int ps = 0; ps < C::PASSES; ++ps)
              sc[ps][m] += __shfl_xor_sync(0xffffffffu, sc[ps][m], off);
          }
        }
      }
      // online softmax update (per warp); probabilities overwrite the scores
#pragma unroll
      for (int m = 0; m < MAXM; ++m) {
        if (m < p.M) {
          float mt = -INFINITY;
#pragma unroll
          for (int ps = 0; ps < C::PASSES; ++ps) {
            const long long jr = row0 + warp * C::RPW + ps * C::RPP + rip;
            const long long js = jr - vb;       // index among the staged rows
            const bool vis = jr < nvis[m] ||
                             (js >= 0 && js < 32 && ((qmask[m] >> (js & 31)) & 1u));
            if (!vis) sc[ps][m] = -INFINITY;
            mt = fmaxf(mt, sc[ps][m]);
          }
#pragma unroll
          for (int off = C::LPR; off < 32; off <<= 1)
            mt = fmaxf(mt, __shfl_xor_sync(0xffffffffu, mt, off));
          const float mn = fmaxf(mw[m], mt);
          if (mn == -INFINITY) {
#pragma unroll
            for (int ps = 0; ps < C::PASSES; ++ps) sc[ps][m] = 0.f;
            continue;
          }
          float tsum = 0.f;
#pragma unroll
          for (int ps = 0; ps < C::PASSES; ++ps) {
            sc[ps][m] = fast_exp2(sc[ps][m] - mn);
            tsum += sc[ps][m];
          }
          if (mn != mw[m]) {
            const float alpha = fast_exp2(mw[m] - mn);
            lsum[m] *= alpha;
            const float2 a2 = make_float2(alpha, alpha);
#pragma unroll
            for (int e = 0; e < C::EL2; ++e) o2[m][e] = __fmul2_rn(o2[m][e], a2);
            mw[m] = mn;
          }
          lsum[m] += tsum;
        }
      }
      // P . V (rows past the end of a ragged last tile were never loaded)
      float2 vf[C::PASSES][C::EL2];
#pragma unroll
      for (int ps = 0; ps < C::PASSES; ++ps) {
        const int row = warp * C::RPW + ps * C::RPP + rip;
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
          const uint4 raw = *reinterpret_cast<const uint4*>(sv + row * C::ROWB + chunk[c] * 16);
          Chunk<T>::load(raw, vf[ps] + c * (C::EPC / 2));
        }
      }
#pragma unroll
      for (int ps = 0; ps < C::PASSES; ++ps) {
        const int row = warp * C::RPW + ps * C::RPP + rip;
        if (row < rows_in_tile) {
#pragma unroll
          for (int m = 0; m < MAXM; ++m) {
            if (m < p.M) {
              const float2 pp = make_float2(sc[ps][m], sc[ps][m]);
#pragma unroll
              for (int e = 0; e < C::EL2; ++e) o2[m][e] = __ffma2_rn(pp, vf[ps][e], o2[m][e]);
            }
          }
        }
      }
    }
    if (tid == 0 && ld.Ksrc != nullptr) bulk_wait_read();   // before the stage is refilled
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[stage]);
    if (tid == 0 && pi < t_end) {
      // refill this stage once every warp has released it
      mbar_wait(&empty[stage], phase);
      issue();
    }
    if (++stage == S) { stage = 0; phase ^= 1; }

    // ------------------------------------------------------ segment end
    const Cursor cs = cc;     // the unit this tile belongs to
    const bool seg_last = (i + 1 == t_end) || (cc.j + 1 == ld.tpu);
    advance(p, cc);
    if (!seg_last) continue;
    seg_start = true;
    const LayerDesc& sl = p.layer[cs.l];

    if (lane == 0) {
#pragma unroll
      for (int m = 0; m < MAXM; ++m) sm_m[warp * MAXM + m] = mw[m];
    }
    consumer_sync();
    const long long ufirst = seg_tile0, ulast = seg_tile0 + sl.tpu - 1;
    const int c_lo = cta_of_tile(ufirst, NT, p.ctas);
    const int c_hi = cta_of_tile(ulast, NT, p.ctas);
    const int nseg = c_hi - c_lo + 1;
    const size_t obase = ((size_t)((size_t)cs.b * p.H_q + (size_t)cs.g * p.G) * p.t + p.m0) * D;
    const size_t rec = rec_floats(p.M, D);
    float* my = sl.ws + ((size_t)cta * 2 + (seg_first ? 0 : 1)) * rec;
#pragma unroll
    for (int m = 0; m < MAXM; ++m) {
      if (m >= p.M) continue;
      float mc = -INFINITY;
      for (int w = 0; w < kConsumerWarps; ++w) mc = fmaxf(mc, sm_m[w * MAXM + m]);
      const float f = (mw[m] == -INFINITY) ? 0.f : fast_exp2(mw[m] - mc);
      // lanes of one row group hold the same lsum: sum one lane per group
      float l = lsum[m];
#pragma unroll
      for (int off = C::LPR; off < 32; off <<= 1) l += __shfl_xor_sync(0xffffffffu, l, off);
      // undo the per-row chunk rotation before summing row groups
      if (CPL == 2 && (rip & 1)) {
#pragma unroll
        for (int e = 0; e < C::EL2 / 2; ++e) {
          const float2 tmp = o2[m][e];
          o2[m][e] = o2[m][e + C::EL2 / 2];
          o2[m][e + C::EL2 / 2] = tmp;
        }
      }
#pragma unroll
      for (int e = 0; e < C::EL2; ++e) {
#pragma unroll
        for (int off = C::LPR; off < 32; off <<= 1) {
          o2[m][e].x += __shfl_xor_sync(0xffffffffu, o2[m][e].x, off);
          o2[m][e].y += __shfl_xor_sync(0xffffffffu, o2[m][e].y, off);
        }
      }
      if (rip == 0) {
        float* dst = sm_o + (size_t)warp * D;
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
          const int x0 = (cl + C::LPR * c) * C::EPC;
#pragma unroll
          for (int e = 0; e < C::EPC / 2; ++e) {
            const float2 v = o2[m][c * (C::EPC / 2) + e];
            dst[x0 + 2 * e] = v.x * f;
            dst[x0 + 2 * e + 1] = v.y * f;
          }
        }
        if (lane == 0) sm_l[warp * MAXM + m] = l * f;
      }
      consumer_sync();
      if (tid < D) {
        float o = 0.f, lt = 0.f;
#pragma unroll
        for (int w = 0; w < kConsumerWarps; ++w) {
          o += sm_o[(size_t)w * D + tid];
          lt += sm_l[w * MAXM + m];
        }
        if (nseg == 1) {
          sl.O[obase + (size_t)m * D + tid] = o / lt;
        } else {
          my[(size_t)m * D + tid] = o;
          if (tid == 0) {
            my[(size_t)p.M * D + m] = mc;
            my[(size_t)p.M * D + p.M + m] = lt;
          }
        }
      }
      consumer_sync();
    }
    seg_first = false;
    if (nseg > 1) {
      __threadfence();
      consumer_sync();
      if (tid == 0) {
        const int old = atomicAdd(&sl.counters[cs.u], 1);
        *sm_flag = (old == nseg - 1);
      }
      consumer_sync();
      if (*sm_flag) {
        __threadfence();
        // merge the nseg partial records of this unit (split-K combine)
        combine_unit<2>(sl.ws, rec, c_lo, c_hi, ufirst, NT, p.ctas, p.M, D, sl.O + obase, sm_o,
                     tid, kThreads, [] { consumer_sync(); });
        if (tid == 0) sl.counters[cs.u] = 0;
      }
      consumer_sync();  // the flag and merge buffers are reused by the next segment
    }
  }
  if (tid == 0) bulk_wait_all();   // copy-on-read stores complete before the CTA exits
}

template <typename T, int D, int MAXM, int CPL, int CTAS, int MAXL>
cudaError_t launch_t(const Params<MAXL>& prm_in, int num_sms, cudaStream_t s) {
  using C = Cfg<T, D, MAXM, CPL, CTAS>;
  auto kern = attn_step_kernel<T, D, MAXM, CPL, CTAS, MAXL>;
  static int attr_dev = -1;  // per instantiation
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_dev != dev) {
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::kSmem);
    if (e != cudaSuccess) return e;
    attr_dev = dev;
  }
  Params<MAXL> prm = prm_in;
  int ctas = prm.ctas > 0 ? prm.ctas : num_sms * CTAS;
  if (ctas > prm.total_tiles) ctas = (int)prm.total_tiles;
  prm.ctas = ctas;
  kern<<<ctas, kThreads, C::kSmem, s>>>(prm);
  count_launch();
  return cudaGetLastError();
}

template <typename T, int D, int MAXL>
cudaError_t dispatch_m(const Params<MAXL>& prm, int num_sms, cudaStream_t s) {
  if (prm.M <= 1) return launch_t<T, D, 1, 2, 2, MAXL>(prm, num_sms, s);
  if (prm.M <= 2) return launch_t<T, D, 2, 1, 2, MAXL>(prm, num_sms, s);
  if (prm.M <= 4) return launch_t<T, D, 4, 1, 1, MAXL>(prm, num_sms, s);
  return launch_t<T, D, 8, 1, 1, MAXL>(prm, num_sms, s);
}

template <int MAXL>
cudaError_t launch_chunk(const AttnStepArgs& a, int l0, int nl, int num_sms, cudaStream_t s) {
  Params<MAXL> prm;
  const int TR = kStageBytes / (a.D * (a.dtype == BMC_BF16 ? 2 : 4));
  prm.L = nl;
  prm.U = a.B * a.H_kv;
  prm.H_kv = a.H_kv;
  prm.H_q = a.H_q;
  prm.G = a.H_q / a.H_kv;
  prm.t = a.t;
  prm.ctas = a.ctas;
  prm.qscale = kLog2e / sqrtf((float)a.D);
  prm.tree = a.tree;
  for (int i = 0; i < 32; ++i) prm.anc[i] = a.anc[i];
  for (int b = 0; b < a.B; ++b) prm.valid[b] = a.valid[b];
  long long tiles = 0;
  for (int i = 0; i < nl; ++i) {
    const AttnLayer& h = a.layers[l0 + i];
    LayerDesc& d = prm.layer[i];
    d.K = (const uint8_t*)h.K;
    d.V = (const uint8_t*)h.V;
    d.Ksrc = (const uint8_t*)h.Ksrc;
    d.Vsrc = (const uint8_t*)h.Vsrc;
    d.cap_src = h.cap_src;
    d.rows_src = h.rows_src;
    if (d.Ksrc && h.scan > 0 && h.scan < h.cap) return cudaErrorInvalidValue;
    d.Q = (const uint8_t*)h.Q;
    d.O = h.O;
    d.Knew = (const uint8_t*)h.Knew;
    d.Vnew = (const uint8_t*)h.Vnew;
    d.Kd = (const uint8_t*)h.Kd;
    d.Vd = (const uint8_t*)h.Vd;
    d.ws = h.ws;
    d.counters = h.counters;
    d.cap = h.cap;
    d.scan = h.scan > 0 ? h.scan : h.cap;
    d.tpu = (int)((d.scan + TR - 1) / TR);
    d.tile0 = tiles;
    d.n_app = h.n_app;
    d.n_draft = h.n_draft;
    d.kd_stride = h.kd_stride;
    tiles += (long long)prm.U * d.tpu;
  }
  prm.total_tiles = tiles;
  if (tiles == 0) return cudaSuccess;
  const int Mu = prm.G * a.t;
  // query rows in groups of at most 8 per launch (CUDA-core path)
  for (int m0 = 0; m0 < Mu; m0 += 8) {
    prm.m0 = m0;
    prm.M = Mu - m0 < 8 ? Mu - m0 : 8;
    cudaError_t e;
    if (a.dtype == BMC_BF16) {
      e = a.D == 128 ? dispatch_m<__nv_bfloat16, 128, MAXL>(prm, num_sms, s)
                     : dispatch_m<__nv_bfloat16, 64, MAXL>(prm, num_sms, s);
    } else {
      e = a.D == 128 ? dispatch_m<float, 128, MAXL>(prm, num_sms, s)
                     : dispatch_m<float, 64, MAXL>(prm, num_sms, s);
    }
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace attn

size_t attn_workspace_floats(int M, int D, int max_ctas) {
  return (size_t)max_ctas * 2 * rec_floats(M, D);
}

cudaError_t launch_attn_step(const AttnStepArgs& a, int num_sms, cudaStream_t s) {
  if (a.L == 1) return attn::launch_chunk<1>(a, 0, 1, num_sms, s);
  for (int l0 = 0; l0 < a.L; l0 += kMaxLayersPerLaunch) {
    const int nl = a.L - l0 < kMaxLayersPerLaunch ? a.L - l0 : kMaxLayersPerLaunch;
    cudaError_t e = attn::launch_chunk<kMaxLayersPerLaunch>(a, l0, nl, num_sms, s);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace bmc
