// attn_tc.cu -- speculative-verify attention on the 5th-generation tensor
// cores (tcgen05 + TMEM + TMA), sm_100a, bf16 cache, head dim 128.
//
// Same computation as attn_decode.cu (mask P:L846-853, GQA
// P:L834-844, SD query block P:L444-448, verify GEMM P:L905): for a
// (batch b, kv head g) unit, its M = G*t query rows (M <= 128) attend the
// unit's cap key rows; row tau = m % t sees keys [0, valid_b + tau).
// Used when M is large enough to make a real tensor-core tile (the 70B
// config's M = 8*(1+k_adm) <= 72); CUDA cores otherwise (north_star item 4).
//
// Per CTA (persistent, one per SM) the launch's (unit, 64-key tile) stream is
// split into equal contiguous shares; a CTA processes the runs of its share
// that fall into one unit ("items") one after the other:
//   warps 0, 6: TMA producers -- 2D tensor-map loads (SWIZZLE_128B) of the K
//             and the V tile (64 keys x 128 dims, 2 boxes each) into two
//             4-stage rings; a K stage is released as soon as its Q.K^T
//             MMAs complete, a V stage after its P.V MMAs;
//   warps 1, 11: TMEM allocator + Q.K^T issuer (warp 1), P.V issuer (warp
//             11); two issuers so that Q.K^T of later tiles never waits behind
//             the P.V of a tile whose softmax is still running:
//               S[b]  (TMEM, 128 lanes x 64 cols fp32) = Q . K^T
//                     M=128 x N=64 x K=128, A = Q (K-major SW128, smem),
//                     B = K tile (K-major SW128);
//               O     (TMEM, 128 x 128 fp32)          += P . V
//                     M=128 x N=128 x K=64, A = P (bf16, K-major SW128),
//                     B = V tile (MN-major SW128), issued twice: P_hi, P_lo;
//   warps 2-9: softmax / epilogue, two threads per query row (TMEM lane):
//             warps 2-5 own key columns 0-31 of every S tile and O columns
//             0-63, warps 6-9 key columns 32-63 and O columns 64-127; the
//             row max is exchanged through shared memory each tile.
//             tcgen05.ld of the S half-row, mask, online softmax with lazy
//             rescaling of O (only when the running max grows by > 8 in
//             log2 units; O is rescaled in TMEM with tcgen05.ld/st), and
//             P = exp2(s - m) split into bf16 hi + lo (P = hi + lo to 2^-17),
//             written to smem in the UMMA layout.
// The bf16 rounding of P alone (2^-9 relative) could spend the whole 2e-3
// budget on a near one-hot row; the hi/lo split makes P exact to ~2^-17 at the
// price of a second P.V MMA, which the tensor pipe has ample room for (this
// kernel is HBM-bound: 32 KiB of K+V per 3.1 M MACs).
// Split units use the same partial-record + last-CTA combine as attn_decode.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "bmc_internal.h"
#include "combine.cuh"
#include "tc_common.cuh"

namespace bmc {
namespace tc {

constexpr int D = 128;            // head dim (bf16)
constexpr int KT = 64;            // keys per tile
constexpr int MM = 128;           // MMA M (query rows, padded)
constexpr int KS = 6;             // K ring stages (released right after Q.K^T)
constexpr int VS = 7;             // V ring stages (held until P.V completes: deeper)
constexpr int NB = 2;             // S and P buffers (tiles in flight)
constexpr int kThreads = 384;     // 12 warps: K/V producers, QK / PV issuers, 2 x 4 softmax
constexpr uint32_t kTileBytes = KT * D * 2;            // 16 KiB per tensor per tile
constexpr uint32_t kBox = 64 * KT * 2;                 // one 64-col box: 8 KiB
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kRescale = 8.0f;  // lazy-rescale threshold (log2 units)
#ifndef BMC_TC_HALVES
#define BMC_TC_HALVES 2           // P.V issued for P_hi and P_lo
#endif

// Tensor memory (512 columns x 128 lanes x 32 bit):
constexpr uint32_t TM_S = 0;      // S[b]: 64 fp32 columns each (b < NB)
constexpr uint32_t TM_O = 128;    // O: 128 fp32 columns
constexpr uint32_t TM_Q = 256;    // Q: 128 bf16 = 64 packed columns (MMA A operand)
constexpr uint32_t TM_P = 320;    // P[b][hi|lo]: 64 bf16 = 32 packed columns each
// Shared memory holds only the K and V rings: the MMA A operands (Q, P) are
// read from TMEM, so per 64-key tile the tensor core reads just K (16 KiB) and
// V (2 x 16 KiB) from shared memory instead of also Q (32 KiB) and P (32 KiB).
constexpr uint32_t OFF_K = 0;                                  // [stage][2 boxes][64][128 B]
constexpr uint32_t OFF_V = OFF_K + KS * kTileBytes;
constexpr uint32_t OFF_BAR = OFF_V + VS * kTileBytes;
constexpr uint32_t OFF_X = OFF_BAR + 512;                      // [2 parity][2 halves][128] f32
constexpr uint32_t kSmem = OFF_X + 2048;   // the dynamic window starts 1024-aligned (checked)
static_assert(kSmem <= 232448, "shared memory");

#ifdef BMC_TC_TRACE
// Debug timeline (CTA 0 only): trace[event][tile] = clock64 at that point.
__device__ long long g_tc_trace[16][256];
__device__ long long g_tc_mma[2][256][9];
__device__ long long g_tc_sm[8][256][4];
__device__ long long g_tc_cta[160][4];   // per CTA: clock64 / globaltimer at entry and exit
__device__ __forceinline__ long long gtime() {
  long long c;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(c));
  return c;
}    // per softmax warp: S ready, pair, Pempty, Pfull
#define TRACE_W(ev, i) do { if (blockIdx.x == 0 && lane == 0 && (i) < 256) g_tc_sm[warp - 2][i][ev] = clk(); } while (0)   // per issuer, per tile: before each MMA + after last
__device__ __forceinline__ long long clk() {
  long long c;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
  return c;
}
#define TRACE(ev, i) do { if (blockIdx.x == 0 && (i) < 256) g_tc_trace[ev][i] = clk(); } while (0)
#else
#define TRACE(ev, i) do { } while (0)
#define TRACE_W(ev, i) do { } while (0)
#endif

struct Params {
  CUtensorMap tmK;   // [U*cap rows][128] bf16, box 64 x 64, SWIZZLE_128B
  CUtensorMap tmV;
  const __nv_bfloat16* Q;   // [B][H_q][t][D]
  float* O;                 // [B][H_q][t][D]
  const uint8_t* Knew;      // pending appended row [B][H_kv][D] (n_app == 1)
  const uint8_t* Vnew;
  const uint8_t* Kd;        // pending drafts [B][H_kv][kd_stride][D]
  const uint8_t* Vd;
  uint8_t* Kc;              // cache base (pending rows are stored here)
  uint8_t* Vc;
  int n_app, n_draft, kd_stride;
  float* ws;
  int* counters;
  long long cap;
  long long total_tiles;
  int tpu, U, H_kv, H_q, G, t, M, ctas;
  float qscale;
  int tree;                 // staged rows form a token tree (else a chain)
  uint32_t anc[32];         // tree: bit j of anc[i] = node j is node i or its ancestor
  int valid[BMC_MAX_B];
};

using namespace tcc;

__device__ __forceinline__ void softmax_sync() {  // the 8 softmax warps (2..9)
  asm volatile("bar.sync 1, 256;" ::: "memory");
}
__device__ __forceinline__ void pair_sync() {     // the 8 softmax warps, per-tile exchange
  asm volatile("bar.sync 2, 256;" ::: "memory");
}

__global__ void __launch_bounds__(kThreads, 1) attn_tc_kernel(const __grid_constant__ Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // the SWIZZLE_128B atoms need 1024-byte alignment of the dynamic window
  uint8_t* smem = smem_raw;
  const uint32_t sbase = su32(smem);
  if (sbase & 1023u) __trap();
#ifdef BMC_TC_TRACE
  if (threadIdx.x == 0) { g_tc_cta[blockIdx.x][0] = clk(); g_tc_cta[blockIdx.x][1] = gtime(); }
#endif
  const uint32_t bar0 = sbase + OFF_BAR;
  // mbarriers (8 bytes each)
  auto FULLK = [&](int s) { return bar0 + 8u * s; };               // TMA -> MMA
  auto EMPTYK = [&](int s) { return bar0 + 8u * (6 + s); };        // MMA -> TMA
  auto FULLV = [&](int s) { return bar0 + 8u * (12 + s); };
  auto EMPTYV = [&](int s) { return bar0 + 8u * (24 + s); };
  auto SFULL = [&](int b) { return bar0 + 8u * (36 + b); };        // MMA -> softmax
  auto SEMPTY = [&](int b) { return bar0 + 8u * (40 + b); };       // softmax -> MMA
  auto PFULL = [&](int b) { return bar0 + 8u * (44 + b); };        // softmax -> MMA
  auto PEMPTY = [&](int b) { return bar0 + 8u * (48 + b); };       // MMA -> softmax
  const uint32_t QFULL = bar0 + 8u * 52;                           // softmax -> MMA
  const uint32_t ODONE = bar0 + 8u * 53;                           // PV issuer -> softmax
  const uint32_t QDONE = bar0 + 8u * 54;                           // QK issuer -> softmax
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + OFF_BAR + 8 * 55);
  int* sm_flag = reinterpret_cast<int*>(smem + OFF_BAR + 8 * 55 + 8);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const long long NT = p.total_tiles;
  const long long t_begin = tile_begin(blockIdx.x, NT, p.ctas);
  const long long t_end = tile_begin(blockIdx.x + 1, NT, p.ctas);

  if (threadIdx.x == 0) {
    for (int s = 0; s < KS; ++s) {
      mbar_init(FULLK(s), 1);
      mbar_init(EMPTYK(s), 1);
    }
    for (int s = 0; s < VS; ++s) {
      mbar_init(FULLV(s), 1);
      mbar_init(EMPTYV(s), 1);
    }
    for (int b = 0; b < NB; ++b) {
      mbar_init(SFULL(b), 1);
      mbar_init(SEMPTY(b), 256);
      mbar_init(PFULL(b), 256);
      mbar_init(PEMPTY(b), 1);
    }
    mbar_init(QFULL, 256);
    mbar_init(ODONE, 1);
    mbar_init(QDONE, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     su32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // Rows >= M of Q and P in TMEM are never initialised: they only feed rows
  // of S and O that are never read (each output row depends on its own A row).
  // fused KV-cache update: rows appended / drafted since the last launch that
  // fall into this CTA's tiles are stored into the cache before its TMA loads
  // read them (P:L609 in-place update), so no separate write kernel runs
  if (p.n_app || p.n_draft) {
    constexpr int CHR = D * 2 / 16;                  // 16-byte chunks per row
    const int per_unit = (p.n_app + p.n_draft) * 2 * CHR;
    const long long u0 = t_begin / p.tpu, u1 = (t_end - 1) / p.tpu;
    for (long long x = threadIdx.x; x < (u1 - u0 + 1) * per_unit; x += kThreads) {
      const long long uu = u0 + x / per_unit;
      const int y = (int)(x % per_unit);
      const int ck = y % CHR, tensor = (y / CHR) & 1, ri = y / (2 * CHR);
      const int vb = p.valid[(int)(uu / p.H_kv)];
      int row;
      const uint8_t* src;
      if (p.n_app && ri == 0) {
        row = vb - 1;
        src = (tensor ? p.Vnew : p.Knew) + (size_t)uu * (D * 2);
      } else {
        const int di = ri - p.n_app;
        row = vb + di;
        src = (tensor ? p.Vd : p.Kd) + ((size_t)uu * p.kd_stride + di) * (D * 2);
      }
      const long long tile = uu * p.tpu + row / KT;
      if (tile < t_begin || tile >= t_end) continue;     // another CTA owns it
      const uint4 v = *reinterpret_cast<const uint4*>(src + ck * 16);
      *reinterpret_cast<uint4*>((tensor ? p.Vc : p.Kc) + ((size_t)uu * p.cap + row) * (D * 2) +
                                ck * 16) = v;
    }
    asm volatile("fence.proxy.async.global;" ::: "memory");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tO = tmem + TM_O;

  if (warp == 0 || warp == 10) {
    // ------------------------------------------------------ TMA producers
    if (lane == 0) {
      const bool isK = warp == 0;
      const CUtensorMap* tm = isK ? &p.tmK : &p.tmV;
      const int NS = isK ? KS : VS;
      const uint32_t ring = sbase + (isK ? OFF_K : OFF_V);
      const uint64_t pol = evict_first_policy();
      int s = 0;
      uint32_t ph = 0;
      long long u = t_begin / p.tpu;
      int j = (int)(t_begin % p.tpu);
      for (long long i = t_begin; i < t_end; ++i) {
        mbar_wait(isK ? EMPTYK(s) : EMPTYV(s), ph ^ 1);
        TRACE(isK ? 0 : 1, (int)(i - t_begin));
        const int row = (int)(u * p.cap + (long long)j * KT);
        const uint32_t dst = ring + s * kTileBytes;
        const uint32_t fb = isK ? FULLK(s) : FULLV(s);
        mbar_expect_tx(fb, kTileBytes);
        tma_load_2d(dst, tm, 0, row, fb, pol);
        tma_load_2d(dst + kBox, tm, 64, row, fb, pol);
        if (++j == p.tpu) { j = 0; ++u; }
        if (++s == NS) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------ Q.K^T issuer
    if (lane == 0) {
      constexpr uint32_t IQK = idesc_bf16(MM, KT, 0, 0);   // S = Q K^T, B K-major
      int ks = 0;
      uint32_t kph = 0, qph = 0;
      long long i = t_begin;
      int tcount = 0;                 // tiles of this CTA so far (S buffer index)
      while (i < t_end) {
        const long long u = i / p.tpu;
        const long long iend = min(t_end, (u + 1) * p.tpu);
        mbar_wait(QFULL, qph);        // Q of this unit is in smem
        qph ^= 1;
        fence_after();
        const int n = (int)(iend - i);
        for (int k = 0; k < n; ++k) {
          // tile c uses buffer c % NB for the (c / NB)-th time: every phase
          // parity follows from the CTA's tile counter
          const int tc = tcount + k;
          const int b = tc % NB;
          mbar_wait(FULLK(ks), kph);
          TRACE(2, tc);
          mbar_wait(SEMPTY(b), ((tc / NB) & 1) ^ 1);   // released by its previous use
          fence_after();
          const uint32_t kt = sbase + OFF_K + ks * kTileBytes;
          const uint32_t tS = tmem + TM_S + 64 * b;
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t ka = kt + (kk >> 2) * kBox + (kk & 3) * 32;
            // A = Q from TMEM: 16 bf16 of K per step = 8 packed columns
#ifdef BMC_TC_TRACE
            if (blockIdx.x == 0 && tc < 256) g_tc_mma[0][tc][kk] = clk();
#endif
            umma_f16_ts(tS, tmem + TM_Q + kk * 8, sdesc(ka, 16, 1024), IQK, kk > 0);
          }
          TRACE(3, tc);
#ifdef BMC_TC_TRACE
          if (blockIdx.x == 0 && tc < 256) g_tc_mma[0][tc][8] = clk();
#endif
          umma_commit(SFULL(b));
          umma_commit(EMPTYK(ks));    // K stage reusable once Q.K^T completed
          if (++ks == KS) { ks = 0; kph ^= 1; }
        }
        umma_commit(QDONE);           // Q may be overwritten for the next item
        tcount += n;
        i = iend;
      }
    }
  } else if (warp == 11) {
    // ------------------------------------------------------ P.V issuer
    if (lane == 0) {
      constexpr uint32_t IPV = idesc_bf16(MM, D, 0, 1);    // O += P V, B MN-major
      int vs = 0;
      uint32_t vph = 0;
      long long i = t_begin;
      int tcount = 0;
      while (i < t_end) {
        const long long u = i / p.tpu;
        const long long iend = min(t_end, (u + 1) * p.tpu);
        const int n = (int)(iend - i);
        for (int k = 0; k < n; ++k) {
          const int tc = tcount + k;
          const int b = tc % NB;
          mbar_wait(PFULL(b), (tc / NB) & 1);
          TRACE(4, tc);
          mbar_wait(FULLV(vs), vph);
          TRACE(5, tc);
          fence_after();
          const uint32_t vt = sbase + OFF_V + vs * kTileBytes;
#pragma unroll
          for (int hl = 0; hl < BMC_TC_HALVES; ++hl) {
            const uint32_t pa0 = tmem + TM_P + b * 64 + hl * 32;   // A = P from TMEM
#pragma unroll
            for (int kk = 0; kk < KT / 16; ++kk) {
              const uint32_t va = vt + kk * 2048;   // 16 keys = two 8-row groups
#ifdef BMC_TC_TRACE
              if (blockIdx.x == 0 && tc < 256) g_tc_mma[1][tc][hl * 4 + kk] = clk();
#endif
              umma_f16_ts(tO, pa0 + kk * 8, sdesc(va, kBox, 1024), IPV,
                          (k > 0 || hl > 0 || kk > 0) ? 1u : 0u);
            }
          }
#ifdef BMC_TC_TRACE
          if (blockIdx.x == 0 && tc < 256) g_tc_mma[1][tc][8] = clk();
#endif
          umma_commit(PEMPTY(b));     // P buffer b reusable, O updated
          umma_commit(EMPTYV(vs));    // V stage reusable
          if (++vs == VS) { vs = 0; vph ^= 1; }
        }
        umma_commit(ODONE);           // every P.V of this item is complete
        tcount += n;
        i = iend;
      }
    }
  } else {
    // ------------------------------------------------ softmax + epilogue
    const int half = (warp - 2) >> 2;   // 0: key cols 0-31 / O cols 0-63; 1: the rest
    const int quarter = warp & 3;       // TMEM lanes 32*quarter .. +31
    const int row = quarter * 32 + lane;
    const bool active = row < p.M;
    const uint32_t lane_addr = (uint32_t)(quarter * 32) << 16;
    const int stid = threadIdx.x - 64;  // 0..255
    float* xch = reinterpret_cast<float*>(smem + OFF_X);   // [2][128]
    uint32_t oph = 0, qdph = 0;
    long long i = t_begin;
    int tcount = 0;
    bool first_item = true;
    while (i < t_end) {
      const long long u = i / p.tpu;
      const long long iend = min(t_end, (u + 1) * p.tpu);
      const int b_ = (int)(u / p.H_kv), g_ = (int)(u % p.H_kv);
      const int j0 = (int)(i % p.tpu);
      // load this unit's query rows into smem (K-major SW128; scaled in fp32
      // later) once the previous item's Q.K^T MMAs have completed
      if (!first_item) {
        mbar_wait(QDONE, qdph);
        qdph ^= 1;
      }
      // each thread stores the half (64 dims = 32 packed columns) of its row
      {
        const __nv_bfloat16* qrow =
            p.Q + (((size_t)b_ * p.H_q + (size_t)g_ * p.G) * p.t + (active ? row : 0)) * D +
            half * 64;
        uint32_t w[32];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const uint4 v = active ? *reinterpret_cast<const uint4*>(qrow + c * 8)
                                 : make_uint4(0, 0, 0, 0);
          w[4 * c] = v.x; w[4 * c + 1] = v.y; w[4 * c + 2] = v.z; w[4 * c + 3] = v.w;
        }
        tmem_st16(tmem + TM_Q + half * 32 + lane_addr, w);
        tmem_st16(tmem + TM_Q + half * 32 + 16 + lane_addr, w + 16);
        tmem_wait_st();
      }
      fence_before();
      mbar_arrive(QFULL);
      // chain (reading R7): keys [0, valid_b + tau); token tree:
      // the committed keys plus the node's ancestors and itself
      const int vb_ = p.valid[b_];
      const int tau = row % p.t;
      const int nvis = active ? (p.tree ? vb_ : vb_ + tau) : 0;
      const uint32_t qmask = (active && p.tree && tau > 0) ? p.anc[tau - 1] : 0u;
      float m_use = -INFINITY, l = 0.f;   // l: this thread's half of the row sum
      const int n = (int)(iend - i);
      for (int k = 0; k < n; ++k) {
        const int tc = tcount + k;          // this CTA's tile counter
        const int bb = tc % NB;
        const long long key0 = (long long)(j0 + k) * KT + half * 32;
        if (stid == 0) TRACE(6, tc);
        mbar_wait(SFULL(bb), (tc / NB) & 1);
        if (stid == 0) TRACE(7, tc);
        TRACE_W(0, tc);
        fence_after();
        float sv[32];
        tmem_ld32(tmem + 64 * bb + half * 32 + lane_addr, sv);
        fence_before();
        mbar_arrive(SEMPTY(bb));
        // raw-score max of this half (qscale > 0 is applied in the exponent)
        float mt = -INFINITY;
        if (active) {
          if (key0 + 32 <= nvis) {          // fully visible half tile: no mask
            float m4[4] = {sv[0], sv[1], sv[2], sv[3]};   // 4 independent chains
#pragma unroll
            for (int c = 4; c < 32; ++c) m4[c & 3] = fmaxf(m4[c & 3], sv[c]);
            mt = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
          } else {
#pragma unroll
            for (int c = 0; c < 32; ++c) {
              const long long js = key0 + c - vb_;      // index among the staged rows
              const bool vis = key0 + c < nvis ||
                               (js >= 0 && js < 32 && ((qmask >> (js & 31)) & 1u));
              sv[c] = vis ? sv[c] : -INFINITY;
              mt = fmaxf(mt, sv[c]);
            }
          }
        }
        // exchange buffer alternates with the tile parity: the per-tile barrier
        // keeps the two threads of a row within one tile of each other
        float* xk = xch + ((tcount + k) & 1) * 256;
        xk[half * 128 + row] = mt;
        pair_sync();
        if (stid == 0) TRACE(8, tc);
        TRACE_W(1, tc);
        mt = fmaxf(mt, xk[(half ^ 1) * 128 + row]) * p.qscale;
        // P buffer bb was last read by the PV of tile tc - NB: the c-th
        // completion of PEMPTY(bb) belongs to the c-th tile using bb
        if (tc >= NB) mbar_wait(PEMPTY(bb), ((tc / NB) - 1) & 1);
        if (stid == 0) TRACE(9, tc);
        TRACE_W(2, tc);
        // lazy rescale: keep the old max unless the new one exceeds it by > 8
        // (both threads of a row take the same decision from the same values)
        bool rescale = false;
        float alpha = 1.f;
        if (active && mt > m_use + kRescale) {
          alpha = (m_use == -INFINITY) ? 0.f : fast_exp2(m_use - mt);
          rescale = (m_use != -INFINITY) && k > 0;
          m_use = mt;
          l *= alpha;
        }
        // O must not be written by PV(k-1) while it is rescaled
        if (__any_sync(0xffffffffu, rescale)) {
          const int tp = tc - 1;                    // the previous tile's PV has completed
          mbar_wait(PEMPTY(tp % NB), (tp / NB) & 1);
          fence_after();
#pragma unroll 1
          for (int h = 0; h < 2; ++h) {
            float ov[32];
            const uint32_t ta = tO + half * 64 + h * 32 + lane_addr;
            tmem_ld32(ta, ov);
            if (rescale) {
#pragma unroll
              for (int c = 0; c < 32; ++c) ov[c] *= alpha;
            }
            tmem_st32(ta, ov);
          }
          fence_before();
        }
        // P = exp2(s*qscale - m_use) split into bf16 hi + lo, stored packed in
        // TMEM as the A operand of P.V (this thread: 32 keys = 16 columns)
        uint32_t hw16[16], lw16[16];
        if (active) {
          const bool none = (m_use == -INFINITY);
          const float nm = -m_use;
          float2 ts2a = make_float2(0.f, 0.f), ts2b = make_float2(0.f, 0.f);
#pragma unroll
          for (int c8 = 0; c8 < 4; ++c8) {
            uint32_t hw[4], lw[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float p0 = none ? 0.f : fast_exp2(fmaf(sv[c8 * 8 + 2 * e], p.qscale, nm));
              const float p1 =
                  none ? 0.f : fast_exp2(fmaf(sv[c8 * 8 + 2 * e + 1], p.qscale, nm));
              const float2 pp2 = make_float2(p0, p1);
              if (e & 1) ts2b = __fadd2_rn(ts2b, pp2); else ts2a = __fadd2_rn(ts2a, pp2);
              const __nv_bfloat162 h2 = __floats2bfloat162_rn(p0, p1);
              const float2 hf = __bfloat1622float2(h2);
              const float2 lo = __ffma2_rn(hf, make_float2(-1.f, -1.f), pp2);
              const __nv_bfloat162 l2 = __floats2bfloat162_rn(lo.x, lo.y);
              hw[e] = *reinterpret_cast<const uint32_t*>(&h2);
              lw[e] = *reinterpret_cast<const uint32_t*>(&l2);
            }
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              hw16[c8 * 4 + e] = hw[e];
              lw16[c8 * 4 + e] = lw[e];
            }
          }
          l += (ts2a.x + ts2b.x) + (ts2a.y + ts2b.y);
        } else {
#pragma unroll
          for (int e = 0; e < 16; ++e) hw16[e] = lw16[e] = 0u;
        }
        const uint32_t tp = tmem + TM_P + bb * 64 + half * 16 + lane_addr;
        tmem_st16(tp, hw16);
        tmem_st16(tp + 32, lw16);
        tmem_wait_st();
        fence_before();
        mbar_arrive(PFULL(bb));
        if (stid == 0) TRACE(10, tc);
        TRACE_W(3, tc);
      }
      // ---- epilogue of this item: O (TMEM) -> output or partial record
      float* xl = xch + ((tcount + n) & 1) * 256;   // the parity no tile reads now
      xl[half * 128 + row] = l;                 // row sum = both halves
      mbar_wait(ODONE, oph);
      oph ^= 1;
      fence_after();
      softmax_sync();
      const float lrow = l + xl[(half ^ 1) * 128 + row];
      const long long ufirst = u * p.tpu, ulast = ufirst + p.tpu - 1;
      const int c_lo = cta_of_tile(ufirst, NT, p.ctas);
      const int c_hi = cta_of_tile(ulast, NT, p.ctas);
      const int nseg = c_hi - c_lo + 1;
      const size_t rec = rec_floats(p.M, D);
      float* my = p.ws + ((size_t)blockIdx.x * 2 + (first_item ? 0 : 1)) * rec;
      float* orow = p.O + (((size_t)b_ * p.H_q + (size_t)g_ * p.G) * p.t) * D + (size_t)row * D;
      const float inv = 1.f / lrow;
#pragma unroll 1
      for (int h = 0; h < 2; ++h) {
        float ov[32];
        const int col = half * 64 + h * 32;
        tmem_ld32(tO + col + lane_addr, ov);
        if (active) {
          float* dst = (nseg == 1) ? orow + col : my + (size_t)row * D + col;
          const float sc = (nseg == 1) ? inv : 1.f;
#pragma unroll
          for (int c = 0; c < 32; c += 4)
            *reinterpret_cast<float4*>(dst + c) =
                make_float4(ov[c] * sc, ov[c + 1] * sc, ov[c + 2] * sc, ov[c + 3] * sc);
        }
      }
      if (active && nseg > 1 && half == 0) {
        my[(size_t)p.M * D + row] = m_use;
        my[(size_t)p.M * D + p.M + row] = lrow;
      }
      fence_before();
      if (nseg > 1) {
        __threadfence();
        softmax_sync();
        if (stid == 0) {
          const int old = atomicAdd(&p.counters[u], 1);
          *sm_flag = (old == nseg - 1);
        }
        softmax_sync();
        if (*sm_flag) {
          __threadfence();
          if (p.M <= 16)   // few rows: spread the merge over all 256 threads
            combine_chunks<4>(p.ws, rec, c_lo, c_hi, ufirst, NT, p.ctas, p.M, D,
                              p.O + (((size_t)b_ * p.H_q + (size_t)g_ * p.G) * p.t) * D, stid,
                              256);
          else if (active) // two threads per query row merge that row's halves
            combine_row(p.ws, rec, c_lo, c_hi, ufirst, NT, p.ctas, p.M, D, row, orow,
                        half * (D / 2), D / 2);
          if (stid == 0) p.counters[u] = 0;
        }
      }
      softmax_sync();                            // xch / flag reuse by the next item
      tcount += n;
      first_item = false;
      i = iend;
    }
  }
  fence_before();
  __syncthreads();
  fence_after();
#ifdef BMC_TC_TRACE
  if (threadIdx.x == 0) { g_tc_cta[blockIdx.x][2] = clk(); g_tc_cta[blockIdx.x][3] = gtime(); }
#endif
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

}  // namespace tc

// ------------------------------------------------------------------ host

#ifdef BMC_TC_TRACE
extern "C" int bmc_tc_trace(long long* out) {   // 16 x 256 clock64 values of CTA 0
  if (cudaMemcpyFromSymbol(out, tc::g_tc_trace, sizeof(long long) * 16 * 256) != cudaSuccess) return -1;
  if (cudaMemcpyFromSymbol(out + 16 * 256, tc::g_tc_mma, sizeof(long long) * 2 * 256 * 9) != cudaSuccess) return -1;
  if (cudaMemcpyFromSymbol(out + 16 * 256 + 2 * 256 * 9, tc::g_tc_sm, sizeof(long long) * 8 * 256 * 4) != cudaSuccess) return -1;
  return cudaMemcpyFromSymbol(out + 16 * 256 + 2 * 256 * 9 + 8 * 256 * 4, tc::g_tc_cta, sizeof(long long) * 160 * 4) == cudaSuccess ? 0 : -1;
}
#endif

bool attn_tc_supported(int D, int dtype, int M) {
  return D == 128 && dtype == BMC_BF16 && M >= 1 && M <= tc::MM && encode_fn() != nullptr;
}

cudaError_t launch_attn_tc(const AttnStepArgs& a, int num_sms, cudaStream_t s) {
  for (int l = 0; l < a.L; ++l)
    if (a.layers[l].Ksrc) return cudaErrorInvalidValue;   // no copy-on-read in this kernel
  static int attr_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_dev != dev) {
    cudaError_t e = cudaFuncSetAttribute(tc::attn_tc_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tc::kSmem);
    if (e != cudaSuccess) return e;
    attr_dev = dev;
  }
  const AttnLayer& h = a.layers[0];
  tc::Params p;
  const long long U = (long long)a.B * a.H_kv;
  cudaError_t e = make_map(&p.tmK, h.K, U * h.cap, tc::KT);
  if (e == cudaSuccess) e = make_map(&p.tmV, h.V, U * h.cap, tc::KT);
  if (e != cudaSuccess) return e;
  p.Q = (const __nv_bfloat16*)h.Q;
  p.O = h.O;
  p.Knew = (const uint8_t*)h.Knew;
  p.Vnew = (const uint8_t*)h.Vnew;
  p.Kd = (const uint8_t*)h.Kd;
  p.Vd = (const uint8_t*)h.Vd;
  p.Kc = (uint8_t*)h.K;
  p.Vc = (uint8_t*)h.V;
  p.n_app = h.n_app;
  p.n_draft = h.n_draft;
  p.kd_stride = h.kd_stride;
  p.ws = h.ws;
  p.counters = h.counters;
  p.cap = h.cap;
  p.tpu = (int)(((h.scan > 0 ? h.scan : h.cap) + tc::KT - 1) / tc::KT);
  p.U = (int)U;
  p.total_tiles = U * p.tpu;
  p.H_kv = a.H_kv;
  p.H_q = a.H_q;
  p.G = a.H_q / a.H_kv;
  p.t = a.t;
  p.M = p.G * a.t;
  p.qscale = tc::kLog2e / sqrtf((float)tc::D);
  p.tree = a.tree;
  for (int i = 0; i < 32; ++i) p.anc[i] = a.anc[i];
  for (int b = 0; b < a.B; ++b) p.valid[b] = a.valid[b];
  int ctas = a.ctas > 0 ? a.ctas : num_sms;
  if (ctas > p.total_tiles) ctas = (int)p.total_tiles;
  p.ctas = ctas;
  if (p.total_tiles == 0) return cudaSuccess;
  tc::attn_tc_kernel<<<ctas, tc::kThreads, tc::kSmem, s>>>(p);
  count_launch();
  return cudaGetLastError();
}

}  // namespace bmc
