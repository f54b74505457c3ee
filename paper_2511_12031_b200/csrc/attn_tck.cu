// attn_tck.cu -- GQA / speculative-verify attention on the 5th-generation
// tensor cores with the KEYS on the TMEM lanes, sm_100a, bf16 cache, D = 128.
//
// Same computation as attn_decode.cu and attn_tc.cu (mask
// P:L846-853, GQA P:L834-844, SD query block P:L444-448, token trees
// P:L863-866): for a (batch b, kv head g) unit, its M = G*t query rows
// attend the unit's cap key rows; row tau = m % t sees keys [0, valid_b + tau)
// (chain) or the committed keys plus its node's ancestors (tree).
//
// Why this orientation: attn_tc.cu puts the M query rows on the TMEM lanes
// (S = Q K^T, MMA M = 128 rows).  A TMEM lane quadrant q is reachable only
// from warps with warp % 4 == q, which is also the SM sub-partition, so for
// M <= 32 every exp2 / convert of the softmax lands on one SMSP: ~1000 cycles
// per 64-key tile, the kernel's measured bottleneck (profiles/
// r01_tc_trace_findings.txt).  Here the 128 keys of a tile are the MMA M:
//     S^T[b] (TMEM, 128 key lanes x N cols fp32) = K_tile . Q^T
//            M=128 (keys) x N (queries, M padded to 16 or 32) x K=128 (dims),
//            A = K tile (K-major SW128), B = Q (K-major SW128, smem);
//     O^T    (TMEM, 128 dim lanes x 2N cols fp32) += V_tile^T . [P_hi; P_lo]^T
//            M=128 (dims) x 2N x K=128 (keys), A = V tile (MN-major SW128),
//            B = P^T hi columns then lo columns (MN-major SWIZZLE_32B, smem:
//            a thread holds one key and N/2 consecutive queries, so its P
//            values are contiguous and go out as 16-byte stores),
// so every lane of every softmax warp carries one key and a thread's work per
// tile is the N/2 queries of its half, not 32 keys: the exp2 / pack work is
// spread over all four SMSPs and shrinks by 128/N.
//
// Roles (384 threads, one persistent CTA per SM, stream-K tile split):
//   warp 0 / 10: TMA producers of the K / V rings (2D tensor maps, boxes of
//                64 dims x 128 keys, SWIZZLE_128B);
//   warp 1:      TMEM allocator + S^T issuer;  warp 11: O^T issuer;
//   warps 2-9:   softmax; warp w owns TMEM lane quadrant w % 4 (keys
//                32*(w%4) .. +31 of each tile, dims 32*(w%4) .. of O^T) and
//                query half (w - 2) / 4 (columns h*N/2 .. +N/2).
// Online softmax with a lazy max (P:L274-276 restated as exp2 of
// log2-scaled scores): a column's running max m only moves when a score
// exceeds it by more than 8 (log2 units); the check is one barrier-reduction
// (bar.red.or) per tile over the 4 warps of a half, and the column maxima are
// reduced only when it fires.  P = 2^(s - m) is split into bf16 hi (upper 16
// bits) + lo (rounded remainder): P = hi + lo to ~2^-16 relative, so the
// tensor-core P.V keeps the bf16 path inside its 2e-3 budget.
// Split units use the partial-record + last-CTA combine of combine.cuh.
// Copy-on-read growth (as in attn_decode.cu): when the launch
// follows a BMC growth, the producers load 3D boxes {dims, keys, unit} of the
// OLD buffer (rows >= cap_old are out of bounds: TMA fills zeros), the MMA
// issuers patch the pending appended / drafted rows into the staged tile and
// TMA-store it into the NEW buffer before their MMAs, so the growth needs no
// realloc kernel and the new buffer is written once, never read back.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <limits.h>
#include <math.h>
#include <stdint.h>

#include <unordered_map>

#include "bmc_internal.h"
#include "combine.cuh"
#include "tc_common.cuh"

namespace bmc {
namespace tck {
using namespace tcc;

constexpr int D = 128;            // head dim (bf16)
constexpr int KT = 128;           // keys per tile = MMA M of S^T
constexpr int NB = 2;             // S^T / P^T buffers (tiles in flight)
constexpr uint32_t kTileBytes = KT * D * 2;   // 32 KiB per tensor per tile
constexpr uint32_t kBox = 64 * 2 * KT;        // one 64-dim box of a tile: 16 KiB
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kRescale = 8.0f;

// NG column groups of softmax warps (4 warps each, one per TMEM lane
// quadrant): 2 (384 threads) or 4 (640 threads: twice the warps per SMSP to
// hide the TMEM / shared-memory / barrier latencies of large N)
// NS <= N: query columns the softmax handles (the MMAs run N, a multiple of
// 16).  Softmax over 72 of 80 columns at M = 72 and over 8 of 16 at M = 1
// measured no faster (same-box A/Bs: the M = 72 tile period is set by
// shared-memory traffic, M = 1 is HBM-bound), so the launcher uses NS = N.
template <int N, int NG, int NS = N>
struct Cfg {
  static_assert(N % 16 == 0 && N >= 16 && N <= 80, "query columns");
  static_assert(NG >= 2 && NG <= 4, "column groups");
  static_assert(NS <= N && NS % (4 * NG) == 0, "softmax columns");
  static constexpr int NH = NS / NG;                        // columns per softmax group
  static constexpr int kSoftmax = NG * 128;                 // softmax threads
  static constexpr int kThreads = 128 + kSoftmax;
  static constexpr int kWarpV = 2 + 4 * NG;                 // V producer
  static constexpr int kWarpPV = 3 + 4 * NG;                // O^T issuer
  // NS < N (the 70B verify, M = 72 in an N = 80 tile): the hi / lo stack of
  // P^T is 2*NS columns wide (PV MMA N = 144, not 160), which frees the shared
  // memory for a second P^T buffer once Q is single-buffered and loaded by TMA
  // (QTMA): the softmax of tile i+1 then stores its P^T while the O^T MMAs of
  // tile i read the other buffer instead of waiting for them
  static constexpr bool QTMA = NS < N;
  static constexpr int QB = QTMA ? 1 : 2;                   // Q buffers
#ifdef BMC_M72_KS3   // experiment: a third K stage instead of the second P^T buffer
  static constexpr int NBP = N < 64 ? 2 : 1;                // P^T buffers
  static constexpr int KS = (N <= 16 || QTMA) ? 3 : 2;      // K ring stages
#else
  static constexpr int NBP = (N < 64 || QTMA) ? 2 : 1;      // P^T buffers
  static constexpr int KS = N <= 16 ? 3 : 2;                // K ring stages
#endif
  static constexpr int VS = N <= 32 ? 3 : 2;                // V ring stages
  static constexpr int NQK = QTMA ? NS : N;                 // S^T MMA N (query columns)
  static constexpr uint32_t OFF_K = 0;
  static constexpr uint32_t OFF_V = OFF_K + KS * kTileBytes;
  static constexpr uint32_t OFF_Q = OFF_V + VS * kTileBytes;   // [QB bufs][2 dim atoms][N][128 B]
  static constexpr uint32_t kQAtom = N * 128;
  static constexpr uint32_t kQBytes = 2 * kQAtom;
  // P^T (MN-major SWIZZLE_32B): [NBP][2NS/16 query blocks][128 keys][32 B]
  static constexpr uint32_t OFF_P = OFF_Q + QB * kQBytes;
  static constexpr uint32_t kPBlock = KT * 32;                 // LBO: one 16-query block
  static constexpr uint32_t kPBytes = 2 * NS / 16 * kPBlock;
  static constexpr uint32_t OFF_BAR = OFF_P + NBP * kPBytes;
  static constexpr uint32_t OFF_RED = OFF_BAR + 512;            // [NG][4 quadrants][NH] f32
  static constexpr uint32_t OFF_SUM = OFF_RED + NG * 4 * NH * 4;  // [NG][4][NH] f32
  // running maxima: [NG][2 versions][m, m-or-0, m+8][NH] f32
  static constexpr uint32_t OFF_M = OFF_SUM + NG * 4 * NH * 4;
  static constexpr uint32_t OFF_A = OFF_M + NG * 2 * 3 * NH * 4;  // [NG][NH] rescale factors
  static constexpr uint32_t OFF_LIM = OFF_A + NG * NH * 4;        // [NG][NH] int visible-key limit
  static constexpr uint32_t OFF_QM = OFF_LIM + NG * NH * 4;       // [NG][NH] ancestor masks
  static constexpr uint32_t kSmem = OFF_QM + NG * NH * 4;
  static_assert(kSmem <= 232448, "shared memory");
  static_assert(kQAtom % 1024 == 0 && kPBytes % 1024 == 0, "swizzle atoms");
  static_assert(NH % 4 == 0, "8- or 16-byte P stores");
  static constexpr int CS = NH % 8 == 0 ? 8 : 4;               // column step of TMEM / P chunks
  static_assert(NBP * kPBytes >= (4 + 2) * N * 4, "combine scratch in the P area");
  static_assert((2 * NS) % 16 == 0 && NQK % 8 == 0, "MMA N");
  // TMEM columns: S^T[b] at b*N, O^T (hi NS cols, lo NS cols) at NB*N
  static constexpr uint32_t TM_O = NB * N;
  static constexpr uint32_t kTmemCols = (NB * N + 2 * NS <= 256) ? 256 : 512;
};

#ifdef BMC_TC_TRACE
// Debug timeline (CTA 0): per tile clock64 at each wait / issue point; per CTA entry / exit.
__device__ long long g_tck_trace[16][256];
__device__ long long g_tck_cta[160][4];
__device__ __forceinline__ long long clk() {
  long long c;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
  return c;
}
__device__ __forceinline__ long long gtime() {
  long long c;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(c));
  return c;
}
__device__ int g_tck_trace_cta;
#define TRACE(ev, i) do { if (blockIdx.x == g_tck_trace_cta && (i) < 256) g_tck_trace[ev][i] = clk(); } while (0)
#else
#define TRACE(ev, i) do { } while (0)
#endif

// One layer of a launch (a decode step fuses up to 32 layers of one shape)
struct LayerP {
  CUtensorMap tmK;          // [U*cap rows][128] bf16, box 64 x 128, SWIZZLE_128B
  CUtensorMap tmV;          //   (copy-on-read: [U][cap_old][128] of the old buffer, 3D boxes)
  CUtensorMap tmKd;         // copy-on-read only: [U][cap][128] of the new buffer
  CUtensorMap tmVd;
  CUtensorMap tmQ;          // QTMA only: [B*H_q*t rows][128] bf16, box 64 x N, SWIZZLE_128B
  const __nv_bfloat16* Q;   // [B][H_q][t][D]
  float* O;                 // [B][H_q][t][D]
  const uint8_t* Knew;      // pending appended row [B][H_kv][D] (n_app == 1)
  const uint8_t* Vnew;
  const uint8_t* Kd;        // pending drafts [B][H_kv][kd_stride][D]
  const uint8_t* Vd;
  uint8_t* Kc;              // cache base (pending rows are stored here)
  uint8_t* Vc;
  float* ws;                // split-K partial records of this layer
  int* counters;            // [U]
};
template <int MAXL>
struct Params {
  LayerP lay[MAXL];
  int L;
  int n_app, n_draft, kd_stride;
  long long cap;            // rows per unit (every layer of a launch)
  long long total_tiles;    // L * U * tpu
  int tpu, U, H_kv, H_q, G, t, M, ctas;
  float qscale;
  int tree;
  int cor;                  // copy-on-read growth launch
  int pf;                   // L2 prefetch distance of the K / V producers (tiles; 0 = off)
  uint32_t anc[32];
  int valid[BMC_MAX_B];
};

// Copy-on-read: write the pending appended / drafted rows of unit uu that fall
// into tile rows [row0, row0 + KT) into the staged K or V tile (SWIZZLE_128B
// boxes of 64 dims x 128 keys); one thread, rare (about one tile per unit).
template <int MAXL>
__device__ __forceinline__ void patch_pending(const Params<MAXL>& p, const LayerP& ly, long long uu,
                                              int row0, uint32_t tile, bool isV) {
  const int vb = p.valid[(int)(uu / p.H_kv)];
  const int n = p.n_app + p.n_draft;
  for (int ri = 0; ri < n; ++ri) {
    int row;
    const uint8_t* src;
    if (p.n_app && ri == 0) {
      row = vb - 1;
      src = (isV ? ly.Vnew : ly.Knew) + (size_t)uu * (D * 2);
    } else {
      const int di = ri - p.n_app;
      row = vb + di;
      src = (isV ? ly.Vd : ly.Kd) + ((size_t)uu * p.kd_stride + di) * (D * 2);
    }
    const int r = row - row0;
    if (r < 0 || r >= KT) continue;
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      const uint4 v = *reinterpret_cast<const uint4*>(src + c * 16);
      const uint32_t off = (uint32_t)(c >> 3) * kBox + sw128((uint32_t)r, (uint32_t)(c & 7));
      asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(tile + off), "r"(v.x), "r"(v.y),
                   "r"(v.z), "r"(v.w)
                   : "memory");
    }
  }
}

template <int NT>
__device__ __forceinline__ void softmax_sync() {   // the softmax warps
  asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
}
__device__ __forceinline__ void half_sync(int h) {  // the 4 warps of one column group
  asm volatile("bar.sync %0, 128;" ::"r"(2 + h) : "memory");
}
// OR of `pred` over the 4 warps of query half h (a barrier with reduction)
__device__ __forceinline__ bool half_any(int h, bool pred) {
  uint32_t r;
  asm volatile(
      "{\n\t.reg .pred p, q;\n\t"
      "setp.ne.u32 p, %2, 0;\n\t"
      "bar.red.or.pred q, %1, 128, p;\n\t"
      "selp.u32 %0, 1, 0, q;\n\t}"
      : "=r"(r)
      : "r"(2 + h), "r"((uint32_t)pred)
      : "memory");
  return r != 0;
}
__device__ __forceinline__ void sts_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c,
                                       uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c),
               "r"(d)
               : "memory");
}
__device__ __forceinline__ void fence_proxy_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// NC consecutive fp32 TMEM columns of this warp's lane quadrant (NC % 4 == 0)
template <int NC>
__device__ __forceinline__ void tmem_ld_cols(uint32_t taddr, float* v) {
#pragma unroll
  for (int c = 0; c + 8 <= NC; c += 8) {
    uint32_t* r = reinterpret_cast<uint32_t*>(v + c);
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7])
        : "r"(taddr + c));
  }
  if constexpr (NC % 8 == 4) {
    uint32_t* r = reinterpret_cast<uint32_t*>(v + NC - 4);
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(taddr + NC - 4));
  }
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
template <int NC>
__device__ __forceinline__ void tmem_st_cols(uint32_t taddr, const float* v) {
#pragma unroll
  for (int c = 0; c + 8 <= NC; c += 8) {
    const uint32_t* r = reinterpret_cast<const uint32_t*>(v + c);
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr + c),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
        : "memory");
  }
  if constexpr (NC % 8 == 4) {
    const uint32_t* r = reinterpret_cast<const uint32_t*>(v + NC - 4);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr + NC - 4),
                 "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3])
                 : "memory");
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void sts_v2(uint32_t addr, uint32_t a, uint32_t b) {
  asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(addr), "r"(a), "r"(b) : "memory");
}
__device__ __forceinline__ float warp_max(float x) {   // one CREDUX on sm_100a
  float y;
  asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float warp_sum(float x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

template <int N, int MAXL, int NG, int NS>
__global__ void __launch_bounds__(Cfg<N, NG, NS>::kThreads, 1)
    attn_tck_kernel(const __grid_constant__ Params<MAXL> p) {
  using C = Cfg<N, NG, NS>;
  constexpr int kThreads = C::kThreads;
  constexpr int NH = C::NH;
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sbase = su32(smem);
  if (sbase & 1023u) __trap();
#ifdef BMC_TC_TRACE
  if (threadIdx.x == 0) { g_tck_cta[blockIdx.x][0] = clk(); g_tck_cta[blockIdx.x][1] = gtime(); }
#endif
  const uint32_t bar0 = sbase + C::OFF_BAR;
  auto FULLK = [&](int s) { return bar0 + 8u * s; };
  auto EMPTYK = [&](int s) { return bar0 + 8u * (4 + s); };
  auto FULLV = [&](int s) { return bar0 + 8u * (8 + s); };
  auto EMPTYV = [&](int s) { return bar0 + 8u * (12 + s); };
  auto SFULL = [&](int b) { return bar0 + 8u * (16 + b); };    // S^T MMA -> softmax
  auto SEMPTY = [&](int b) { return bar0 + 8u * (18 + b); };   // softmax read S^T[b]
  auto PFULL = [&](int b) { return bar0 + 8u * (20 + b); };    // P^T[b] in smem
  auto PEMPTY = [&](int b) { return bar0 + 8u * (22 + b); };   // O^T MMA read P^T[b]
  auto QFULL = [&](int b) { return bar0 + 8u * (24 + b); };    // Q buffer b written
  auto QDONE = [&](int b) { return bar0 + 8u * (26 + b); };    // S^T MMAs done with Q buffer b
  const uint32_t ODONE = bar0 + 8u * 28;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::OFF_BAR + 8 * 30);
  int* sm_flag = reinterpret_cast<int*>(smem + C::OFF_BAR + 8 * 31);
  int* resc_flag = reinterpret_cast<int*>(smem + C::OFF_BAR + 8 * 32);   // [2 halves]

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const long long NT = p.total_tiles;
  const long long t_begin = tile_begin(blockIdx.x, NT, p.ctas);
  const long long t_end = tile_begin(blockIdx.x + 1, NT, p.ctas);

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::KS; ++s) {
      mbar_init(FULLK(s), 1);
      mbar_init(EMPTYK(s), 1);
    }
    for (int s = 0; s < C::VS; ++s) {
      mbar_init(FULLV(s), 1);
      mbar_init(EMPTYV(s), 1);
    }
    for (int b = 0; b < NB; ++b) {
      mbar_init(SFULL(b), 1);
      mbar_init(SEMPTY(b), C::kSoftmax);
    }
    for (int b = 0; b < C::NBP; ++b) {
      mbar_init(PFULL(b), C::kSoftmax);
      mbar_init(PEMPTY(b), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(QFULL(b), C::QTMA ? 1 : C::kSoftmax);   // QTMA: the K producer's expect_tx
      mbar_init(QDONE(b), 1);
    }
    mbar_init(ODONE, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     su32(tmem_slot)), "n"(C::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // fused KV-cache update: the pending appended / drafted rows that
  // fall into this CTA's tiles are stored before its TMA loads read them
  if (p.n_app || p.n_draft) {
    constexpr int CHR = D * 2 / 16;
    const int per_unit = (p.n_app + p.n_draft) * 2 * CHR;
    const long long u0 = t_begin / p.tpu, u1 = (t_end - 1) / p.tpu;
    for (long long x = threadIdx.x; x < (u1 - u0 + 1) * per_unit; x += kThreads) {
      const long long gu = u0 + x / per_unit;          // global unit: layer * U + unit
      const LayerP& ly = p.lay[MAXL == 1 ? 0 : (int)(gu / p.U)];
      const long long uu = gu % p.U;
      const int y = (int)(x % per_unit);
      const int ck = y % CHR, tensor = (y / CHR) & 1, ri = y / (2 * CHR);
      const int vb = p.valid[(int)(uu / p.H_kv)];
      int row;
      const uint8_t* src;
      if (p.n_app && ri == 0) {
        row = vb - 1;
        src = (tensor ? ly.Vnew : ly.Knew) + (size_t)uu * (D * 2);
      } else {
        const int di = ri - p.n_app;
        row = vb + di;
        src = (tensor ? ly.Vd : ly.Kd) + ((size_t)uu * p.kd_stride + di) * (D * 2);
      }
      const long long tile = gu * p.tpu + row / KT;
      if (tile < t_begin || tile >= t_end) continue;
      const uint4 v = *reinterpret_cast<const uint4*>(src + ck * 16);
      *reinterpret_cast<uint4*>((tensor ? ly.Vc : ly.Kc) + ((size_t)uu * p.cap + row) * (D * 2) +
                                ck * 16) = v;
    }
    asm volatile("fence.proxy.async.global;" ::: "memory");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 || warp == C::kWarpV) {
    // ------------------------------------------------------ TMA producers
    if (lane == 0) {
      const bool isK = warp == 0;
      const int nst = isK ? C::KS : C::VS;
      const uint32_t ring = sbase + (isK ? C::OFF_K : C::OFF_V);
      const uint64_t pol = evict_first_policy();
      int s = 0;
      uint32_t ph = 0;
      long long gu = t_begin / p.tpu;               // global unit
      int j = (int)(t_begin % p.tpu);
      int item = 0;
      for (long long i = t_begin; i < t_end; ++i) {
        if constexpr (C::QTMA) {
          // the item's Q rows (M of N loaded; the rest are neighbouring rows in
          // softmax columns >= NS that nobody reads) into the single Q buffer
          // once the S^T MMAs of the previous item are done with it
          if (isK && (i == t_begin || j == 0)) {
            if (item > 0) mbar_wait(QDONE(0), (item - 1) & 1);
            const LayerP& lq = p.lay[MAXL == 1 ? 0 : (int)(gu / p.U)];
            const long long uq = gu % p.U;
            const int row = (int)(((uq / p.H_kv) * p.H_q + (uq % p.H_kv) * p.G) * p.t);
            const uint32_t qs = sbase + C::OFF_Q;
            mbar_expect_tx(QFULL(0), C::kQBytes);
            tma_load_2d(qs, &lq.tmQ, 0, row, QFULL(0), pol);
            tma_load_2d(qs + C::kQAtom, &lq.tmQ, 64, row, QFULL(0), pol);
            ++item;
          }
        }
        mbar_wait(isK ? EMPTYK(s) : EMPTYV(s), ph ^ 1);
        TRACE(isK ? 0 : 1, (int)(i - t_begin));
        const LayerP& ly = p.lay[MAXL == 1 ? 0 : (int)(gu / p.U)];
        const CUtensorMap* tm = isK ? &ly.tmK : &ly.tmV;
        const uint32_t dst = ring + s * kTileBytes;
        const uint32_t fb = isK ? FULLK(s) : FULLV(s);
        mbar_expect_tx(fb, kTileBytes);
        if (p.cor) {   // old buffer, zeros past its rows
          const int uu = (int)(gu % p.U);
          tma_load_3d(dst, tm, 0, j * KT, uu, fb, pol);
          tma_load_3d(dst + kBox, tm, 64, j * KT, uu, fb, pol);
        } else {
          const int row = (int)((gu % p.U) * p.cap + (long long)j * KT);
          tma_load_2d(dst, tm, 0, row, fb, pol);
          tma_load_2d(dst + kBox, tm, 64, row, fb, pol);
        }
        // the tile pf ahead of this one into L2 (under full HBM load a TMA
        // load takes ~2-4 us; the ring's 2-3 stages alone cannot cover it)
        if (p.pf > 0 && i + p.pf < t_end) {
          const long long ip = i + p.pf;
          const long long gp = ip / p.tpu;
          const int jp = (int)(ip % p.tpu);
          const LayerP& lp = p.lay[MAXL == 1 ? 0 : (int)(gp / p.U)];
          const CUtensorMap* tp = isK ? &lp.tmK : &lp.tmV;
          if (p.cor) {
            tma_prefetch_3d(tp, 0, jp * KT, (int)(gp % p.U));
            tma_prefetch_3d(tp, 64, jp * KT, (int)(gp % p.U));
          } else {
            const int rp = (int)((gp % p.U) * p.cap + (long long)jp * KT);
            tma_prefetch_2d(tp, 0, rp);
            tma_prefetch_2d(tp, 64, rp);
          }
        }
        if (++j == p.tpu) { j = 0; ++gu; }
        if (++s == nst) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------ S^T = K Q^T issuer
    if (lane == 0) {
      constexpr uint32_t IQK = idesc_bf16(KT, C::NQK, 0, 0);
      int ks = 0;
      uint32_t kph = 0;
      long long i = t_begin;
      int tcount = 0, item = 0;
      while (i < t_end) {
        const long long gu = i / p.tpu;
        const long long iend = min(t_end, (gu + 1) * p.tpu);
        const int qb = C::QB == 1 ? 0 : (item & 1);
        const uint32_t qs = sbase + C::OFF_Q + qb * C::kQBytes;
        mbar_wait(QFULL(qb), C::QB == 1 ? (item & 1) : ((item >> 1) & 1));
        fence_after();
        const int n = (int)(iend - i);
        for (int k = 0; k < n; ++k) {
          const int tc = tcount + k;
          const int b = tc % NB;
          mbar_wait(FULLK(ks), kph);
          TRACE(2, tc);
          const uint32_t kt = sbase + C::OFF_K + ks * kTileBytes;
          if (p.cor) {   // copy-on-read: patched tile -> new buffer (read before the refill)
            const long long gk = i + k;
            const LayerP& ly = p.lay[MAXL == 1 ? 0 : (int)((gk / p.tpu) / p.U)];
            const long long uu = (gk / p.tpu) % p.U;
            const int row0 = (int)(gk % p.tpu) * KT;
            patch_pending(p, ly, uu, row0, kt, false);
            fence_proxy_smem();
            tma_store_3d(&ly.tmKd, kt, 0, row0, (int)uu);
            tma_store_3d(&ly.tmKd, kt + kBox, 64, row0, (int)uu);
            bulk_commit_wait_read();
          }
          mbar_wait(SEMPTY(b), ((tc / NB) & 1) ^ 1);
          TRACE(3, tc);
          fence_after();
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t koff = (kk >> 2) * kBox + (kk & 3) * 32;
            const uint32_t qoff = (kk >> 2) * C::kQAtom + (kk & 3) * 32;
            umma_f16(tmem + b * N, sdesc(kt + koff, 16, 1024), sdesc(qs + qoff, 16, 1024), IQK,
                     kk > 0);
          }
          TRACE(4, tc);
          umma_commit(SFULL(b));
          umma_commit(EMPTYK(ks));
          if (++ks == C::KS) { ks = 0; kph ^= 1; }
        }
        umma_commit(QDONE(qb));
        tcount += n;
        ++item;
        i = iend;
      }
      if (p.cor) bulk_wait_all();
    }
  } else if (warp == C::kWarpPV) {
    // ------------------------------------------------------ O^T += V^T P^T issuer
    if (lane == 0) {
      constexpr uint32_t IPV = idesc_bf16(D, 2 * NS, 1, 1);  // A = V tile, B = P^T: MN-major
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
          const int b = tc % C::NBP;
          mbar_wait(PFULL(b), (tc / C::NBP) & 1);
          TRACE(5, tc);
          mbar_wait(FULLV(vs), vph);
          TRACE(6, tc);
          const uint32_t vt = sbase + C::OFF_V + vs * kTileBytes;
          if (p.cor) {
            const long long gk = i + k;
            const LayerP& ly = p.lay[MAXL == 1 ? 0 : (int)((gk / p.tpu) / p.U)];
            const long long uu = (gk / p.tpu) % p.U;
            const int row0 = (int)(gk % p.tpu) * KT;
            patch_pending(p, ly, uu, row0, vt, true);
            fence_proxy_smem();
            tma_store_3d(&ly.tmVd, vt, 0, row0, (int)uu);
            tma_store_3d(&ly.tmVd, vt + kBox, 64, row0, (int)uu);
            bulk_commit_wait_read();
          }
          fence_after();
          const uint32_t pb = sbase + C::OFF_P + b * C::kPBytes;
#pragma unroll
          for (int kk = 0; kk < KT / 16; ++kk) {
            // 16 keys = two 8-key groups of 256 B (SBO); 16-query blocks kPBlock apart (LBO)
            umma_f16(tmem + C::TM_O, sdesc(vt + kk * 2048, kBox, 1024),
                     sdesc_sw32(pb + kk * 512, C::kPBlock, 256), IPV, (k > 0 || kk > 0) ? 1u : 0u);
          }
          TRACE(7, tc);
          umma_commit(PEMPTY(b));
          umma_commit(EMPTYV(vs));
          if (++vs == C::VS) { vs = 0; vph ^= 1; }
        }
        umma_commit(ODONE);
        tcount += n;
        i = iend;
      }
      if (p.cor) bulk_wait_all();
    }
  } else {
    // ------------------------------------------------ softmax + epilogue
    const int h = (warp - 2) >> 2;        // column group: columns h*NH .. +NH
    const int q = warp & 3;               // TMEM lane quadrant: keys / dims 32q .. +31
    const int kl = q * 32 + lane;         // this thread's key (in a tile) / dim (in O^T)
    const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
    const int stid = threadIdx.x - 64;
    float* red = reinterpret_cast<float*>(smem + C::OFF_RED) + h * 4 * NH;   // [4][NH]
    float* sums = reinterpret_cast<float*>(smem + C::OFF_SUM) + h * 4 * NH;  // [4][NH]
    // per version: m (true running max), m or 0 (exponent offset), m + 8 (threshold)
    float* msm = reinterpret_cast<float*>(smem + C::OFF_M) + h * 2 * 3 * NH;
    float* asm_ = reinterpret_cast<float*>(smem + C::OFF_A) + h * NH;        // rescale factors
    int* lim = reinterpret_cast<int*>(smem + C::OFF_LIM) + h * NH;           // keys < lim visible
    uint32_t* qmk = reinterpret_cast<uint32_t*>(smem + C::OFF_QM) + h * NH;  // + these drafts
    // P^T (MN-major SWIZZLE_32B) address of key kl's 8-query chunk e:
    //   (e/2)*kPBlock + (kl/8)*256 + (kl%8)*32 + (((e&1) ^ bit2(kl)) << 4);
    // the 8 lanes of a store phase cover all 32 banks
    const uint32_t pkey = (uint32_t)(kl >> 3) * 256u + (uint32_t)(kl & 7) * 32u;
    const uint32_t pswz = (uint32_t)(kl >> 2) & 1u;
    auto paddr = [&](int e) -> uint32_t {
      return (uint32_t)(e >> 1) * C::kPBlock + pkey + ((((uint32_t)e & 1u) ^ pswz) << 4);
    };
    // Q rows of the item starting at tile x0 (zero beyond M) into Q buffer qb
    auto load_q = [&](long long x0, int qb) {
      const long long guq = x0 / p.tpu;
      const __nv_bfloat16* Qs = p.lay[MAXL == 1 ? 0 : (int)(guq / p.U)].Q;
      const long long uq = guq % p.U;
      const int bq = (int)(uq / p.H_kv), gq = (int)(uq % p.H_kv);
      const size_t r0 = ((size_t)bq * p.H_q + (size_t)gq * p.G) * p.t;
      for (int x = stid; x < N * 16; x += C::kSoftmax) {
        const int m = x >> 4, c = x & 15;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (m < p.M) v = *reinterpret_cast<const uint4*>(Qs + (r0 + m) * D + c * 8);
        const uint32_t off = (uint32_t)qb * C::kQBytes + (uint32_t)(c >> 3) * C::kQAtom +
                             (uint32_t)m * 128 + ((((uint32_t)c & 7u) ^ ((uint32_t)m & 7u)) << 4);
        *reinterpret_cast<uint4*>(smem + C::OFF_Q + off) = v;
      }
      fence_proxy_smem();
      mbar_arrive(QFULL(qb));
    };
    uint32_t oph = 0;
    long long i = t_begin;
    int tcount = 0, item = 0;
    if (!C::QTMA && i < t_end) load_q(i, 0);
    while (i < t_end) {
      const long long gu = i / p.tpu;                // global unit: layer * U + unit
      const long long iend = min(t_end, (gu + 1) * p.tpu);
      const LayerP& ly = p.lay[MAXL == 1 ? 0 : (int)(gu / p.U)];
      const long long u = gu % p.U;
      const int b_ = (int)(u / p.H_kv), g_ = (int)(u % p.H_kv);
      const int j0 = (int)(i % p.tpu);
      const size_t qrow0 = ((size_t)b_ * p.H_q + (size_t)g_ * p.G) * p.t;   // first query row
      // prefetch the next item's Q into the other buffer once the S^T MMAs of
      // the item before this one are done with it
      if (!C::QTMA && iend < t_end) {
        if (item >= 1) mbar_wait(QDONE((item - 1) & 1), ((item - 1) >> 1) & 1);
        load_q(iend, (item + 1) & 1);
      }
      const int vb_ = p.valid[b_];
      // per-column state of this half, written by the half's quadrant-0 warp
      // (ordered before its first use by the first tile's barrier-reduction):
      // running max (version 0) = -inf, visibility rule (chain: keys < valid_b
      // + tau; tree: committed keys + the node's ancestors)
      int mv = 0;                          // current version of msm
      if (q == 0) {
        for (int c = lane; c < NH; c += 32) {
          const int m = h * NH + c;
          const int tau = m % p.t;
          msm[c] = -INFINITY;
          msm[NH + c] = 0.f;
          msm[2 * NH + c] = -INFINITY;
          lim[c] = m < p.M ? vb_ + (p.tree ? 0 : tau) : INT_MIN;
          qmk[c] = (m < p.M && p.tree && tau > 0) ? p.anc[tau - 1] : 0u;
        }
      }
      half_sync(h);
      float2 l2[NH / 2];                   // this key lane's partial row sums
#pragma unroll
      for (int c = 0; c < NH / 2; ++c) l2[c] = make_float2(0.f, 0.f);
      const int n = (int)(iend - i);
      for (int k = 0; k < n; ++k) {
        const int tc = tcount + k;
        const int bb = tc % NB;
        const int pb = tc % C::NBP;
        const long long kidx = (long long)(j0 + k) * KT + kl;   // this thread's key row
        if (stid == 0) TRACE(8, tc);
        mbar_wait(SFULL(bb), (tc / NB) & 1);
        if (stid == 0) TRACE(9, tc);
        fence_after();
        float x[NH];
        tmem_ld_cols<NH>(tmem + bb * N + h * NH + lane_addr, x);
        fence_before();
        mbar_arrive(SEMPTY(bb));
        // log2 scaling and mask.  Tiles inside the committed rows need no mask
        // (padding columns have Q = 0: finite scores in outputs nobody
        // reads); the (at most two per item) tiles reaching past them build
        // the per-column visibility in a compact loop (cold code stays small:
        // an instruction-cache miss costs an L2 round trip under full HBM load)
        const float2 qs2 = make_float2(p.qscale, p.qscale);
#pragma unroll
        for (int c = 0; c < NH; c += 2) {
          const float2 y = __fmul2_rn(make_float2(x[c], x[c + 1]), qs2);
          x[c] = y.x;
          x[c + 1] = y.y;
        }
        if ((long long)(j0 + k + 1) * KT > vb_) {
          const long long js = kidx - vb_;
          uint64_t vm = 0;
#pragma unroll 8
          for (int c = 0; c < NH; ++c) {
            const uint32_t qm = qmk[c];
            const bool v = kidx < (long long)lim[c] || (js >= 0 && js < 32 && ((qm >> js) & 1u));
            vm |= (uint64_t)v << c;
          }
#pragma unroll
          for (int c = 0; c < NH; ++c) x[c] = ((vm >> c) & 1ull) ? x[c] : -INFINITY;
        }
        const float* mthr = msm + mv * 3 * NH + 2 * NH;
        bool need = false;
#pragma unroll
        for (int c0 = 0; c0 < NH; c0 += 4) {
          float mr[4];
          *reinterpret_cast<float4*>(mr) = *reinterpret_cast<const float4*>(mthr + c0);
#pragma unroll
          for (int e = 0; e < 4; ++e) need |= x[c0 + e] > mr[e];
        }
        const bool any_ = half_any(h, need);
        if (stid == 0) TRACE(10, tc);
        if (any_) {
          // column maxima of this tile over the half's 4 warps
#pragma unroll
          for (int c = 0; c < NH; ++c) {
            const float wm = warp_max(x[c]);
            if (lane == 0) red[q * NH + c] = wm;
          }
          half_sync(h);
          // the quadrant-0 warp moves the running maxima into the other
          // version (readers of the current one are ordered by the barriers)
          if (q == 0) {
            const float* mold = msm + mv * 3 * NH;   // quadrant maxima of this group: red[4][NH]
            float* mnew = msm + (mv ^ 1) * 3 * NH;
            bool resc = false;
            for (int c = lane; c < NH; c += 32) {
              const float mt =
                  fmaxf(fmaxf(red[c], red[NH + c]), fmaxf(red[2 * NH + c], red[3 * NH + c]));
              const float mo = mold[c];
              float mnx = mo, alpha = 1.f;
              if (mt > mo + kRescale) {
                alpha = (mo == -INFINITY) ? 0.f : fast_exp2(mo - mt);
                mnx = mt;
                resc |= (mo != -INFINITY);
              }
              mnew[c] = mnx;
              mnew[NH + c] = mnx == -INFINITY ? 0.f : mnx;
              mnew[2 * NH + c] = mnx + kRescale;
              asm_[c] = alpha;
            }
            resc = __any_sync(0xffffffffu, resc);
            if (lane == 0) resc_flag[h] = resc;
          }
          half_sync(h);
          mv ^= 1;
#pragma unroll
          for (int c0 = 0; c0 < NH; c0 += 4) {
            const float4 a4 = *reinterpret_cast<const float4*>(asm_ + c0);
            l2[c0 / 2] = __fmul2_rn(l2[c0 / 2], make_float2(a4.x, a4.y));
            l2[c0 / 2 + 1] = __fmul2_rn(l2[c0 / 2 + 1], make_float2(a4.z, a4.w));
          }
          // O^T columns of this half (rows = dims of this quadrant) are
          // rescaled once the previous tile's O^T MMAs have completed
          if (resc_flag[h] && k > 0) {
            const int tp = tc - 1;
            mbar_wait(PEMPTY(tp % C::NBP), (tp / C::NBP) & 1);
            fence_after();
#pragma unroll 1
            for (int cc = 0; cc < 2 * NH; cc += C::CS) {
              const int hl = cc >= NH, c0 = cc - hl * NH;
              float ov[C::CS];
              const uint32_t ta = tmem + C::TM_O + hl * NS + h * NH + c0 + lane_addr;
              tmem_ld_cols<C::CS>(ta, ov);
#pragma unroll
              for (int e = 0; e < C::CS; ++e) ov[e] *= asm_[c0 + e];
              tmem_st_cols<C::CS>(ta, ov);
            }
            fence_before();
          }
        }
        // P = 2^(x - m) and its bf16 hi / lo halves, packed two queries per
        // word, before waiting for the P^T buffer (overlaps the previous
        // tile's O^T MMAs)
        const float* msf = msm + mv * 3 * NH + NH;   // m, or 0 while m = -inf (then x = -inf)
        uint32_t phi[NH / 2], plo[NH / 2];
#pragma unroll
        for (int c0 = 0; c0 < NH; c0 += 4) {
          float mr[4];
          *reinterpret_cast<float4*>(mr) = *reinterpret_cast<const float4*>(msf + c0);
#pragma unroll
          for (int e = 0; e < 4; e += 2) {
            const int c = c0 + e;
            const float2 d = __fadd2_rn(make_float2(x[c], x[c + 1]), make_float2(-mr[e], -mr[e + 1]));
            const float2 pv = make_float2(fast_exp2(d.x), fast_exp2(d.y));
            l2[c / 2] = __fadd2_rn(l2[c / 2], pv);
            const uint32_t bx = __float_as_uint(pv.x), by = __float_as_uint(pv.y);
            phi[c / 2] = __byte_perm(bx, by, 0x7632);          // upper halves: bf16 hi (truncated)
            const float2 lo = __fadd2_rn(pv, make_float2(-__uint_as_float(bx & 0xffff0000u),
                                                          -__uint_as_float(by & 0xffff0000u)));
            const __nv_bfloat162 lb = __floats2bfloat162_rn(lo.x, lo.y);
            plo[c / 2] = *reinterpret_cast<const uint32_t*>(&lb);
          }
        }
        // P^T[pb] was last read by the O^T MMAs of tile tc - NBP
        if (stid == 0) TRACE(11, tc);
        if (tc >= C::NBP) mbar_wait(PEMPTY(pb), ((tc / C::NBP) - 1) & 1);
        if (stid == 0) TRACE(12, tc);
        const uint32_t pbase = sbase + C::OFF_P + pb * C::kPBytes;
        if constexpr (NH % 8 == 0) {
#pragma unroll
          for (int e = 0; e < NH / 8; ++e) {
            const int eh = h * (NH / 8) + e;             // hi chunk; lo chunks follow N / 8 later
            sts_v4(pbase + paddr(eh), phi[4 * e], phi[4 * e + 1], phi[4 * e + 2], phi[4 * e + 3]);
            sts_v4(pbase + paddr(eh + NS / 8), plo[4 * e], plo[4 * e + 1], plo[4 * e + 2],
                   plo[4 * e + 3]);
          }
        } else {   // groups of 4 queries: 8-byte halves of the 16-byte chunks
#pragma unroll
          for (int e = 0; e < NH / 4; ++e) {
            const int col = h * NH + 4 * e;
            const uint32_t half = (uint32_t)((col >> 2) & 1) * 8u;
            sts_v2(pbase + paddr(col >> 3) + half, phi[2 * e], phi[2 * e + 1]);
            sts_v2(pbase + paddr((col >> 3) + NS / 8) + half, plo[2 * e], plo[2 * e + 1]);
          }
        }
        fence_proxy_smem();
        mbar_arrive(PFULL(pb));
        if (stid == 0) TRACE(13, tc);
      }
      // ---- epilogue of this item: column sums, O^T (TMEM) -> output / record
#pragma unroll
      for (int c = 0; c < NH; ++c) {
        const float ws_ = warp_sum((c & 1) ? l2[c / 2].y : l2[c / 2].x);
        if (lane == 0) sums[q * NH + c] = ws_;
      }
      if (stid == 0) TRACE(14, tcount);
      mbar_wait(ODONE, oph);
      oph ^= 1;
      if (stid == 0) TRACE(15, tcount);
      fence_after();
      half_sync(h);
      const long long ufirst = gu * p.tpu, ulast = ufirst + p.tpu - 1;
      const int c_lo = cta_of_tile(ufirst, NT, p.ctas);
      const int c_hi = cta_of_tile(ulast, NT, p.ctas);
      const int nseg = c_hi - c_lo + 1;
      const size_t rec = rec_floats(p.M, D);
      float* my = ly.ws + ((size_t)blockIdx.x * 2 + (item == 0 ? 0 : 1)) * rec;
      const float* mfin = msm + mv * 3 * NH;
#pragma unroll 1
      for (int c0 = 0; c0 < NH; c0 += C::CS) {
        float o_hi[C::CS], o_lo[C::CS];
        tmem_ld_cols<C::CS>(tmem + C::TM_O + h * NH + c0 + lane_addr, o_hi);
        tmem_ld_cols<C::CS>(tmem + C::TM_O + NS + h * NH + c0 + lane_addr, o_lo);
#pragma unroll
        for (int e = 0; e < C::CS; ++e) {
          const int c = c0 + e;
          const int m = h * NH + c;
          if (m < p.M) {
            const float L = (sums[c] + sums[NH + c]) + (sums[2 * NH + c] + sums[3 * NH + c]);
            const float o = o_hi[e] + o_lo[e];
            if (nseg == 1) {
              ly.O[(qrow0 + m) * D + kl] = o / L;
            } else {
              my[(size_t)m * D + kl] = o;
              if (kl == 0) {
                my[(size_t)p.M * D + m] = mfin[c];
                my[(size_t)p.M * D + p.M + m] = L;
              }
            }
          }
        }
      }
      fence_before();
      if (nseg > 1) {
        __threadfence();
        softmax_sync<C::kSoftmax>();
        if (stid == 0) {
          const int old = atomicAdd(&ly.counters[u], 1);
          *sm_flag = (old == nseg - 1);
        }
        softmax_sync<C::kSoftmax>();
        if (*sm_flag) {
          __threadfence();
          // scratch: the P^T buffers (every O^T MMA of this item has completed)
          combine_unit<4>(ly.ws, rec, c_lo, c_hi, ufirst, NT, p.ctas, p.M, D, ly.O + qrow0 * D,
                          reinterpret_cast<float*>(smem + C::OFF_P), stid, C::kSoftmax,
                          [] { softmax_sync<C::kSoftmax>(); });
          if (stid == 0) ly.counters[u] = 0;
        }
      }
      softmax_sync<C::kSoftmax>();   // sums / column state / flag reuse by the next item
      if (stid == 0) TRACE(14, tcount + 1);
      tcount += n;
      ++item;
      i = iend;
    }
  }
  fence_before();
  __syncthreads();
  fence_after();
#ifdef BMC_TC_TRACE
  if (threadIdx.x == 0) { g_tck_cta[blockIdx.x][2] = clk(); g_tck_cta[blockIdx.x][3] = gtime(); }
#endif
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(C::kTmemCols));
  }
}

}  // namespace tck

// ------------------------------------------------------------------ host

#ifdef BMC_TC_TRACE
extern "C" int bmc_tck_trace_cta(int c) {
  return cudaMemcpyToSymbol(tck::g_tck_trace_cta, &c, sizeof(int)) == cudaSuccess ? 0 : -1;
}
extern "C" int bmc_tck_trace(long long* out) {   // [16][256] tile events, then [160][4] CTAs
  if (cudaMemcpyFromSymbol(out, tck::g_tck_trace, sizeof(long long) * 16 * 256) != cudaSuccess)
    return -1;
  return cudaMemcpyFromSymbol(out + 16 * 256, tck::g_tck_cta, sizeof(long long) * 160 * 4) ==
                 cudaSuccess ? 0 : -1;
}
#endif

// L2 prefetch distance (tiles ahead of the ring's loads) unless overridden
// with BMC_OPT_TCK_PREFETCH
static constexpr int kDefaultPrefetch = 0;

bool attn_tck_supported(int D, int dtype, int M) {
  return D == 128 && dtype == BMC_BF16 && M >= 1 && M <= 80 && encode_fn() != nullptr;
}

template <int N, int MAXL, int NG, int NS = N>
static cudaError_t launch_ng(const tck::Params<MAXL>& p, int ctas, cudaStream_t s) {
  using C = tck::Cfg<N, NG, NS>;
  static int attr_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_dev != dev) {
    cudaError_t e = cudaFuncSetAttribute(tck::attn_tck_kernel<N, MAXL, NG, NS>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)C::kSmem);
    if (e != cudaSuccess) return e;
    attr_dev = dev;
  }
  tck::attn_tck_kernel<N, MAXL, NG, NS><<<ctas, C::kThreads, C::kSmem, s>>>(p);
  count_launch();
  return cudaGetLastError();
}
// softmax column groups: 4 (640 threads) for N = 32 ... 64, else 2 (measured
// on the 70B shape, tools/microbench.py --what tcgroups: +1..7% at M = 32..64;
// at N = 80 the 96-register budget of 640 threads spills, at N = 16 the
// groups are too narrow); groups != 0 forces (BMC_OPT_TCK_GROUPS, A/B runs)
template <int N, int MAXL>
static cudaError_t launch_n(const tck::Params<MAXL>& p, int ctas, cudaStream_t s, int groups) {
  const int ng = groups ? groups : ((N >= 32 && N <= 64) ? 4 : 2);
  return ng == 4 ? launch_ng<N, MAXL, 4>(p, ctas, s) : launch_ng<N, MAXL, 2>(p, ctas, s);
}

// Tensor maps are pure functions of (base, rows): cache them so a fused
// 32-layer step does not re-encode 64 maps on the host every token.
// units > 0: the 3D [units][rows][128] map of a copy-on-read launch.
static cudaError_t cached_map(CUtensorMap* m, const void* base, long long rows,
                              long long units = 0, int box_rows = tck::KT) {
  struct Key {
    const void* base;
    long long rows, units;
    int box;
    bool operator==(const Key& o) const {
      return base == o.base && rows == o.rows && units == o.units && box == o.box;
    }
  };
  // splitmix64-mixed fields: the earlier XOR of (address, rows * 31, ...)
  // collided for whole families of keys (4 KiB-aligned buffer addresses and
  // capacities in steps of 128 rows), so lookups walked long bucket chains
  struct Hash {
    static uint64_t mix(uint64_t x) {
      x += 0x9e3779b97f4a7c15ull;
      x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
      x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
      return x ^ (x >> 31);
    }
    size_t operator()(const Key& k) const {
      uint64_t h = mix((uint64_t)(uintptr_t)k.base);
      h = mix(h ^ (uint64_t)k.rows);
      h = mix(h ^ (uint64_t)k.units);
      return (size_t)mix(h ^ (uint64_t)k.box);
    }
  };
  static thread_local std::unordered_map<Key, CUtensorMap, Hash> cache;
  const Key k{base, rows, units, box_rows};
  auto it = cache.find(k);
  if (it != cache.end()) {
    *m = it->second;
    return cudaSuccess;
  }
  cudaError_t e = units > 0 ? make_map3(m, base, units, rows, box_rows)
                            : make_map(m, base, rows, box_rows);
  if (e != cudaSuccess) return e;
  if (cache.size() > 4096) cache.clear();
  cache.emplace(k, *m);
  return cudaSuccess;
}

template <int MAXL>
static cudaError_t launch_layers(const AttnStepArgs& a, int l0, int nl, int num_sms,
                                 cudaStream_t s) {
  tck::Params<MAXL> p;
  const AttnLayer& h0 = a.layers[l0];
  const long long U = (long long)a.B * a.H_kv;
  p.cor = h0.Ksrc != nullptr;
  for (int l = 0; l < nl; ++l) {
    const AttnLayer& h = a.layers[l0 + l];
    if (h.cap != h0.cap || h.scan != h0.scan || h.n_app != h0.n_app ||
        h.n_draft != h0.n_draft || h.kd_stride != h0.kd_stride ||
        (h.Ksrc != nullptr) != (p.cor != 0) || h.cap_src != h0.cap_src)
      return cudaErrorInvalidValue;   // the caller launches such layers one by one
    if (p.cor && ((h.scan > 0 && h.scan < h.cap) || h.rows_src != h.cap_src))
      return cudaErrorInvalidValue;   // copy-on-read streams every row of the old buffer
    tck::LayerP& ly = p.lay[l];
    cudaError_t e;
    if (p.cor) {
      e = cached_map(&ly.tmK, h.Ksrc, h.cap_src, U);
      if (e == cudaSuccess) e = cached_map(&ly.tmV, h.Vsrc, h.cap_src, U);
      if (e == cudaSuccess) e = cached_map(&ly.tmKd, h.K, h.cap, U);
      if (e == cudaSuccess) e = cached_map(&ly.tmVd, h.V, h.cap, U);
    } else {
      e = cached_map(&ly.tmK, h.K, U * h.cap);
      if (e == cudaSuccess) e = cached_map(&ly.tmV, h.V, U * h.cap);
    }
    if (e != cudaSuccess) return e;
    // Q rows by TMA (the M = 72 verify variant, box of 80 rows); Q is never
    // written by the library, so the map is keyed on the caller's pointer
    if (e == cudaSuccess && a.H_q / a.H_kv * a.t > 64 && a.H_q / a.H_kv * a.t <= 72)
      e = cached_map(&ly.tmQ, h.Q, (long long)a.B * a.H_q * a.t, 0, 80);
    if (e != cudaSuccess) return e;
    ly.Q = (const __nv_bfloat16*)h.Q;
    ly.O = h.O;
    ly.Knew = (const uint8_t*)h.Knew;
    ly.Vnew = (const uint8_t*)h.Vnew;
    ly.Kd = (const uint8_t*)h.Kd;
    ly.Vd = (const uint8_t*)h.Vd;
    ly.Kc = (uint8_t*)h.K;
    ly.Vc = (uint8_t*)h.V;
    ly.ws = h.ws;
    ly.counters = h.counters;
  }
  p.L = nl;
  p.n_app = h0.n_app;
  p.n_draft = h0.n_draft;
  p.kd_stride = h0.kd_stride;
  p.cap = h0.cap;
  p.tpu = (int)(((h0.scan > 0 ? h0.scan : h0.cap) + tck::KT - 1) / tck::KT);
  p.U = (int)U;
  p.total_tiles = (long long)nl * U * p.tpu;
  p.H_kv = a.H_kv;
  p.H_q = a.H_q;
  p.G = a.H_q / a.H_kv;
  p.t = a.t;
  p.M = p.G * a.t;
  p.qscale = tck::kLog2e / sqrtf((float)tck::D);
  p.tree = a.tree;
  p.pf = a.tck_prefetch >= 0 ? a.tck_prefetch : kDefaultPrefetch;
  for (int i = 0; i < 32; ++i) p.anc[i] = a.anc[i];
  for (int b = 0; b < a.B; ++b) p.valid[b] = a.valid[b];
  int ctas = a.ctas > 0 ? a.ctas : num_sms;
  if (ctas > p.total_tiles) ctas = (int)p.total_tiles;
  p.ctas = ctas;
  if (p.total_tiles == 0) return cudaSuccess;
  if constexpr (MAXL > 1) {   // multi-layer launches: GQA decode and speculative steps
    if (p.M <= 16) return launch_n<16, MAXL>(p, ctas, s, a.tck_groups);
    if (p.M <= 32) return launch_n<32, MAXL>(p, ctas, s, a.tck_groups);
    if (p.M <= 48) return launch_n<48, MAXL>(p, ctas, s, a.tck_groups);
    if (p.M <= 64) return launch_n<64, MAXL>(p, ctas, s, a.tck_groups);
    if (p.M <= 72)   // 64 < M <= 72: the 70B verify tile (3 softmax groups; 2 for A/B)
      return a.tck_groups == 2 ? launch_ng<80, MAXL, 2, 72>(p, ctas, s)
                               : launch_ng<80, MAXL, 3, 72>(p, ctas, s);
    return launch_n<80, MAXL>(p, ctas, s, a.tck_groups);
  } else {
    if (p.M <= 16) return launch_n<16, 1>(p, ctas, s, a.tck_groups);
    if (p.M <= 32) return launch_n<32, 1>(p, ctas, s, a.tck_groups);
    if (p.M <= 48) return launch_n<48, 1>(p, ctas, s, a.tck_groups);
    if (p.M <= 64) return launch_n<64, 1>(p, ctas, s, a.tck_groups);
    if (p.M <= 72)   // 64 < M <= 72: the 70B verify tile (3 softmax groups; 2 for A/B)
      return a.tck_groups == 2 ? launch_ng<80, 1, 2, 72>(p, ctas, s)
                               : launch_ng<80, 1, 3, 72>(p, ctas, s);
    return launch_n<80, 1>(p, ctas, s, a.tck_groups);
  }
}

cudaError_t launch_attn_tck(const AttnStepArgs& a, int num_sms, cudaStream_t s) {
  if (a.L == 1) return launch_layers<1>(a, 0, 1, num_sms, s);
  for (int l0 = 0; l0 < a.L; l0 += kMaxLayersPerLaunch) {
    const int nl = a.L - l0 < kMaxLayersPerLaunch ? a.L - l0 : kMaxLayersPerLaunch;
    cudaError_t e = launch_layers<kMaxLayersPerLaunch>(a, l0, nl, num_sms, s);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace bmc
