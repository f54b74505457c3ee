// bmc_internal.h -- internal interfaces between the C-ABI state machine
// (bmc_abi.cpp), the chunk-growth arena (arena.cpp) and the sm_100a kernels
// (bmc_kernels.cu, attn_decode.cu).  Not part of the public ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/bmc.h"

namespace bmc {

// ---------------------------------------------------------------- kernels
// Every launcher returns the cudaError_t of its launch and bumps the global
// launch counter.

struct ReallocArgs {
  const void* src_k; const void* src_v;   // [U][cap_old][D] (may be null if copy_rows == 0)
  void* dst_k; void* dst_v;               // [U][cap_new][D]
  long long U;
  long long cap_old, cap_new;             // rows
  long long copy_rows;                    // rows [0, copy_rows) copied, rest zeroed
  int row_bytes;                          // D * element size, multiple of 16
};
cudaError_t launch_realloc_copy_zero(const ReallocArgs& a, cudaStream_t s);

struct RowsArgs {
  const void* src_k; const void* src_v;   // [B][H_kv][nsrc][D]
  void* dst_k; void* dst_v;               // [U][cap][D]
  int B, H_kv, nsrc, nwrite;              // write rows i < nwrite of the source
  long long cap;
  int row_bytes;
  int row0[BMC_MAX_B];                    // destination row of source row 0, per batch row
};
cudaError_t launch_write_rows(const RowsArgs& a, cudaStream_t s);

constexpr int kMaxZeroLayers = 32;
struct ZeroArgs {
  void* k[kMaxZeroLayers];                // per layer [U][cap][D] (L layers of one shape)
  void* v[kMaxZeroLayers];
  int L;
  int B, H_kv;
  long long cap;
  int row_bytes;
  int row_lo[BMC_MAX_B], row_hi[BMC_MAX_B];   // zero rows [lo, hi) of batch row b
  int max_rows;                           // max(hi - lo)
};
cudaError_t launch_zero_rows(const ZeroArgs& a, cudaStream_t s);

struct PathArgs {
  void* k[kMaxZeroLayers];                // per layer [U][cap][D] (L layers of one shape)
  void* v[kMaxZeroLayers];
  int L;
  int B, H_kv, staged;
  long long cap;
  int row_bytes;
  int valid[BMC_MAX_B];                   // committed rows before the commit
  unsigned char m[BMC_MAX_B];             // accepted path length per batch row
  unsigned char path[BMC_MAX_B][32];      // accepted node indices, root first
};
// Compact the accepted tree path of every unit behind its committed rows and
// zero the remaining staged rows (one warp per (unit, tensor, layer)).
cudaError_t launch_commit_path(const PathArgs& a, cudaStream_t s);

// One layer of an attention launch.
struct AttnLayer {
  const void* K; const void* V;           // cache [U][cap][D]
  // copy-on-read growth (CUDA-core kernel only): old buffer [U][cap_src][D]
  // whose first rows_src rows per unit the attention copies into K / V while
  // streaming them (null: no growth pending)
  const void* Ksrc = nullptr; const void* Vsrc = nullptr;
  long long cap_src = 0, rows_src = 0;
  const void* Q;                          // [B][H_q][t][D]
  float* O;                               // [B][H_q][t][D]
  const void* Knew; const void* Vnew;     // pending appended row [B][H_kv][D] (n_app = 1)
  const void* Kd; const void* Vd;         // pending drafts [B][H_kv][kd_stride][D]
  float* ws;                              // partial records
  int* counters;                          // [U], zero between launches
  long long cap;
  long long scan;                         // rows to stream per unit (0 = cap)
  int n_app, n_draft, kd_stride;
};
constexpr int kMaxLayersPerLaunch = 32;
struct AttnStepArgs {
  int B, H_kv, H_q, D, t, dtype;
  int ctas;                               // 0 = auto
  int tree;                               // staged rows form a token tree
  int tck_groups = 0;                     // keys-on-lanes kernel softmax groups (0 auto, 2, 3, 4)
  int tck_prefetch = -1;                  // keys-on-lanes kernel L2 prefetch distance (-1 auto)
  uint32_t anc[32];                       // tree: bit j of anc[i] = node j is i or an ancestor
  int valid[BMC_MAX_B];                   // committed rows incl. the pending append
  int L;
  const AttnLayer* layers;
};
size_t attn_workspace_floats(int M, int D, int max_ctas);
// floats of one split-K partial record (M rows of o[D], then M maxima and M
// sums), rounded up to 16 bytes so every record starts 16-byte aligned
__host__ __device__ inline size_t rec_floats(int M, int D) {
  return ((size_t)M * (D + 2) + 3) / 4 * 4;
}
// Masked SDPA of L layers in one persistent launch (per 32 layers), with the
// pending appended / drafted rows written into each cache on the way.
cudaError_t launch_attn_step(const AttnStepArgs& a, int num_sms, cudaStream_t s);
// tcgen05 verify attention (single layer, bf16, D = 128, M = G*t <= 128);
// writes the layer's pending rows into the cache itself, like attn_step.
bool attn_tc_supported(int D, int dtype, int M);
cudaError_t launch_attn_tc(const AttnStepArgs& a, int num_sms, cudaStream_t s);
// tcgen05 attention with the keys on the TMEM lanes (attn_tck.cu; bf16,
// D = 128, M = G*t <= 80): the default tensor-core kernel up to M = 80.
bool attn_tck_supported(int D, int dtype, int M);
cudaError_t launch_attn_tck(const AttnStepArgs& a, int num_sms, cudaStream_t s);

void count_launch();
unsigned long long launch_count();
// Host-time diagnostics (bmc_host_profile): nanoseconds and calls per category
enum HostCat { kHostAlloc = 0, kHostRelease, kHostLaunch, kHostPremap, kHostSyncMap, kHostCats };
void host_time_add(int cat, long long ns);
void host_time_read(long long* ns, long long* calls, bool reset);
long long host_now_ns();

// ------------------------------------------------------------------ arena
// Chunk-growth allocator: each handle owns one arena with two ping-pong
// slots of reserved virtual address space per tensor; physical 2 MiB
// granules come from a process-wide pool and are mapped on growth.
struct Arena;
struct Buffer {
  void* ptr = nullptr;
  size_t bytes = 0;
  int slot = -1;        // arena slot (VMM) or region end, -1 = pool allocation
  int kind = 0;         // 0 VMM, 1 pool, 2 two-ended region
};
Arena* arena_create(int device, size_t max_bytes_per_tensor, int* err);
int pool_reserve(int device, size_t bytes);
int pool_trim(int device);
// (Re)create the device's two-ended growth region of `bytes` (0: free it);
// STATE while buffers of the old region are live.
int region_reserve(int device, size_t bytes);
bool region_present(int device);
// Obtain a buffer of `bytes` for tensor (0 = K, 1 = V) in the slot not
// holding `keep` (the tensor's live buffer).  kind 0 = VMM slot, 1 =
// stream-ordered pool allocation (also the fallback when VMM is unsupported),
// 2 = the end of the growth region opposite to `keep` (pool when full).
int arena_alloc(Arena* a, int tensor, size_t bytes, int kind, const Buffer* keep,
                cudaStream_t s, Buffer* out);
// Release a buffer once all work enqueued so far on s has finished with it.
int arena_release(Arena* a, Buffer* b, cudaStream_t s);
// VMM arenas: map (on a helper thread, asynchronously) the physical chunks a
// future arena_alloc of `bytes` for tensor will need in the slot that is not
// live; a no-op for pool arenas or when already mapped.
int arena_premap(Arena* a, int tensor, size_t bytes);
void arena_destroy(Arena* a);

// 0 device / managed, 1 page-locked host, 2 pageable host (cached by range).
int pointer_kind(const void* p);
// Drop a cached device range (its memory is being freed or unmapped).
void forget_range(const void* p);

}  // namespace bmc
