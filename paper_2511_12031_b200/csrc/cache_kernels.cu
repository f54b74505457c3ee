#include <chrono>
// cache_kernels.cu -- KV-cache update kernels of the BMC hot path (sm_100a).
//
//   realloc_copy_zero : the BMC growth step: for every
//       (batch, kv-head) unit copy rows [0, copy_rows) from the old slab
//       (stride cap_old rows) to the new slab (stride cap_new rows) and zero
//       rows [copy_rows, cap_new).  Pure HBM move: 128-bit coalesced loads
//       and stores, 4 independent 16-byte loads in flight per thread.
//   write_rows        : in-place append of the new K/V rows
//       and placement of speculative drafts in the padded rows.
//   zero_rows         : rollback of rejected drafts after a commit (
//       reading R9 re-zeroes them).
//
// Cache layout: [U = B*H_kv][cap][D], element bytes 2 (bf16) or 4 (fp32);
// every row is D*eb bytes, a multiple of 16.
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#include "bmc_internal.h"

namespace bmc {

static std::atomic<unsigned long long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
static std::atomic<long long> g_host_ns[kHostCats], g_host_calls[kHostCats];
void host_time_add(int cat, long long ns) {
  g_host_ns[cat].fetch_add(ns, std::memory_order_relaxed);
  g_host_calls[cat].fetch_add(1, std::memory_order_relaxed);
}
void host_time_read(long long* ns, long long* calls, bool reset) {
  for (int i = 0; i < kHostCats; ++i) {
    ns[i] = reset ? g_host_ns[i].exchange(0) : g_host_ns[i].load();
    calls[i] = reset ? g_host_calls[i].exchange(0) : g_host_calls[i].load();
  }
}
long long host_now_ns() {
  return std::chrono::duration_cast<std::chrono::nanoseconds>(
             std::chrono::steady_clock::now().time_since_epoch()).count();
}
unsigned long long launch_count() { return g_launches.load(std::memory_order_relaxed); }

__device__ __forceinline__ int4 ld_stream(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ void st_stream(int4* p, int4 v) {
  asm volatile("st.global.L1::no_allocate.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

constexpr int kCopyThreads = 256;
constexpr int kCopyVPT = 4;  // 16-byte vectors per thread per block pass

// grid: x = vector blocks over one destination slab, y = unit, z = tensor (K/V)
__global__ void __launch_bounds__(kCopyThreads)
realloc_copy_zero_kernel(const int4* __restrict__ src_k, const int4* __restrict__ src_v,
                         int4* __restrict__ dst_k, int4* __restrict__ dst_v,
                         long long src_slab_vec, long long dst_slab_vec,
                         long long copy_vec) {
  const long long u = blockIdx.y;
  const int4* src = (blockIdx.z == 0 ? src_k : src_v) + u * src_slab_vec;
  int4* dst = (blockIdx.z == 0 ? dst_k : dst_v) + u * dst_slab_vec;
  const long long base = (long long)blockIdx.x * (kCopyThreads * kCopyVPT) + threadIdx.x;
  int4 v[kCopyVPT];
#pragma unroll
  for (int i = 0; i < kCopyVPT; ++i) {
    const long long e = base + (long long)i * kCopyThreads;
    v[i] = make_int4(0, 0, 0, 0);
    if (e < copy_vec) v[i] = ld_stream(src + e);
  }
#pragma unroll
  for (int i = 0; i < kCopyVPT; ++i) {
    const long long e = base + (long long)i * kCopyThreads;
    if (e < dst_slab_vec) st_stream(dst + e, v[i]);
  }
}

cudaError_t launch_realloc_copy_zero(const ReallocArgs& a, cudaStream_t s) {
  const long long row_vec = a.row_bytes / 16;
  const long long dst_slab = a.cap_new * row_vec;
  const long long per_block = (long long)kCopyThreads * kCopyVPT;
  dim3 grid((unsigned)((dst_slab + per_block - 1) / per_block), (unsigned)a.U, 2);
  if (grid.x == 0 || a.U == 0) return cudaSuccess;
  realloc_copy_zero_kernel<<<grid, kCopyThreads, 0, s>>>(
      (const int4*)a.src_k, (const int4*)a.src_v, (int4*)a.dst_k, (int4*)a.dst_v,
      a.cap_old * row_vec, dst_slab, a.copy_rows * row_vec);
  count_launch();
  return cudaGetLastError();
}

// One thread per 16-byte vector of (tensor, unit, source row, vector).
__global__ void write_rows_kernel(const RowsArgs a) {
  const int row_vec = a.row_bytes / 16;
  const long long per_tensor = (long long)a.B * a.H_kv * a.nwrite * row_vec;
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 2 * per_tensor) return;
  const int tensor = (int)(i / per_tensor);
  i -= tensor * per_tensor;
  const int vec = (int)(i % row_vec);
  long long r = i / row_vec;
  const int row = (int)(r % a.nwrite);
  const long long u = r / a.nwrite;
  const int b = (int)(u / a.H_kv);
  const int4* src = (const int4*)(tensor == 0 ? a.src_k : a.src_v);
  int4* dst = (int4*)(tensor == 0 ? a.dst_k : a.dst_v);
  const int4 val = src[(u * a.nsrc + row) * row_vec + vec];
  dst[(u * a.cap + a.row0[b] + row) * row_vec + vec] = val;
}

cudaError_t launch_write_rows(const RowsArgs& a, cudaStream_t s) {
  const long long total = 2LL * a.B * a.H_kv * a.nwrite * (a.row_bytes / 16);
  if (total == 0) return cudaSuccess;
  const int threads = 256;
  write_rows_kernel<<<(unsigned)((total + threads - 1) / threads), threads, 0, s>>>(a);
  count_launch();
  return cudaGetLastError();
}

// grid covers L layers x {K, V} x units x max_rows x 16-byte chunks
__global__ void zero_rows_kernel(const __grid_constant__ ZeroArgs a) {
  const int row_vec = a.row_bytes / 16;
  const long long per_tensor = (long long)a.B * a.H_kv * a.max_rows * row_vec;
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 2 * a.L * per_tensor) return;
  const int layer = (int)(i / (2 * per_tensor));
  i -= layer * 2 * per_tensor;
  const int tensor = (int)(i / per_tensor);
  i -= tensor * per_tensor;
  const int vec = (int)(i % row_vec);
  long long r = i / row_vec;
  const int row = (int)(r % a.max_rows);
  const long long u = r / a.max_rows;
  const int b = (int)(u / a.H_kv);
  const int lo = a.row_lo[b], hi = a.row_hi[b];
  if (lo + row >= hi) return;
  int4* dst = (int4*)(tensor == 0 ? a.k[layer] : a.v[layer]);
  dst[(u * a.cap + lo + row) * row_vec + vec] = make_int4(0, 0, 0, 0);
}

cudaError_t launch_zero_rows(const ZeroArgs& a, cudaStream_t s) {
  const long long total = 2LL * a.L * a.B * a.H_kv * a.max_rows * (a.row_bytes / 16);
  if (total == 0) return cudaSuccess;
  const int threads = 256;
  zero_rows_kernel<<<(unsigned)((total + threads - 1) / threads), threads, 0, s>>>(a);
  count_launch();
  return cudaGetLastError();
}

// One warp per (unit, tensor): rows are moved in depth order (path[i] >= i,
// so no destination is a row still to be read), then the rest is zeroed.
__global__ void commit_path_kernel(const __grid_constant__ PathArgs a) {
  const long long u = blockIdx.x;
  const int tensor = blockIdx.y;
  const int l = blockIdx.z;
  const int b = (int)(u / a.H_kv);
  const int lane = threadIdx.x;
  const int row_vec = a.row_bytes / 16;
  int4* base = (int4*)(tensor == 0 ? a.k[l] : a.v[l]) + (u * a.cap + a.valid[b]) * row_vec;
  const int m = a.m[b];
  for (int i = 0; i < m; ++i) {
    const int src = a.path[b][i];
    if (src != i)
      for (int c = lane; c < row_vec; c += 32) base[(long long)i * row_vec + c] = base[(long long)src * row_vec + c];
    __syncwarp();
  }
  for (int x = lane; x < (a.staged - m) * row_vec; x += 32)
    base[(long long)m * row_vec + x] = make_int4(0, 0, 0, 0);
}

cudaError_t launch_commit_path(const PathArgs& a, cudaStream_t s) {
  const long long U = (long long)a.B * a.H_kv;
  if (U == 0 || a.staged == 0 || a.L < 1) return cudaSuccess;
  commit_path_kernel<<<dim3((unsigned)U, 2, (unsigned)a.L), 32, 0, s>>>(a);
  count_launch();
  return cudaGetLastError();
}

}  // namespace bmc
