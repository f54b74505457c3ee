// arena.cpp -- chunk-growth allocator for the BMC KV cache.
//
// BMC reallocates every r tokens; the paper's implementation
// calls the framework allocator each time.  Here a handle
// (one layer) owns one Arena:
//   kind 0 (VMM): for each tensor (K, V) two ping-pong slots of reserved
//     virtual address space, each large enough for N_max rows.  A growth maps
//     only the physical chunks (cuMemCreate, from a process-wide pool) that
//     the slot not holding the live buffer still lacks, the realloc kernel
//     copies, and the old slot simply becomes the target of the next growth:
//     mappings persist, so a growth costs at most a few cuMemMap calls, never
//     an unmap or a host synchronisation.  The price is physical memory: both
//     slots stay mapped (about 2x the live cache), since all layers grow in
//     the same step and cannot lend chunks to each other.  Chunks return to
//     the pool when the handle is destroyed.  Virtual addresses of a handle
//     take only two values per tensor.
//     Growth is predictable (BMC: the next growth is r appends away and its
//     size is cap + r), so the caller asks for the NEXT growth's chunks right
//     after a growth (arena_premap): a process-wide helper thread creates and
//     maps them while the decode steps run, and the growth itself finds its
//     slot mapped -- cuMemCreate / cuMemMap / cuMemSetAccess (~2.5 ms per
//     layer-growth on B200) leave the host's critical path.
//   kind 1 (pool): cudaMallocFromPoolAsync / cudaFreeAsync on a per-device
//     memory pool with an unbounded release threshold (stream-ordered reuse).
//   kind 2 (region): a two-ended stack over one device region reserved up
//     front (region_reserve).  All layers of a model grow in the same step,
//     so a growth moves every buffer of a step to the end of the region
//     opposite to the one holding the buffers it replaces: the new buffers
//     are pushed onto that end, the old ones popped off the other end once
//     released.  The region never fragments and a growth is pointer
//     arithmetic (no driver call, no host wait), in a region of twice the
//     final cache (the peak of a copy growth: old and new buffers of every
//     layer of a step at once).  The stream-ordered pool and the VMM slots
//     stalled the host for up to ~1 s at some L3-8B growth steps (a
//     fragmented pool mapping memory and waiting for the device;
//     cuMemMap ~5 ms per chunk under full HBM load), profiles/
//     r02_growth_cost_l3.txt.  A request the region cannot hold falls back to
//     the pool.
#include <cstdlib>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <condition_variable>
#include <deque>
#include <map>
#include <mutex>
#include <set>
#include <thread>
#include <vector>

#include "bmc_internal.h"

namespace bmc {

namespace {

struct ChunkPool {
  int device = 0;
  size_t chunk = 0;
  std::vector<CUmemGenericAllocationHandle> free_list;
};

struct Slot {
  std::vector<CUmemGenericAllocationHandle> chunks;  // mapped, in address order
  cudaEvent_t pending = nullptr;                          // release requested, not yet reclaimed
};

// Driver entry points resolved through the runtime at first use, so that
// libbmc.so does not link libcuda.so.1 (it loads on machines without a GPU).
struct Driver {
  PFN_cuMemGetAllocationGranularity granularity = nullptr;
  PFN_cuMemAddressReserve reserve = nullptr;
  PFN_cuMemAddressFree addr_free = nullptr;
  PFN_cuMemCreate create = nullptr;
  PFN_cuMemMap map = nullptr;
  PFN_cuMemUnmap unmap = nullptr;
  PFN_cuMemSetAccess set_access = nullptr;
  PFN_cuDeviceGet device_get = nullptr;
  PFN_cuDeviceGetAttribute device_attr = nullptr;
  PFN_cuMemGetAddressRange range = nullptr;
  bool ok = false;
  bool tried = false;
};
Driver g_drv;

template <typename F>
bool resolve(const char* name, F* fn) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !p)
    return false;
  *fn = reinterpret_cast<F>(p);
  return true;
}

const Driver& drv() {
  if (!g_drv.tried) {
    g_drv.tried = true;
    g_drv.ok = resolve("cuMemGetAllocationGranularity", &g_drv.granularity) &&
               resolve("cuMemAddressReserve", &g_drv.reserve) &&
               resolve("cuMemAddressFree", &g_drv.addr_free) &&
               resolve("cuMemCreate", &g_drv.create) && resolve("cuMemMap", &g_drv.map) &&
               resolve("cuMemUnmap", &g_drv.unmap) &&
               resolve("cuMemSetAccess", &g_drv.set_access) &&
               resolve("cuDeviceGet", &g_drv.device_get) &&
               resolve("cuDeviceGetAttribute", &g_drv.device_attr) &&
               resolve("cuMemGetAddressRange", &g_drv.range);
  }
  return g_drv;
}

std::mutex g_mu;
std::map<std::pair<int, size_t>, ChunkPool*> g_pools;
std::map<int, cudaMemPool_t> g_mempools;
std::set<Arena*> g_arenas;

}  // namespace

struct Arena {
  std::mutex mu;          // slot mappings (the helper thread maps ahead)
  int device = 0;
  size_t slot_bytes = 0;  // reserved VA per slot (multiple of chunk)
  size_t chunk = 0;
  CUdeviceptr base = 0;
  Slot slots[2][2];       // [tensor][slot]
  int live[2] = {-1, -1}; // live VMM slot per tensor
  ChunkPool* pool = nullptr;
  bool vmm_ok = false;
};

static int cu_ok(CUresult r) { return r == CUDA_SUCCESS ? 0 : BMC_ERR_CUDA; }
static bool region_alloc(int device, size_t bytes, int pref, cudaStream_t s, Buffer* out);
static int region_release(int device, Buffer* b, cudaStream_t s);

static size_t round_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

static ChunkPool* pool_for(int device, size_t chunk) {
  auto key = std::make_pair(device, chunk);
  auto it = g_pools.find(key);
  if (it != g_pools.end()) return it->second;
  ChunkPool* p = new ChunkPool();
  p->device = device;
  p->chunk = chunk;
  g_pools[key] = p;
  return p;
}

static cudaMemPool_t mempool_for(int device) {
  auto it = g_mempools.find(device);
  if (it != g_mempools.end()) return it->second;
  cudaMemPoolProps props = {};
  props.allocType = cudaMemAllocationTypePinned;
  props.handleTypes = cudaMemHandleTypeNone;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = device;
  cudaMemPool_t mp = nullptr;
  if (cudaMemPoolCreate(&mp, &props) != cudaSuccess) return nullptr;
  unsigned long long thr = ~0ull;
  cudaMemPoolSetAttribute(mp, cudaMemPoolAttrReleaseThreshold, &thr);
  g_mempools[device] = mp;
  return mp;
}

// Unmap a slot's chunks and give them back to the pool (caller holds g_mu and
// has established that the GPU is done with the slot).
static void unmap_slot(Arena* a, Slot& s, int tensor, int slot) {
  CUdeviceptr va = a->base + (CUdeviceptr)((tensor * 2 + slot) * a->slot_bytes);
  if (!s.chunks.empty()) drv().unmap(va, s.chunks.size() * a->chunk);
  for (auto h : s.chunks) a->pool->free_list.push_back(h);
  s.chunks.clear();
  if (s.pending) {
    cudaEventDestroy(s.pending);
    s.pending = nullptr;
  }
}

Arena* arena_create(int device, size_t max_bytes_per_tensor, int* err) {
  *err = 0;
  Arena* a = new Arena();
  a->device = device;
  std::lock_guard<std::mutex> lk(g_mu);
  // VMM setup (kind 0); falls back to pool-only if unsupported.
  int vmm = 0;
  CUdevice dev = 0;
  if (drv().ok && drv().device_get(&dev, device) == CUDA_SUCCESS &&
      drv().device_attr(&vmm, CU_DEVICE_ATTRIBUTE_VIRTUAL_MEMORY_MANAGEMENT_SUPPORTED, dev) ==
          CUDA_SUCCESS &&
      vmm) {
    CUmemAllocationProp prop = {};
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = device;
    size_t gran = 0;
    if (drv().granularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED) ==
            CUDA_SUCCESS &&
        gran > 0) {
      // chunk: >= 1/16 of the largest buffer (few map calls per growth),
      // 2 MiB for small caches, at most 64 MiB.
      size_t chunk = gran;
      while (chunk < max_bytes_per_tensor / 16 && chunk < (64u << 20)) chunk *= 2;
      a->chunk = chunk;
      a->slot_bytes = round_up(std::max<size_t>(max_bytes_per_tensor, 1), chunk);
      if (drv().reserve(&a->base, 4 * a->slot_bytes, chunk, 0, 0) == CUDA_SUCCESS) {
        a->pool = pool_for(device, chunk);
        a->vmm_ok = true;
      }
    }
  }
  g_arenas.insert(a);
  return a;
}

static int map_slot(Arena* a, int tensor, int slot, size_t bytes) {
  Slot& sl = a->slots[tensor][slot];
  const size_t need = (bytes + a->chunk - 1) / a->chunk;
  CUdeviceptr va = a->base + (CUdeviceptr)((tensor * 2 + slot) * a->slot_bytes);
  const size_t have = sl.chunks.size();
  if (need <= have) return 0;
  CUmemAllocationProp prop = {};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = a->device;
  if (cudaSetDevice(a->device) != cudaSuccess) return BMC_ERR_CUDA;   // helper thread
  for (size_t i = have; i < need; ++i) {
    CUmemGenericAllocationHandle h;
    bool reuse = false;
    {
      std::lock_guard<std::mutex> lk(g_mu);
      if (!a->pool->free_list.empty()) {
        h = a->pool->free_list.back();
        a->pool->free_list.pop_back();
        reuse = true;
      }
    }
    if (!reuse) {
      CUresult r = drv().create(&h, a->chunk, &prop, 0);
      if (r == CUDA_ERROR_OUT_OF_MEMORY) return BMC_ERR_OOM;
      if (r != CUDA_SUCCESS) return BMC_ERR_CUDA;
    }
    if (drv().map(va + i * a->chunk, a->chunk, 0, h, 0) != CUDA_SUCCESS) {
      std::lock_guard<std::mutex> lk(g_mu);
      a->pool->free_list.push_back(h);
      return BMC_ERR_CUDA;
    }
    sl.chunks.push_back(h);
  }
  CUmemAccessDesc acc = {};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = a->device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  return cu_ok(drv().set_access(va + have * a->chunk, (need - have) * a->chunk, &acc, 1));
}

int arena_alloc(Arena* a, int tensor, size_t bytes, int kind, const Buffer* keep,
                cudaStream_t s, Buffer* out) {
  // `keep` is the tensor's live buffer (its slot is not reused).
  *out = Buffer();
  if (bytes == 0) bytes = 16;
  if (kind == 0 && a->vmm_ok) {
    std::lock_guard<std::mutex> lk(a->mu);   // waits only if a premap of this arena is running
    int slot = (keep && keep->ptr && keep->kind == 0) ? 1 - keep->slot : 0;
    Slot& sl = a->slots[tensor][slot];
    // the slot's previous contents were last used earlier on this stream, so
    // the realloc kernel may overwrite them in stream order: only missing
    // chunks are mapped (persistent mappings)
    if (sl.pending) {
      cudaEventDestroy(sl.pending);
      sl.pending = nullptr;
    }
    const bool missing = (bytes + a->chunk - 1) / a->chunk > a->slots[tensor][slot].chunks.size();
    const long long t0 = host_now_ns();
    int rc = map_slot(a, tensor, slot, bytes);
    if (missing) host_time_add(kHostSyncMap, host_now_ns() - t0);   // not premapped in time
    if (rc) return rc;
    out->ptr = (void*)(a->base + (CUdeviceptr)((tensor * 2 + slot) * a->slot_bytes));
    out->bytes = bytes;
    out->slot = slot;
    out->kind = 0;
    a->live[tensor] = slot;
    return 0;
  }
  if (kind == 2) {
    // the end opposite to the live buffer (a copy growth: both live at once)
    const int pref = (keep && keep->ptr && keep->kind == 2) ? 1 - keep->slot : 0;
    if (region_alloc(a->device, bytes, pref, s, out)) return 0;
  }
  cudaMemPool_t mp;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    mp = mempool_for(a->device);
  }
  if (!mp) return BMC_ERR_CUDA;
  void* p = nullptr;
  cudaError_t e = cudaMallocFromPoolAsync(&p, bytes, mp, s);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();   // not sticky: clear it so later launch checks do not report it
    return BMC_ERR_OOM;
  }
  if (e != cudaSuccess) return BMC_ERR_CUDA;
  out->ptr = p;
  out->bytes = bytes;
  out->slot = -1;
  out->kind = 1;
  return 0;
}

int arena_release(Arena* a, Buffer* b, cudaStream_t s) {
  if (!b->ptr) return 0;
  int rc = 0;
  if (b->kind == 1) {
    rc = cudaFreeAsync(b->ptr, s) == cudaSuccess ? 0 : BMC_ERR_CUDA;
  } else if (b->kind == 2) {
    rc = region_release(a->device, b, s);
  } else {
    // VMM slot: the mapping persists for the next growth (see header); nothing
    // to do until the arena is destroyed
    (void)a;
  }
  *b = Buffer();
  return rc;
}

// Map `bytes` of physical memory into the device's stream-ordered pool now
// (allocate + free once; the release threshold keeps it), so later growth
// allocations are carved from it instead of waiting for the driver to grow
// the pool (measured: up to 0.6 s host stalls per growth step otherwise).
int pool_reserve(int device, size_t bytes) {
  std::lock_guard<std::mutex> lk(g_mu);
  cudaMemPool_t mp = mempool_for(device);
  if (!mp) return BMC_ERR_CUDA;
  if (bytes == 0) return 0;
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != device && cudaSetDevice(device) != cudaSuccess) return BMC_ERR_CUDA;
  void* p = nullptr;
  int rc = 0;
  cudaError_t e = cudaMallocFromPoolAsync(&p, bytes, mp, 0);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    rc = BMC_ERR_OOM;
  } else if (e != cudaSuccess || cudaFreeAsync(p, 0) != cudaSuccess ||
             cudaStreamSynchronize(0) != cudaSuccess) {
    rc = BMC_ERR_CUDA;
  }
  if (prev != device) cudaSetDevice(prev);
  return rc;
}

// ------------------------------------------------- asynchronous pre-mapping
namespace {
struct PremapTask { Arena* a; int tensor, slot; size_t bytes; };
struct Premapper {
  std::mutex mu;
  std::condition_variable cv, idle;
  std::deque<PremapTask> q;
  Arena* running = nullptr;
  bool started = false;
  unsigned long long done = 0, late = 0;
  void loop() {
    for (;;) {
      PremapTask t;
      {
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [&] { return !q.empty(); });
        t = q.front();
        q.pop_front();
        running = t.a;
      }
      {
        std::lock_guard<std::mutex> lk(t.a->mu);
        // the live buffer moved to the target slot in the meantime: the
        // request is stale (the growth it prepared for has happened)
        if (t.a->live[t.tensor] != t.slot) {
          const long long t0 = host_now_ns();
          map_slot(t.a, t.tensor, t.slot, t.bytes);
          host_time_add(kHostPremap, host_now_ns() - t0);
        }
      }
      {
        std::lock_guard<std::mutex> lk(mu);
        running = nullptr;
        ++done;
      }
      idle.notify_all();
    }
  }
};
Premapper* g_premap = nullptr;
std::mutex g_premap_mu;

Premapper* premapper() {
  std::lock_guard<std::mutex> lk(g_premap_mu);
  if (!g_premap) {
    g_premap = new Premapper();   // process lifetime (the thread never exits)
    std::thread([p = g_premap] { p->loop(); }).detach();
  }
  return g_premap;
}
}  // namespace

int arena_premap(Arena* a, int tensor, size_t bytes) {
  if (!a || !a->vmm_ok || tensor < 0 || tensor > 1) return 0;
  int slot;
  {
    std::lock_guard<std::mutex> lk(a->mu);
    slot = a->live[tensor] < 0 ? 0 : 1 - a->live[tensor];
    const size_t need = (std::max<size_t>(bytes, 16) + a->chunk - 1) / a->chunk;
    if (need <= a->slots[tensor][slot].chunks.size()) return 0;   // already mapped
  }
  Premapper* p = premapper();
  {
    std::lock_guard<std::mutex> lk(p->mu);
    p->q.push_back(PremapTask{a, tensor, slot, bytes});
  }
  p->cv.notify_one();
  return 0;
}

// Return the pool's unused physical memory to the driver (between workloads).
int pool_trim(int device) {
  std::lock_guard<std::mutex> lk(g_mu);
  cudaMemPool_t mp = mempool_for(device);
  if (!mp) return BMC_ERR_CUDA;
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != device && cudaSetDevice(device) != cudaSuccess) return BMC_ERR_CUDA;
  const int rc = (cudaDeviceSynchronize() == cudaSuccess && cudaMemPoolTrimTo(mp, 0) == cudaSuccess)
                     ? 0 : BMC_ERR_CUDA;
  if (prev != device) cudaSetDevice(prev);
  return rc;
}

void arena_destroy(Arena* a) {
  if (!a) return;
  if (g_premap) {   // no helper-thread work may touch the arena after this
    std::unique_lock<std::mutex> lk(g_premap->mu);
    for (auto it = g_premap->q.begin(); it != g_premap->q.end();)
      it = it->a == a ? g_premap->q.erase(it) : it + 1;
    g_premap->idle.wait(lk, [&] { return g_premap->running != a; });
  }
  std::lock_guard<std::mutex> lk(g_mu);
  for (int t = 0; t < 2; ++t)
    for (int s = 0; s < 2; ++s) {
      Slot& sl = a->slots[t][s];
      if (sl.pending) cudaEventSynchronize(sl.pending);
      if (a->vmm_ok) unmap_slot(a, sl, t, s);
    }
  if (a->base) drv().addr_free(a->base, 4 * a->slot_bytes);
  g_arenas.erase(a);
  delete a;
}

// ------------------------------------------------- two-ended growth region
namespace {
struct RBlk {
  size_t off, bytes;
  bool freed;
  cudaStream_t s;        // releasing stream
  cudaEvent_t ev;        // recorded on s at the release
};
struct Region {
  uint8_t* base = nullptr;
  size_t size = 0;
  std::vector<RBlk> stk[2];   // end 0 grows up from 0, end 1 down from size
  size_t used[2] = {0, 0};
  // latest popped release per stream: space it freed may be handed out on
  // another stream only after it (same-stream reuse is ordered already)
  std::vector<std::pair<cudaStream_t, cudaEvent_t>> fence;
  std::vector<cudaEvent_t> spare;
};
std::mutex g_regmu;
std::map<int, Region*> g_region;
constexpr size_t kRegionAlign = 4096;

cudaEvent_t region_event(Region* r) {
  if (!r->spare.empty()) {
    cudaEvent_t e = r->spare.back();
    r->spare.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return e;
}
}  // namespace

int region_reserve(int device, size_t bytes) {
  std::lock_guard<std::mutex> lk(g_regmu);
  Region*& r = g_region[device];
  if (r && (!r->stk[0].empty() || !r->stk[1].empty())) return BMC_ERR_STATE;   // buffers live
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != device && cudaSetDevice(device) != cudaSuccess) return BMC_ERR_CUDA;
  int rc = 0;
  if (r) {
    cudaDeviceSynchronize();
    forget_range(r->base);
    cudaFree(r->base);
    for (auto& f : r->fence) cudaEventDestroy(f.second);
    for (auto e : r->spare) cudaEventDestroy(e);
    delete r;
    r = nullptr;
  }
  if (bytes > 0) {
    void* p = nullptr;
    const cudaError_t e = cudaMalloc(&p, bytes);
    if (e != cudaSuccess) {
      cudaGetLastError();
      rc = e == cudaErrorMemoryAllocation ? BMC_ERR_OOM : BMC_ERR_CUDA;
    } else {
      r = new Region();
      r->base = static_cast<uint8_t*>(p);
      r->size = bytes / kRegionAlign * kRegionAlign;
    }
  }
  if (prev != device) cudaSetDevice(prev);
  return rc;
}

bool region_present(int device) {
  std::lock_guard<std::mutex> lk(g_regmu);
  auto it = g_region.find(device);
  return it != g_region.end() && it->second;
}

// A block of the region at end `pref` (else the other end) on stream s;
// returns false when the region is absent or full.
static bool region_alloc(int device, size_t bytes, int pref, cudaStream_t s, Buffer* out) {
  std::lock_guard<std::mutex> lk(g_regmu);
  auto it = g_region.find(device);
  if (it == g_region.end() || !it->second) return false;
  Region* r = it->second;
  bytes = (bytes + kRegionAlign - 1) / kRegionAlign * kRegionAlign;
  for (int k = 0; k < 2; ++k) {
    const int e = k == 0 ? pref : 1 - pref;
    if (r->used[0] + r->used[1] + bytes > r->size) continue;
    const size_t off = e == 0 ? r->used[0] : r->size - r->used[1] - bytes;
    r->used[e] += bytes;
    r->stk[e].push_back(RBlk{off, bytes, false, nullptr, nullptr});
    for (auto& f : r->fence)
      if (f.first != s) cudaStreamWaitEvent(s, f.second, 0);
    out->ptr = r->base + off;
    out->bytes = bytes;
    out->slot = e;
    out->kind = 2;
    return true;
  }
  return false;
}

static int region_release(int device, Buffer* b, cudaStream_t s) {
  std::lock_guard<std::mutex> lk(g_regmu);
  auto it = g_region.find(device);
  if (it == g_region.end() || !it->second) return BMC_ERR_CUDA;
  Region* r = it->second;
  const size_t off = static_cast<uint8_t*>(b->ptr) - r->base;
  auto& st = r->stk[b->slot];
  size_t i = st.size();
  while (i > 0 && st[i - 1].off != off) --i;
  if (i == 0) return BMC_ERR_CUDA;
  RBlk& blk = st[i - 1];
  blk.freed = true;
  blk.s = s;
  blk.ev = region_event(r);
  if (!blk.ev || cudaEventRecord(blk.ev, s) != cudaSuccess) return BMC_ERR_CUDA;
  while (!st.empty() && st.back().freed) {   // pop released blocks off this end
    RBlk t = st.back();
    st.pop_back();
    r->used[b->slot] -= t.bytes;
    bool seen = false;
    for (auto& f : r->fence)
      if (f.first == t.s) {   // a later release on the same stream covers the earlier one
        r->spare.push_back(f.second);
        f.second = t.ev;
        seen = true;
      }
    if (!seen) r->fence.emplace_back(t.s, t.ev);
  }
  return 0;
}

// ------------------------------------------------------ pointer classes
// cudaPointerGetAttributes costs microseconds; the hot path calls it for every
// tensor argument.  Device allocations are remembered by address range (a
// device range never turns into host memory under UVA), so repeat calls with
// pointers into known device allocations cost a short scan.
namespace {
struct Range { uintptr_t base, end; int kind; };
std::mutex g_rmu;
std::vector<Range> g_ranges;
}  // namespace

int pointer_kind(const void* ptr) {
  const uintptr_t p = (uintptr_t)ptr;
  {
    std::lock_guard<std::mutex> lk(g_rmu);
    for (size_t i = 0; i < g_ranges.size(); ++i) {
      if (p >= g_ranges[i].base && p < g_ranges[i].end) {
        const int k = g_ranges[i].kind;
        if (i > 0) std::swap(g_ranges[i], g_ranges[i - 1]);  // keep hot ranges in front
        return k;
      }
    }
  }
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
    cudaGetLastError();
    return 2;
  }
  const int kind = (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) ? 0
                   : (a.type == cudaMemoryTypeHost ? 1 : 2);
  if (kind == 0) {
    // device allocations are mapped into the unified address space: remember
    // their whole range.  Page-locked host ranges are not cached: after
    // cudaFreeHost / cudaHostUnregister the same address can come back as
    // pageable memory, which must take the pageable (synchronising) paths.
    CUdeviceptr base = 0;
    size_t size = 0;
    const CUdeviceptr q = (CUdeviceptr)p;
    if (drv().ok && drv().range(&base, &size, q) == CUDA_SUCCESS &&
        size > 0) {
      std::lock_guard<std::mutex> lk(g_rmu);
      if (g_ranges.size() >= 256) g_ranges.pop_back();
      g_ranges.insert(g_ranges.begin(), Range{(uintptr_t)base, (uintptr_t)base + size, kind});
    } else {
      cudaGetLastError();
    }
  }
  return kind;
}

void forget_range(const void* ptr) {
  std::lock_guard<std::mutex> lk(g_rmu);
  const uintptr_t p = (uintptr_t)ptr;
  for (size_t i = 0; i < g_ranges.size(); ++i)
    if (p >= g_ranges[i].base && p < g_ranges[i].end) {
      g_ranges.erase(g_ranges.begin() + i);
      return;
    }
}

}  // namespace bmc
