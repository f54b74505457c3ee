// bmc_abi.cpp -- the C-ABI state machine of libbmc.so (include/bmc.h).
//
// The host keeps an exact shadow of every length (valid_b, cap, staged), so
// no call ever reads anything back from the device on the hot path; all
// validation happens before anything is enqueued.
//
// Row writes are deferred: bmc_append / bmc_spec_write only record the
// caller's row pointers ("pending rows"); the next bmc_sdpa writes them into
// the cache inside the attention kernel (the kernel that owns the tile holding
// the row patches its staged copy and stores the row), so a decode step is one
// launch per layer (one per <=32 layers through bmc_decode_step).  Any other
// operation that needs the rows in memory first flushes them with the
// standalone write_rows kernel.  Launches per call:
//   bmc_append      [growth: arena + realloc_copy_zero]
//   bmc_spec_write  [ITERATIVE growth]
//   bmc_sdpa        attn_step (split-K, in-kernel combine, fused row writes)
//   bmc_commit      zero_rows (rejected drafts only)
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <vector>

#include "bmc_internal.h"

using bmc::Buffer;

struct bmc_ctx {
  int B = 0, H_kv = 0, H_q = 0, D = 0, r = 0, N_max = 0;
  bmc_dtype dt = BMC_BF16;
  bmc_policy pol = BMC_POLICY_BMC;
  int device = 0;
  cudaStream_t stream = nullptr;
  int eb = 2, row_bytes = 0;
  long long U = 0;
  long long cap = 0;
  std::vector<int> valid;
  int staged = 0;
  Buffer kbuf, vbuf;
  bmc::Arena* arena = nullptr;
  int arena_kind = 1;   // stream-ordered pool (measured fastest); 0 = VMM slots
  float* ws = nullptr;
  size_t ws_floats = 0;
  int* counters = nullptr;
  int num_sms = 148;
  int max_ctas = 148;
  int attn_ctas = 0;
  int attn_path = 0;
  int skip_padding = 0;          // length-aware ablation, off by default
  int copy_on_read = 1;          // BMC growth inside the fused decode step
  int tck_groups = 0;            // keys-on-lanes kernel softmax column groups (0 auto)
  int tck_prefetch = -1;         // keys-on-lanes kernel L2 prefetch distance (-1 auto)
  int fault_oom = 0;             // test hook: the next n growth allocations fail (BMC_OPT_FAULT_OOM)
  // a growth whose copy the next attention launch performs (copy-on-read):
  // the old buffers and the rows to carry over; never observable between API
  // calls (bmc_decode_step launches the consuming kernel in the same call)
  bool cor = false;
  Buffer cor_k, cor_v;
  long long cor_cap = 0, cor_rows = 0;
  bmc_stats_t st = {};
  int sticky = 0;
  // staging of host-pointer arguments: 0 appended rows, 1 drafts, 2 Q
  void* stage_in[3] = {nullptr, nullptr, nullptr};
  size_t stage_in_bytes[3] = {0, 0, 0};
  float* stage_out = nullptr;
  size_t stage_out_bytes = 0;
  // rows recorded by append / spec_write, not yet written to the cache
  const void* knew = nullptr;
  const void* vnew = nullptr;
  const void* kd = nullptr;
  const void* vd = nullptr;
  int n_app = 0, n_draft = 0, kd_stride = 0;
  int tree = 0;                  // staged rows form a token tree
  uint32_t anc[32] = {};         // bit j of anc[i]: node j is node i or its ancestor
  struct Pipe* pipe = nullptr;   // host-I/O pipeline of bmc_decode_step (first layer owns it)
  struct HostIO* hio = nullptr;  // copy streams of the per-call API's pinned host arguments
};

// Pinned-host arguments of the per-call API (append, spec_write, sdpa) are
// copied on the handle's own upload / download streams, ordered against the
// compute stream with events, so the copies of layer l+1 overlap the kernel of
// layer l (the per-layer speculative-decoding loop's end-to-end path).
struct HostIO {
  cudaStream_t up = nullptr, down = nullptr;
  cudaEvent_t in_ready[3] = {}, in_free[3] = {}, alloc_done = nullptr;
  bool in_used[3] = {false, false, false};
  cudaEvent_t out_ready = nullptr, out_free = nullptr;
  bool out_used = false;
};

static void hio_destroy(HostIO* x) {
  if (!x) return;
  if (x->up) cudaStreamSynchronize(x->up);
  if (x->down) cudaStreamSynchronize(x->down);
  for (int i = 0; i < 3; ++i) {
    if (x->in_ready[i]) cudaEventDestroy(x->in_ready[i]);
    if (x->in_free[i]) cudaEventDestroy(x->in_free[i]);
  }
  if (x->alloc_done) cudaEventDestroy(x->alloc_done);
  if (x->out_ready) cudaEventDestroy(x->out_ready);
  if (x->out_free) cudaEventDestroy(x->out_free);
  if (x->up) cudaStreamDestroy(x->up);
  if (x->down) cudaStreamDestroy(x->down);
  delete x;
}

// Host-I/O pipeline of bmc_decode_step: two staging slots, a copy stream and
// events, so that the host->device copy of step s+1 and the device->host copy
// of step s's outputs overlap the kernels of step s (e2e path).
struct Pipe {
  cudaStream_t copy = nullptr;   // uploads (host -> device)
  cudaStream_t down = nullptr;   // downloads (device -> host), so neither waits for the other
  cudaEvent_t in_ready[2] = {}, compute_done[2] = {}, out_done[2] = {};
  char* in_slot[2] = {nullptr, nullptr};
  char* out_slot[2] = {nullptr, nullptr};
  size_t in_bytes = 0, out_bytes = 0;
  long long step = 0;
  bool primed[2] = {false, false};
};

static void pipe_destroy(Pipe* p) {
  if (!p) return;
  if (p->copy) cudaStreamSynchronize(p->copy);
  if (p->down) cudaStreamSynchronize(p->down);
  for (int i = 0; i < 2; ++i) {
    if (p->in_ready[i]) cudaEventDestroy(p->in_ready[i]);
    if (p->compute_done[i]) cudaEventDestroy(p->compute_done[i]);
    if (p->out_done[i]) cudaEventDestroy(p->out_done[i]);
    if (p->in_slot[i]) cudaFree(p->in_slot[i]);
    if (p->out_slot[i]) cudaFree(p->out_slot[i]);
  }
  if (p->copy) cudaStreamDestroy(p->copy);
  if (p->down) cudaStreamDestroy(p->down);
  delete p;
}

static thread_local std::string g_err;
// auto path: tcgen05 (keys on the TMEM lanes) for every M = G*t the kernel
// takes (bf16, D = 128, M <= 80), CUDA cores otherwise (fp32, D = 64).  At
// M = 1 the tensor-core kernel held 1.08x the copy peak where the CUDA-core
// kernel fell to 0.94x on the same power-capped box (SM 1.55-1.64 GHz): its
// per-byte instruction count makes it clock-sensitive
// (profiles/r01_attn_path_ab.jsonl)
static constexpr int kTcMinM = 0;

static int fail(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
static int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

static int cuda_fail(bmc_t h, cudaError_t e, const char* where) {
  if (h) h->sticky = BMC_ERR_CUDA;
  return fail(e == cudaErrorMemoryAllocation ? BMC_ERR_OOM : BMC_ERR_CUDA, "%s: %s", where,
              cudaGetErrorString(e));
}

#define CK(h, expr, where)                                   \
  do {                                                       \
    cudaError_t _e = (expr);                                 \
    if (_e != cudaSuccess) return cuda_fail((h), _e, where); \
  } while (0)

static int cor_materialize(bmc_t h);
static int enter(bmc_t h) {
  if (!h) return fail(BMC_ERR_ARG, "null handle");
  if (h->sticky) return fail(h->sticky, "handle is in a sticky CUDA error state");
  int cur = -1;
  if (cudaGetDevice(&cur) != cudaSuccess || cur != h->device) {
    cudaError_t e = cudaSetDevice(h->device);
    if (e != cudaSuccess) return cuda_fail(h, e, "cudaSetDevice");
  }
  if (h->cor) return cor_materialize(h);   // pending only between bmc_append and bmc_sdpa
  return 0;
}
// enter() for bmc_sdpa: a copy-on-read growth left by bmc_append stays
// pending for the attention launch to carry out
static int enter_keep_growth(bmc_t h) {
  if (!h || !h->cor) return enter(h);
  if (h->sticky) return fail(h->sticky, "handle is in a sticky CUDA error state");
  int cur = -1;
  if (cudaGetDevice(&cur) != cudaSuccess || cur != h->device) {
    cudaError_t e = cudaSetDevice(h->device);
    if (e != cudaSuccess) return cuda_fail(h, e, "cudaSetDevice");
  }
  return 0;
}

static int max_valid(const bmc_t h) { return *std::max_element(h->valid.begin(), h->valid.end()); }
static int min_valid(const bmc_t h) { return *std::min_element(h->valid.begin(), h->valid.end()); }

static int ptr_kind(const void* p) { return bmc::pointer_kind(p); }
static bool is_device_ptr(const void* p) { return ptr_kind(p) == 0; }

static int ensure_stage_in(bmc_t h, int slot, size_t bytes) {
  if (h->stage_in_bytes[slot] >= bytes) return 0;
  if (h->stage_in[slot]) cudaFreeAsync(h->stage_in[slot], h->stream);
  h->stage_in[slot] = nullptr;
  h->stage_in_bytes[slot] = 0;
  CK(h, cudaMallocAsync(&h->stage_in[slot], bytes, h->stream), "stage_in");
  h->stage_in_bytes[slot] = bytes;
  return 0;
}

// Map caller inputs (device or host) to device pointers; host inputs are
// copied into the handle's staging buffer `slot` on its stream.
static int ensure_hio(bmc_t h) {
  if (h->hio) return 0;
  HostIO* x = new HostIO();
  h->hio = x;
  CK(h, cudaStreamCreateWithFlags(&x->up, cudaStreamNonBlocking), "upload stream");
  CK(h, cudaStreamCreateWithFlags(&x->down, cudaStreamNonBlocking), "download stream");
  for (int i = 0; i < 3; ++i) {
    CK(h, cudaEventCreateWithFlags(&x->in_ready[i], cudaEventDisableTiming), "event");
    CK(h, cudaEventCreateWithFlags(&x->in_free[i], cudaEventDisableTiming), "event");
  }
  CK(h, cudaEventCreateWithFlags(&x->alloc_done, cudaEventDisableTiming), "event");
  CK(h, cudaEventCreateWithFlags(&x->out_ready, cudaEventDisableTiming), "event");
  CK(h, cudaEventCreateWithFlags(&x->out_free, cudaEventDisableTiming), "event");
  return 0;
}

// The staged inputs of every slot have been consumed by the kernels enqueued
// on the compute stream so far (called after each launch that reads them).
static int inputs_consumed(bmc_t h) {
  if (!h->hio) return 0;
  for (int i = 0; i < 3; ++i)
    if (h->hio->in_used[i]) CK(h, cudaEventRecord(h->hio->in_free[i], h->stream), "event");
  return 0;
}

// Device pointers for the op's inputs: device arguments are used in place,
// host arguments are copied into staging slot `slot` -- pinned ones on the
// upload stream (overlapping earlier kernels), pageable ones on the compute
// stream.
static int device_inputs(bmc_t h, int slot, const void** ptrs, const size_t* bytes, int n,
                         const void** dev) {
  size_t need = 0;
  bool any_host = false, all_pinned = true;
  int kind[8];
  for (int i = 0; i < n; ++i) {
    kind[i] = ptr_kind(ptrs[i]);
    if (kind[i] != 0) {
      any_host = true;
      if (kind[i] != 1) all_pinned = false;
      need += (bytes[i] + 255) / 256 * 256;
    }
  }
  if (!any_host) {
    for (int i = 0; i < n; ++i) dev[i] = ptrs[i];
    return 0;
  }
  const bool grew = h->stage_in_bytes[slot] < need;
  int rc = ensure_stage_in(h, slot, need);
  if (rc) return rc;
  cudaStream_t cs = h->stream;
  if (all_pinned) {
    rc = ensure_hio(h);
    if (rc) return rc;
    HostIO* x = h->hio;
    cs = x->up;
    if (grew) {   // the new slot was allocated on the compute stream
      CK(h, cudaEventRecord(x->alloc_done, h->stream), "event");
      CK(h, cudaStreamWaitEvent(cs, x->alloc_done, 0), "wait");
    }
    if (x->in_used[slot]) CK(h, cudaStreamWaitEvent(cs, x->in_free[slot], 0), "wait");
  }
  size_t off = 0;
  for (int i = 0; i < n; ++i) {
    if (kind[i] == 0) {
      dev[i] = ptrs[i];
    } else {
      void* d = (char*)h->stage_in[slot] + off;
      CK(h, cudaMemcpyAsync(d, ptrs[i], bytes[i], cudaMemcpyHostToDevice, cs), "H2D");
      dev[i] = d;
      off += (bytes[i] + 255) / 256 * 256;
    }
  }
  if (all_pinned) {
    HostIO* x = h->hio;
    CK(h, cudaEventRecord(x->in_ready[slot], cs), "event");
    CK(h, cudaStreamWaitEvent(h->stream, x->in_ready[slot], 0), "wait");
    x->in_used[slot] = true;
  }
  return 0;
}

static int cor_materialize(bmc_t h);

// Replace the cache buffers by [U][new_cap][D] buffers holding the first
// copy_rows rows of every unit, zero elsewhere.  defer: the
// copy and zero fill are left to the next attention launch (copy-on-read);
// the ledger is the same either way.
static int reallocate(bmc_t h, long long new_cap, long long copy_rows, bool defer = false) {
  if (h->cor) {
    int rc = cor_materialize(h);
    if (rc) return rc;
  }
  if (h->fault_oom > 0) {
    --h->fault_oom;
    return fail(BMC_ERR_OOM, "injected allocation failure (BMC_OPT_FAULT_OOM)");
  }
  const size_t bytes = (size_t)h->U * new_cap * h->row_bytes;
  Buffer nk, nv;
  const long long t_alloc = bmc::host_now_ns();
  int rc = bmc::arena_alloc(h->arena, 0, bytes, h->arena_kind, &h->kbuf, h->stream, &nk);
  if (rc) return fail(rc, "arena_alloc(K, %zu bytes) failed", bytes);
  rc = bmc::arena_alloc(h->arena, 1, bytes, h->arena_kind, &h->vbuf, h->stream, &nv);
  bmc::host_time_add(bmc::kHostAlloc, bmc::host_now_ns() - t_alloc);
  if (rc) {
    bmc::arena_release(h->arena, &nk, h->stream);
    return fail(rc, "arena_alloc(V, %zu bytes) failed", bytes);
  }
  // VMM arena: map the NEXT growth's chunks on the helper thread now (BMC:
  // r appends away, size cap + r; ITERATIVE: a few rows more)
  if (h->arena_kind == 0 && h->pol != BMC_POLICY_UPFRONT) {
    const long long nxt = h->pol == BMC_POLICY_BMC ? std::min<long long>(new_cap + h->r, h->N_max)
                                                   : std::min<long long>(new_cap + 64, h->N_max);
    if (nxt > new_cap) {
      bmc::arena_premap(h->arena, 0, (size_t)h->U * nxt * h->row_bytes);
      bmc::arena_premap(h->arena, 1, (size_t)h->U * nxt * h->row_bytes);
    }
  }
  if (h->cap > 0) h->st.copy_events += 1;
  h->st.alloc_events += 1;
  h->st.copied_bytes += 2LL * h->U * copy_rows * h->row_bytes;
  h->st.init_written_bytes += 2LL * h->U * new_cap * h->row_bytes;
  if (defer && h->cap > 0 && copy_rows > 0) {
    h->cor = true;
    h->cor_k = h->kbuf;
    h->cor_v = h->vbuf;
    h->cor_cap = h->cap;
    h->cor_rows = copy_rows;
    h->kbuf = nk;
    h->vbuf = nv;
    h->cap = new_cap;
    return 0;
  }
  bmc::ReallocArgs a;
  a.src_k = h->kbuf.ptr;
  a.src_v = h->vbuf.ptr;
  a.dst_k = nk.ptr;
  a.dst_v = nv.ptr;
  a.U = h->U;
  a.cap_old = h->cap;
  a.cap_new = new_cap;
  a.copy_rows = copy_rows;
  a.row_bytes = h->row_bytes;
  CK(h, bmc::launch_realloc_copy_zero(a, h->stream), "realloc_copy_zero");
  if (bmc::arena_release(h->arena, &h->kbuf, h->stream) ||
      bmc::arena_release(h->arena, &h->vbuf, h->stream)) {
    h->sticky = BMC_ERR_CUDA;
    return fail(BMC_ERR_CUDA, "arena_release failed");
  }
  h->kbuf = nk;
  h->vbuf = nv;
  h->cap = new_cap;
  return 0;
}

// The old buffers of a copy-on-read growth are free once the consuming
// attention launch is enqueued (stream-ordered release).
static int cor_release(bmc_t h) {
  if (!h->cor) return 0;
  h->cor = false;
  const long long t0 = bmc::host_now_ns();
  if (bmc::arena_release(h->arena, &h->cor_k, h->stream) ||
      bmc::arena_release(h->arena, &h->cor_v, h->stream)) {
    h->sticky = BMC_ERR_CUDA;
    return fail(BMC_ERR_CUDA, "arena_release failed");
  }
  bmc::host_time_add(bmc::kHostRelease, bmc::host_now_ns() - t0);
  return 0;
}

// A deferred growth whose attention launch will not happen: do the copy and
// zero fill with the realloc kernel after all.
static int cor_materialize(bmc_t h) {
  if (!h->cor) return 0;
  bmc::ReallocArgs a;
  a.src_k = h->cor_k.ptr;
  a.src_v = h->cor_v.ptr;
  a.dst_k = h->kbuf.ptr;
  a.dst_v = h->vbuf.ptr;
  a.U = h->U;
  a.cap_old = h->cor_cap;
  a.cap_new = h->cap;
  a.copy_rows = h->cor_rows;
  a.row_bytes = h->row_bytes;
  CK(h, bmc::launch_realloc_copy_zero(a, h->stream), "realloc_copy_zero");
  return cor_release(h);
}

static int write_rows(bmc_t h, const void* K, const void* V, int nsrc, int nwrite, int row_shift) {
  bmc::RowsArgs a;
  a.src_k = K;
  a.src_v = V;
  a.dst_k = h->kbuf.ptr;
  a.dst_v = h->vbuf.ptr;
  a.B = h->B;
  a.H_kv = h->H_kv;
  a.nsrc = nsrc;
  a.nwrite = nwrite;
  a.cap = h->cap;
  a.row_bytes = h->row_bytes;
  for (int b = 0; b < h->B; ++b) a.row0[b] = h->valid[b] + row_shift;
  CK(h, bmc::launch_write_rows(a, h->stream), "write_rows");
  return 0;
}

// Write recorded rows that no attention launch has consumed yet.
static int flush_pending(bmc_t h) {
  int rc = 0;
  if (h->n_app) rc = write_rows(h, h->knew, h->vnew, 1, 1, -1);   // row valid_b - 1
  if (!rc && h->n_draft) rc = write_rows(h, h->kd, h->vd, h->kd_stride, h->n_draft, 0);
  h->n_app = h->n_draft = 0;
  if (!rc) rc = inputs_consumed(h);
  return rc;
}

// Partial-record workspace for up to M query rows per unit (grown on demand).
static int ensure_workspace(bmc_t h, int M) {
  const size_t need = bmc::attn_workspace_floats(M, h->D, h->max_ctas);
  if (need <= h->ws_floats) return 0;
  cudaFreeAsync(h->ws, h->stream);
  h->ws = nullptr;
  CK(h, cudaMallocAsync((void**)&h->ws, need * sizeof(float), h->stream), "workspace");
  h->ws_floats = need;
  return 0;
}

static void fill_layer(bmc_t h, const void* Q, float* O, bmc::AttnLayer* l) {
  l->K = h->kbuf.ptr;
  l->V = h->vbuf.ptr;
  l->Ksrc = h->cor ? h->cor_k.ptr : nullptr;
  l->Vsrc = h->cor ? h->cor_v.ptr : nullptr;
  l->cap_src = h->cor ? h->cor_cap : 0;
  l->rows_src = h->cor ? h->cor_rows : 0;
  l->Q = Q;
  l->O = O;
  l->Knew = h->knew;
  l->Vnew = h->vnew;
  l->Kd = h->kd;
  l->Vd = h->vd;
  l->ws = h->ws;
  l->counters = h->counters;
  l->cap = h->cap;
  // ablation only: stream just the rows some query can see (the method's
  // contract reads all cap rows)
  l->scan = 0;
  if (h->skip_padding) {
    const long long vis = (long long)max_valid(h) + h->staged;
    l->scan = std::max(1LL, std::min<long long>(h->cap, vis));
  }
  l->n_app = h->n_app;
  l->n_draft = h->n_draft;
  l->kd_stride = h->kd_stride;
}

static void fill_args(bmc_t h, int t, bmc::AttnStepArgs* a) {
  a->B = h->B;
  a->H_kv = h->H_kv;
  a->H_q = h->H_q;
  a->D = h->D;
  a->t = t;
  a->dtype = h->dt;
  a->ctas = std::min(h->attn_ctas, h->max_ctas);
  a->tree = h->tree;
  a->tck_groups = h->tck_groups;
  a->tck_prefetch = h->tck_prefetch;
  for (int i = 0; i < 32; ++i) a->anc[i] = h->anc[i];
  for (int b = 0; b < h->B; ++b) a->valid[b] = h->valid[b];
}

static void account_sdpa(bmc_t h, int t) {
  h->st.sdpa_calls += 1;
  h->st.kv_bytes_read += 2LL * h->U * h->cap * h->row_bytes;
  h->st.macs += 2LL * h->B * h->H_q * t * h->cap * (long long)h->D;
}

extern "C" {

int bmc_create_ex(int B, int H_kv, int H_q, int D, int r, int N_max, bmc_dtype dt,
                  bmc_policy pol, int device, void* cuda_stream, bmc_t* out) {
  if (!out) return fail(BMC_ERR_ARG, "out is null");
  *out = nullptr;
  if (B < 1 || H_kv < 1 || H_q < 1 || D < 1 || N_max < 1)
    return fail(BMC_ERR_ARG, "dims must be >= 1 (B=%d H_kv=%d H_q=%d D=%d N_max=%d)", B, H_kv,
                H_q, D, N_max);
  if (H_q % H_kv != 0) return fail(BMC_ERR_ARG, "H_q %% H_kv != 0");
  if (pol != BMC_POLICY_BMC && pol != BMC_POLICY_ITERATIVE && pol != BMC_POLICY_UPFRONT)
    return fail(BMC_ERR_ARG, "bad policy %d", (int)pol);
  if (pol == BMC_POLICY_BMC && (r < 1 || r > N_max))
    return fail(BMC_ERR_ARG, "r=%d outside [1, N_max=%d]", r, N_max);
  if (D != 64 && D != 128) return fail(BMC_ERR_UNSUPPORTED, "D=%d not in {64,128}", D);
  if (dt != BMC_F32 && dt != BMC_BF16) return fail(BMC_ERR_UNSUPPORTED, "dtype %d", (int)dt);
  if (B > BMC_MAX_B) return fail(BMC_ERR_UNSUPPORTED, "B=%d > BMC_MAX_B", B);

  if (device < 0) {
    cudaError_t e = cudaGetDevice(&device);
    if (e != cudaSuccess) return cuda_fail(nullptr, e, "cudaGetDevice");
  } else {
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return cuda_fail(nullptr, e, "cudaSetDevice");
  }
  bmc_ctx* h = new bmc_ctx();
  h->B = B; h->H_kv = H_kv; h->H_q = H_q; h->D = D; h->r = r; h->N_max = N_max;
  h->dt = dt; h->pol = pol; h->device = device;
  h->stream = (cudaStream_t)cuda_stream;
  h->eb = dt == BMC_BF16 ? 2 : 4;
  h->row_bytes = D * h->eb;
  h->U = (long long)B * H_kv;
  h->valid.assign(B, 0);
  cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, device);
  h->max_ctas = 4 * h->num_sms;
  int err = 0;
  h->arena = bmc::arena_create(device, (size_t)h->U * N_max * h->row_bytes, &err);
  // a device with a growth region: the handle's buffers (the first one too)
  // come from it
  if (bmc::region_present(device)) h->arena_kind = 2;
  const size_t wsf = bmc::attn_workspace_floats(8, D, h->max_ctas);
  h->ws_floats = wsf;
  // stream-ordered: creating a handle never synchronises the device
  cudaError_t e = cudaMallocAsync((void**)&h->ws, wsf * sizeof(float), h->stream);
  if (e == cudaSuccess) e = cudaMallocAsync((void**)&h->counters, (size_t)h->U * sizeof(int), h->stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(h->counters, 0, (size_t)h->U * sizeof(int), h->stream);
  if (e != cudaSuccess) {
    int rc = cuda_fail(nullptr, e, "create workspace");
    bmc_destroy(h);
    return rc;
  }
  int rc = 0;
  if (pol == BMC_POLICY_BMC) rc = reallocate(h, std::min(r, N_max), 0);
  else if (pol == BMC_POLICY_UPFRONT) rc = reallocate(h, N_max, 0);
  if (rc) {
    std::string msg = g_err;
    bmc_destroy(h);
    g_err = msg;
    return rc;
  }
  *out = h;
  return 0;
}

int bmc_create(int B, int H_kv, int H_q, int D, int r, int N_max, bmc_t* out) {
  return bmc_create_ex(B, H_kv, H_q, D, r, N_max, BMC_BF16, BMC_POLICY_BMC, -1, nullptr, out);
}

// Append = growth if needed + record the row (written by the next SDPA).
// defer_growth: a BMC growth's copy is done by the attention launch that the
// caller enqueues next (copy-on-read; only bmc_decode_step's CUDA-core path).
static int append_impl(bmc_t h, const void* K, const void* V, bool defer_growth = false) {
  int rc = 0;
  if (h->n_app || h->n_draft) rc = flush_pending(h);
  if (rc) return rc;
  const int mv = max_valid(h);
  if (h->pol == BMC_POLICY_ITERATIVE) {
    rc = reallocate(h, mv + 1, mv);                      // Fig. AttnBlkListing concat
  } else if (h->pol == BMC_POLICY_BMC && mv == h->cap) {
    rc = reallocate(h, std::min<long long>(h->cap + h->r, h->N_max), h->cap,
                    defer_growth);
  }
  if (rc) return rc;
  const size_t in_bytes = (size_t)h->U * h->row_bytes;
  const void* ptrs[2] = {K, V};
  const size_t sizes[2] = {in_bytes, in_bytes};
  const void* dev[2];
  rc = device_inputs(h, 0, ptrs, sizes, 2, dev);
  if (rc) return rc;
  h->knew = dev[0];
  h->vnew = dev[1];
  h->n_app = 1;
  h->st.append_written_bytes += 2LL * h->U * h->row_bytes;
  for (auto& v : h->valid) v += 1;
  return 0;
}

// Append of layer l inside a fused step whose layers [l0, l) may hold
// deferred (copy-on-read) growths: if deferring this layer's growth runs out
// of memory, those growths are done by the realloc kernel (freeing their old
// buffers) and the append is retried without deferral.
static int append_fused(const bmc_t* hs, int l0, int l, const void* K, const void* V,
                        bool defer) {
  int rc = append_impl(hs[l], K, V, defer);
  if (rc == BMC_ERR_OOM && defer) {
    for (int x = l0; x < l; ++x) {
      rc = cor_materialize(hs[x]);
      if (rc) return rc;
    }
    rc = append_impl(hs[l], K, V, false);
  }
  return rc;
}

// Undo what append_impl (appended) and spec_write_impl did to a layer whose
// attention launch has not been enqueued, after an error later in a fused
// step: a deferred growth is carried out (the new capacity stays, so the
// retried step does not grow again and the ledger totals match an
// uninterrupted run), the lengths and the recorded rows are rolled back.
static void undo_layer_step(bmc_t h, bool appended) {
  cor_materialize(h);
  h->st.append_written_bytes -= 2LL * h->U * h->n_draft * h->row_bytes;
  h->n_draft = 0;
  h->staged = 0;
  h->tree = 0;
  h->kd = h->vd = nullptr;
  if (appended) {
    for (auto& v : h->valid) v -= 1;
    h->st.append_written_bytes -= 2LL * h->U * h->row_bytes;
    h->n_app = 0;
    h->knew = h->vnew = nullptr;
  }
  inputs_consumed(h);
}

// Roll back layers [l0, l_end) of the chunk being built (layers < n_appended
// had their append done) and keep the first error message.
static int rollback_chunk(const bmc_t* hs, int l0, int l_end, int n_appended, int rc) {
  const std::string msg = g_err;
  for (int x = l0; x < l_end; ++x) undo_layer_step(hs[x], x < n_appended);
  g_err = msg;
  return rc;
}

// Chunk order of a fused step.  In the two-ended growth region a growth
// pushes each chunk's new buffers onto one end and pops its old buffers off
// the other; taking the chunks in the reverse of the order that pushed the
// old buffers (last pushed = on top = first moved) lets every chunk's old
// buffers leave the region before the next chunk's new ones arrive, so a
// growth needs the cache plus ONE chunk of new buffers, not twice the cache.
// The buffers sit at end 0 after odd-numbered growths (pushed in forward
// order), at end 1 after even-numbered ones (pushed in reverse order).
static bool chunks_reversed(bmc_t h0) {
  return h0->kbuf.kind == 2 && h0->kbuf.slot == 0;
}

// One chunk's keys-on-lanes launch: all layers in one launch when they agree
// on capacity, copy-on-read state and pending rows (the usual case: one r,
// one step sequence), else one launch per layer (e.g. after an OOM fallback
// carried some layers' growths out with the realloc kernel).
static int launch_tck_chunk(bmc_t h0, const bmc::AttnStepArgs& a, bmc::AttnLayer* layers, int nl) {
  struct T {
    long long t0 = bmc::host_now_ns();
    ~T() { bmc::host_time_add(bmc::kHostLaunch, bmc::host_now_ns() - t0); }
  } timer;
  bool same = true;
  for (int l = 1; l < nl; ++l)
    if (layers[l].cap != layers[0].cap || layers[l].scan != layers[0].scan ||
        (layers[l].Ksrc != nullptr) != (layers[0].Ksrc != nullptr) ||
        layers[l].cap_src != layers[0].cap_src || layers[l].rows_src != layers[0].rows_src ||
        layers[l].n_app != layers[0].n_app || layers[l].n_draft != layers[0].n_draft ||
        layers[l].kd_stride != layers[0].kd_stride)
      same = false;
  if (same) {
    CK(h0, bmc::launch_attn_tck(a, h0->num_sms, h0->stream), "attn_tck");
    return 0;
  }
  for (int l = 0; l < nl; ++l) {
    bmc::AttnStepArgs a1 = a;
    a1.L = 1;
    a1.layers = &layers[l];
    CK(h0, bmc::launch_attn_tck(a1, h0->num_sms, h0->stream), "attn_tck");
  }
  return 0;
}

int bmc_append(bmc_t h, const void* K, const void* V) {
  int rc = enter(h);
  if (rc) return rc;
  if (!K || !V) return fail(BMC_ERR_ARG, "K or V is null");
  if (h->staged > 0) return fail(BMC_ERR_STATE, "append while %d drafts are staged", h->staged);
  if (max_valid(h) >= h->N_max) return fail(BMC_ERR_CAPACITY, "cache full (N_max=%d)", h->N_max);
  // a BMC growth is left to the next bmc_sdpa's attention launch
  // (copy-on-read); any other call carries it out first (enter)
  return append_impl(h, K, V, h->copy_on_read && !h->skip_padding);
}

int bmc_append_n(bmc_t h, const void* K, const void* V, int n) {
  int rc = enter(h);
  if (rc) return rc;
  if (n < 0) return fail(BMC_ERR_ARG, "n=%d < 0", n);
  if (n == 0) return 0;
  if (!K || !V) return fail(BMC_ERR_ARG, "K or V is null");
  if (h->staged > 0) return fail(BMC_ERR_STATE, "append while %d drafts are staged", h->staged);
  const int mv = max_valid(h);
  if ((long long)mv + n > h->N_max)
    return fail(BMC_ERR_CAPACITY, "%d + %d rows exceed N_max=%d", mv, n, h->N_max);
  if (h->n_app || h->n_draft) rc = flush_pending(h);
  if (rc) return rc;
  // one allocation for the whole prompt, to the capacity n single
  // appends would end at; the mv rows that can hold data are copied
  const long long need = (long long)mv + n;
  if (h->pol == BMC_POLICY_ITERATIVE) {
    rc = reallocate(h, need, mv);
  } else if (h->pol == BMC_POLICY_BMC && need > h->cap) {
    const long long chunks = (need - h->cap + h->r - 1) / h->r;
    rc = reallocate(h, std::min<long long>(h->cap + chunks * h->r, h->N_max), mv);
  }
  if (rc) return rc;
  const size_t in_bytes = (size_t)h->U * n * h->row_bytes;
  const void* ptrs[2] = {K, V};
  const size_t sizes[2] = {in_bytes, in_bytes};
  const void* dev[2];
  rc = device_inputs(h, 0, ptrs, sizes, 2, dev);
  if (rc) return rc;
  rc = write_rows(h, dev[0], dev[1], n, n, 0);
  if (!rc) rc = inputs_consumed(h);
  if (rc) return rc;
  h->st.append_written_bytes += 2LL * h->U * n * h->row_bytes;
  for (auto& v : h->valid) v += n;
  return 0;
}

static int spec_write_impl(bmc_t h, const void* K_draft, const void* V_draft, int k);
static void set_tree(bmc_t h, const int* parent, int k_adm);
static int check_parents(const int* parent, int k);

int bmc_spec_write(bmc_t h, const void* K_draft, const void* V_draft, int k) {
  int rc = enter(h);
  if (rc) return rc;
  return spec_write_impl(h, K_draft, V_draft, k);
}

// spec_write without enter(): bmc_spec_step calls it between the (possibly
// deferred, copy-on-read) growth and the attention launch that performs it
static int spec_write_impl(bmc_t h, const void* K_draft, const void* V_draft, int k) {
  int rc = 0;
  if (k < 0) return fail(BMC_ERR_ARG, "k=%d < 0", k);
  if (k > 0 && (!K_draft || !V_draft)) return fail(BMC_ERR_ARG, "draft pointers are null");
  if (h->staged > 0) return fail(BMC_ERR_STATE, "drafts already staged");
  if (k == 0) return 0;
  const int mv = max_valid(h);
  int k_adm;
  if (h->pol == BMC_POLICY_ITERATIVE) {
    k_adm = std::min(k, h->N_max - mv);
    if (k_adm > 0) {
      if (h->n_app) rc = flush_pending(h);                // the copy must see every row
      if (!rc) rc = reallocate(h, (long long)mv + k_adm, mv);
      if (rc) return rc;
    }
  } else {
    k_adm = (int)std::min<long long>(k, h->cap - mv);    // P:L867-869 admission
  }
  if (k_adm > 0) {
    const size_t in_bytes = (size_t)h->U * k * h->row_bytes;
    const void* ptrs[2] = {K_draft, V_draft};
    const size_t sizes[2] = {in_bytes, in_bytes};
    const void* dev[2];
    rc = device_inputs(h, 1, ptrs, sizes, 2, dev);
    if (rc) return rc;
    h->kd = dev[0];
    h->vd = dev[1];
    h->n_draft = k_adm;
    h->kd_stride = k;
    h->st.append_written_bytes += 2LL * h->U * k_adm * h->row_bytes;
  }
  h->staged = k_adm;
  return k_adm;
}

int bmc_spec_write_tree(bmc_t h, const void* K_draft, const void* V_draft, int k,
                        const int* parent_host) {
  int rc = enter(h);
  if (rc) return rc;
  if (k < 0) return fail(BMC_ERR_ARG, "k=%d < 0", k);
  rc = check_parents(parent_host, k);
  if (rc) return rc;
  const int k_adm = spec_write_impl(h, K_draft, V_draft, k);
  if (k_adm < 0) return k_adm;
  set_tree(h, parent_host, k_adm);
  return k_adm;
}

// The attention launch of one layer (t query rows per head): kernel choice
// by M = G*t, workspace, the layer's pending rows consumed.
static int launch_sdpa_layer(bmc_t h, const void* qd, float* od, int t) {
  int rc = 0;
  const int M = (h->H_q / h->H_kv) * t;
  // tensor cores whenever the kernel takes the shape (kTcMinM above): at
  // M = 4, 5 tcgen05 was 1.4x / 2.1x faster than CUDA cores, at M = 1 it is
  // the one that holds HBM bandwidth under the power-capped SM clock
  const bool use_tc = h->attn_path >= 2 ||
                      (h->attn_path == 0 && M > kTcMinM && bmc::attn_tc_supported(h->D, h->dt, M));
  // keys on the TMEM lanes (attn_tck.cu) for M <= 80, queries on the lanes
  // above that or when forced (path 3); path 4 insists on keys on the lanes
  const bool use_tck = use_tc && h->attn_path != 3 &&
                       bmc::attn_tck_supported(h->D, h->dt, M);
  if (h->attn_path == 4 && !use_tck)
    return fail(BMC_ERR_UNSUPPORTED, "keys-on-lanes tcgen05 path needs bf16, D=128, G*t<=80");
  if (use_tc) {
    if (!bmc::attn_tc_supported(h->D, h->dt, M))
      return fail(BMC_ERR_UNSUPPORTED, "tcgen05 path needs bf16, D=128, G*t<=128");
    rc = ensure_workspace(h, M);
    if (rc) return rc;
  }
  // a pending copy-on-read growth (bmc_append -> bmc_sdpa): the CUDA-core and
  // keys-on-lanes kernels copy while they stream, the queries-on-lanes one
  // takes the separate realloc kernel first
  if (h->cor && use_tc && !use_tck) {
    rc = cor_materialize(h);
    if (rc) return rc;
  }
  bmc::AttnLayer layer;
  fill_layer(h, qd, od, &layer);
  bmc::AttnStepArgs a;
  fill_args(h, t, &a);
  a.L = 1;
  a.layers = &layer;
  if (use_tc) {
    a.ctas = std::min(h->attn_ctas, h->num_sms);
    if (use_tck)
      CK(h, bmc::launch_attn_tck(a, h->num_sms, h->stream), "attn_tck");
    else
      CK(h, bmc::launch_attn_tc(a, h->num_sms, h->stream), "attn_tc");
  } else {
    CK(h, bmc::launch_attn_step(a, h->num_sms, h->stream), "attn_step");
  }
  h->n_app = h->n_draft = 0;
  account_sdpa(h, t);
  rc = cor_release(h);
  if (rc) return rc;
  return inputs_consumed(h);
}

int bmc_sdpa(bmc_t h, const void* Q, int n_valid, float* O) {
  int rc = enter_keep_growth(h);
  if (rc) return rc;
  if (!Q || !O) return fail(BMC_ERR_ARG, "Q or O is null");
  if (n_valid == 0) return fail(BMC_ERR_ARG, "n_valid == 0");
  if (n_valid != BMC_PER_ROW) {
    for (int b = 0; b < h->B; ++b)
      if (h->valid[b] != n_valid)
        return fail(BMC_ERR_STATE, "n_valid=%d but row %d holds %d", n_valid, b, h->valid[b]);
  }
  if (min_valid(h) == 0) return fail(BMC_ERR_ARG, "a batch row has no committed token");
  const int t = 1 + h->staged;
  const size_t q_bytes = (size_t)h->B * h->H_q * t * h->row_bytes;
  const size_t o_bytes = (size_t)h->B * h->H_q * t * h->D * sizeof(float);
  const void* qd = nullptr;
  rc = device_inputs(h, 2, &Q, &q_bytes, 1, &qd);
  if (rc) return rc;
  const int out_kind = ptr_kind(O);
  const bool host_out = out_kind != 0;
  float* od = O;
  if (host_out) {
    // the previous download from the staging output must have finished
    if (h->hio && h->hio->out_used)
      CK(h, cudaStreamWaitEvent(h->stream, h->hio->out_free, 0), "wait");
    if (h->stage_out_bytes < o_bytes) {
      if (h->stage_out) cudaFreeAsync(h->stage_out, h->stream);
      h->stage_out = nullptr;
      h->stage_out_bytes = 0;
      CK(h, cudaMallocAsync((void**)&h->stage_out, o_bytes, h->stream), "stage_out");
      h->stage_out_bytes = o_bytes;
    }
    od = h->stage_out;
  }
  rc = launch_sdpa_layer(h, qd, od, t);
  if (rc) return rc;
  if (host_out) {
    if (out_kind == 1) {   // pinned: download on the handle's download stream
      rc = ensure_hio(h);
      if (rc) return rc;
      HostIO* x = h->hio;
      CK(h, cudaEventRecord(x->out_ready, h->stream), "event");
      CK(h, cudaStreamWaitEvent(x->down, x->out_ready, 0), "wait");
      CK(h, cudaMemcpyAsync(O, od, o_bytes, cudaMemcpyDeviceToHost, x->down), "D2H");
      CK(h, cudaEventRecord(x->out_free, x->down), "event");
      x->out_used = true;
    } else {
      CK(h, cudaMemcpyAsync(O, od, o_bytes, cudaMemcpyDeviceToHost, h->stream), "D2H");
      CK(h, cudaStreamSynchronize(h->stream), "sync");
    }
  }
  return 0;
}

int bmc_admissible(bmc_t h, int k) {
  int rc = enter(h);
  if (rc) return rc;
  if (k < 0) return fail(BMC_ERR_ARG, "k=%d < 0", k);
  if (h->staged > 0) return fail(BMC_ERR_STATE, "drafts already staged");
  const long long mv = max_valid(h);
  if (mv >= h->N_max) return fail(BMC_ERR_CAPACITY, "cache full (N_max=%d)", h->N_max);
  // state after the append: growth when full, then admission
  // into the free rows; ITERATIVE is limited by N_max only
  const long long mv1 = mv + 1;
  if (h->pol == BMC_POLICY_ITERATIVE) return (int)std::min<long long>(k, h->N_max - mv1);
  long long cap = h->cap;
  if (h->pol == BMC_POLICY_BMC && mv == h->cap) cap = std::min<long long>(h->cap + h->r, h->N_max);
  return (int)std::min<long long>(k, cap - mv1);
}

static int spec_step_host(const bmc_t* hs, int L, const void* const* K, const void* const* V,
                          const void* const* Kd, const void* const* Vd, int k,
                          const void* const* Q, float* const* O);

// Token-tree form of the drafts just written by spec_write_impl (parent
// validated by the caller): ancestor masks for the verify kernels.
static void set_tree(bmc_t h, const int* parent, int k_adm) {
  for (int i = 0; i < 32; ++i) h->anc[i] = 0;
  for (int i = 0; i < k_adm; ++i)
    h->anc[i] = (1u << i) | (parent[i] >= 0 ? h->anc[parent[i]] : 0u);
  h->tree = k_adm > 0;
}

static int check_parents(const int* parent, int k) {
  if (k > 32) return fail(BMC_ERR_UNSUPPORTED, "token trees of more than 32 nodes");
  if (k > 0 && !parent) return fail(BMC_ERR_ARG, "parent is null");
  for (int i = 0; i < k; ++i)
    if (parent[i] < -1 || parent[i] >= i)
      return fail(BMC_ERR_ARG, "parent[%d]=%d not in [-1, %d) (breadth-first order)", i, parent[i], i);
  return 0;
}

static int spec_step_impl(const bmc_t* hs, int L, const void* const* K, const void* const* V,
                          const void* const* Kd, const void* const* Vd, int k,
                          const int* parent, const void* const* Q, float* const* O);

int bmc_spec_step(const bmc_t* hs, int L, const void* const* K, const void* const* V,
                  const void* const* Kd, const void* const* Vd, int k, const void* const* Q,
                  float* const* O) {
  return spec_step_impl(hs, L, K, V, Kd, Vd, k, nullptr, Q, O);
}

int bmc_spec_step_tree(const bmc_t* hs, int L, const void* const* K, const void* const* V,
                       const void* const* Kd, const void* const* Vd, int k,
                       const int* parent_host, const void* const* Q, float* const* O) {
  if (k < 0) return fail(BMC_ERR_ARG, "k=%d < 0", k);
  int rc = check_parents(parent_host, k);
  if (rc) return rc;
  return spec_step_impl(hs, L, K, V, Kd, Vd, k, parent_host, Q, O);
}

static int spec_step_impl(const bmc_t* hs, int L, const void* const* K, const void* const* V,
                          const void* const* Kd, const void* const* Vd, int k,
                          const int* parent, const void* const* Q, float* const* O) {
  if (!hs || L < 1 || !K || !V || !Q || !O || k < 0 || (k > 0 && (!Kd || !Vd)))
    return fail(BMC_ERR_ARG, "null argument or k < 0");
  if (!parent) {
    // all-host arguments take the pipelined host-I/O path
    bool all_host = true;
    for (int l = 0; l < L && all_host; ++l)
      if (!K[l] || !V[l] || !Q[l] || !O[l] || ptr_kind(K[l]) == 0 || ptr_kind(V[l]) == 0 ||
          ptr_kind(Q[l]) == 0 || ptr_kind(O[l]) == 0 ||
          (k > 0 && (!Kd[l] || !Vd[l] || ptr_kind(Kd[l]) == 0 || ptr_kind(Vd[l]) == 0)))
        all_host = false;
    if (all_host) {
      for (int l = 1; l < L; ++l)
        if (hs[l]->B != hs[0]->B || hs[l]->H_kv != hs[0]->H_kv || hs[l]->H_q != hs[0]->H_q ||
            hs[l]->D != hs[0]->D || hs[l]->dt != hs[0]->dt || hs[l]->stream != hs[0]->stream ||
            hs[l]->device != hs[0]->device)
          return fail(BMC_ERR_ARG, "host-I/O speculative step needs layers of one shape and stream");
      return spec_step_host(hs, L, K, V, Kd, Vd, k, Q, O);
    }
  }
  // validate every layer before enqueueing anything; all layers must admit
  // the same number of drafts (they share the step sequence)
  int k_adm = -1;
  for (int l = 0; l < L; ++l) {
    const int a = bmc_admissible(hs[l], k);
    if (a < 0) return a;
    if (k_adm >= 0 && a != k_adm)
      return fail(BMC_ERR_STATE, "layer %d admits %d drafts, layer 0 %d", l, a, k_adm);
    k_adm = a;
    if (!K[l] || !V[l] || !Q[l] || !O[l] || (k > 0 && (!Kd[l] || !Vd[l])))
      return fail(BMC_ERR_ARG, "layer %d: null tensor", l);
    if (ptr_kind(Q[l]) != 0 || ptr_kind(O[l]) != 0)
      return fail(BMC_ERR_ARG, "layer %d: bmc_spec_step takes device Q and O", l);
  }
  const int t = 1 + k_adm;
  // one launch for the layers when they share shape, stream, lengths and
  // capacity and the kernel takes several layers (CUDA cores, or the
  // keys-on-lanes tcgen05 kernel up to M = 80); else one launch per layer.
  // Decided on the state before the appends (layers that agree now agree
  // after them: they see the same step).
  const bmc_t h0 = hs[0];
  bool fused = true;
  for (int l = 1; l < L; ++l) {
    const bmc_t a = hs[l];
    if (a->B != h0->B || a->H_kv != h0->H_kv || a->H_q != h0->H_q || a->D != h0->D ||
        a->dt != h0->dt || a->stream != h0->stream || a->device != h0->device ||
        a->valid != h0->valid || a->cap != h0->cap || a->attn_path != h0->attn_path ||
        a->skip_padding != h0->skip_padding || a->pol != h0->pol || a->r != h0->r ||
        a->N_max != h0->N_max || a->copy_on_read != h0->copy_on_read)
      fused = false;
  }
  const int M = (h0->H_q / h0->H_kv) * t;
  const bool tc = h0->attn_path >= 2 ||
                  (h0->attn_path == 0 && M > kTcMinM && bmc::attn_tc_supported(h0->D, h0->dt, M));
  const bool tck = tc && h0->attn_path != 3 && bmc::attn_tck_supported(h0->D, h0->dt, M);
  if (tc && !tck) fused = false;
  // everything that can fail without touching device memory is checked on
  // every layer before any layer is mutated
  for (int l = 0; l < L; ++l) {
    const bmc_t h = hs[l];
    const int Ml = (h->H_q / h->H_kv) * t;
    const bool tcl = h->attn_path >= 2 ||
                     (h->attn_path == 0 && Ml > kTcMinM && bmc::attn_tc_supported(h->D, h->dt, Ml));
    if (h->attn_path == 4 && !bmc::attn_tck_supported(h->D, h->dt, Ml))
      return fail(BMC_ERR_UNSUPPORTED, "layer %d: keys-on-lanes tcgen05 path needs bf16, D=128, G*t<=80", l);
    if (tcl && !bmc::attn_tc_supported(h->D, h->dt, Ml))
      return fail(BMC_ERR_UNSUPPORTED, "layer %d: tcgen05 path needs bf16, D=128, G*t<=128", l);
    if (tcl) {
      int rc = ensure_workspace(h, Ml);
      if (rc) return rc;
    }
  }
  if (!fused) {
    // appends and drafts of every layer, then the launches: an error in the
    // first loop rolls the layers back (nothing launched yet)
    for (int l = 0; l < L; ++l) {
      int rc = append_impl(hs[l], K[l], V[l]);
      if (rc) return rollback_chunk(hs, 0, l, l, rc);
      if (!rc && k > 0) {
        rc = spec_write_impl(hs[l], Kd[l], Vd[l], k);
        if (rc >= 0 && parent) set_tree(hs[l], parent, rc);
        if (rc > 0) rc = 0;
      }
      if (rc) return rollback_chunk(hs, 0, l + 1, l + 1, rc);
    }
    for (int l = 0; l < L; ++l) {
      int rc = launch_sdpa_layer(hs[l], Q[l], O[l], t);
      if (rc) return rc;
    }
    return k_adm;
  }
  // Layers in chunks of kMaxLayersPerLaunch: appends + drafts (growths
  // deferred to the attention, copy-on-read), the chunk's verify launch, then
  // the old buffers are released (at most one chunk holds old + new buffers).
  std::vector<bmc::AttnLayer> layers(L);
  const int nchunks = (L + bmc::kMaxLayersPerLaunch - 1) / bmc::kMaxLayersPerLaunch;
  const bool rev = chunks_reversed(h0);
  for (int ci = 0; ci < nchunks; ++ci) {
    const int l0 = (rev ? nchunks - 1 - ci : ci) * bmc::kMaxLayersPerLaunch;
    const int nl = std::min(bmc::kMaxLayersPerLaunch, L - l0);
    for (int l = l0; l < l0 + nl; ++l) {
      const bool defer = hs[l]->copy_on_read && !hs[l]->skip_padding;
      int rc = append_fused(hs, l0, l, K[l], V[l], defer);
      if (rc) return rollback_chunk(hs, l0, l, l, rc);
      if (k > 0) {
        rc = spec_write_impl(hs[l], Kd[l], Vd[l], k);
        if (rc < 0) return rollback_chunk(hs, l0, l + 1, l + 1, rc);
        if (parent) set_tree(hs[l], parent, rc);
      }
    }
    // descriptors only after every append of the chunk: an OOM fallback in
    // append_fused may have carried out earlier layers' deferred growths
    for (int l = l0; l < l0 + nl; ++l) fill_layer(hs[l], Q[l], O[l], &layers[l]);
    bmc::AttnStepArgs a;
    fill_args(hs[l0], t, &a);
    a.L = nl;
    a.layers = &layers[l0];
    if (tck) {
      a.ctas = std::min(h0->attn_ctas, h0->num_sms);
      int rc = launch_tck_chunk(h0, a, &layers[l0], nl);
      if (rc) return rc;
    } else {
      CK(h0, bmc::launch_attn_step(a, h0->num_sms, h0->stream), "attn_step");
    }
    for (int l = l0; l < l0 + nl; ++l) {
      int rc = cor_release(hs[l]);
      if (rc) return rc;
    }
  }
  for (int l = 0; l < L; ++l) {
    hs[l]->n_app = hs[l]->n_draft = 0;
    account_sdpa(hs[l], t);
    int rc = inputs_consumed(hs[l]);
    if (rc) return rc;
  }
  return k_adm;
}


static int decode_step_host(const bmc_t* hs, int L, const void* const* K, const void* const* V,
                            const void* const* Q, float* const* O, int n_valid);

int bmc_decode_step(const bmc_t* hs, int L, const void* const* K, const void* const* V,
                    const void* const* Q, float* const* O, int n_valid) {
  if (!hs || L < 1 || !K || !V || !Q || !O) return fail(BMC_ERR_ARG, "null argument");
  {
    // all-host arguments take the pipelined host-I/O path
    bool all_host = true;
    for (int l = 0; l < L && all_host; ++l)
      if (!K[l] || !V[l] || !Q[l] || !O[l] || ptr_kind(K[l]) == 0 || ptr_kind(V[l]) == 0 ||
          ptr_kind(Q[l]) == 0 || ptr_kind(O[l]) == 0)
        all_host = false;
    if (all_host) return decode_step_host(hs, L, K, V, Q, O, n_valid);
  }
  // validate every layer before enqueueing anything
  for (int l = 0; l < L; ++l) {
    bmc_t h = hs[l];
    int rc = enter(h);
    if (rc) return rc;
    if (!K[l] || !V[l] || !Q[l] || !O[l]) return fail(BMC_ERR_ARG, "layer %d: null tensor", l);
    if (h->staged > 0) return fail(BMC_ERR_STATE, "layer %d: drafts are staged", l);
    if (max_valid(h) >= h->N_max) return fail(BMC_ERR_CAPACITY, "layer %d: cache full", l);
    if (n_valid == 0) return fail(BMC_ERR_ARG, "n_valid == 0");
    if (n_valid != BMC_PER_ROW)
      for (int b = 0; b < h->B; ++b)
        if (h->valid[b] + 1 != n_valid)
          return fail(BMC_ERR_STATE, "layer %d: n_valid=%d but row %d will hold %d", l, n_valid,
                      b, h->valid[b] + 1);
  }
  // one launch for all layers when they share shape, dtype, stream and lengths
  bool fused = true;
  for (int l = 1; l < L; ++l) {
    const bmc_t a = hs[0], b = hs[l];
    if (a->B != b->B || a->H_kv != b->H_kv || a->H_q != b->H_q || a->D != b->D ||
        a->dt != b->dt || a->stream != b->stream || a->device != b->device || a->valid != b->valid)
      fused = false;
  }
  for (int l = 0; l < L; ++l)
    if (ptr_kind(Q[l]) != 0 || ptr_kind(O[l]) != 0) fused = false;
  // GQA groups large enough for the tensor cores take the tcgen05 kernel: the
  // keys-on-lanes kernel fuses the layers (G <= 80), the other runs per layer
  const bmc_t h0 = hs[0];
  const int G = h0->H_q / h0->H_kv;
  const bool tc = h0->attn_path != 1 && (h0->attn_path >= 2 || G > kTcMinM) &&
                  bmc::attn_tc_supported(h0->D, h0->dt, G);
  const bool tck = tc && h0->attn_path != 3 && bmc::attn_tck_supported(h0->D, h0->dt, G);
  for (int l = 1; l < L && tck; ++l)
    if (hs[l]->attn_path != h0->attn_path) fused = false;
  if (tc && !tck) fused = false;
  if (fused && tck)   // workspaces before any layer is mutated
    for (int l = 0; l < L; ++l) {
      int rc = ensure_workspace(hs[l], G);
      if (rc) return rc;
    }
  if (!fused) {
    for (int l = 0; l < L; ++l) {
      int rc = bmc_append(hs[l], K[l], V[l]);
      if (rc) return rc;
      rc = bmc_sdpa(hs[l], Q[l], n_valid, O[l]);
      if (rc) return rc;
    }
    return 0;
  }
  // Layers in chunks of kMaxLayersPerLaunch: appends (growths deferred to
  // the attention, copy-on-read), then the chunk's launch, then the old
  // buffers are released -- so at most one chunk holds old + new buffers.
  std::vector<bmc::AttnLayer> layers(L);
  const int nchunks = (L + bmc::kMaxLayersPerLaunch - 1) / bmc::kMaxLayersPerLaunch;
  const bool rev = chunks_reversed(h0);
  for (int ci = 0; ci < nchunks; ++ci) {
    const int l0 = (rev ? nchunks - 1 - ci : ci) * bmc::kMaxLayersPerLaunch;
    const int nl = std::min(bmc::kMaxLayersPerLaunch, L - l0);
    for (int l = l0; l < l0 + nl; ++l) {
      // copy-on-read growth (BMC policy; CUDA-core or keys-on-lanes kernel;
      // all cap rows streamed)
      const bool defer = hs[l]->copy_on_read && !hs[l]->skip_padding;
      int rc = append_fused(hs, l0, l, K[l], V[l], defer);
      if (rc) return rollback_chunk(hs, l0, l, l, rc);
    }
    // descriptors only after every append of the chunk: an OOM fallback in
    // append_fused may have carried out earlier layers' deferred growths
    for (int l = l0; l < l0 + nl; ++l) fill_layer(hs[l], Q[l], O[l], &layers[l]);
    bmc::AttnStepArgs a;
    fill_args(hs[l0], 1, &a);
    a.L = nl;
    a.layers = &layers[l0];
    if (tck) {
      a.ctas = std::min(h0->attn_ctas, h0->num_sms);
      int rc = launch_tck_chunk(h0, a, &layers[l0], nl);
      if (rc) return rc;
    } else {
      CK(hs[0], bmc::launch_attn_step(a, hs[0]->num_sms, hs[0]->stream), "attn_step");
    }
    for (int l = l0; l < l0 + nl; ++l) {
      int rc = cor_release(hs[l]);
      if (rc) return rc;
    }
  }
  for (int l = 0; l < L; ++l) {
    hs[l]->n_app = hs[l]->n_draft = 0;
    account_sdpa(hs[l], 1);
    int rc = inputs_consumed(hs[l]);
    if (rc) return rc;
  }
  return 0;
}

// Copy L per-layer blocks of sz bytes.  One cudaMemcpyAsync when both sides
// are address-contiguous across the layers and the runtime accepts the span
// (two pinned allocations can merely abut: the span then crosses them and the
// call fails with cudaErrorInvalidValue before enqueueing anything, so the
// copies go layer by layer); else one copy per layer.
static cudaError_t copy_layers(void* const* dst, const void* const* src, size_t sz, int L,
                               cudaMemcpyKind kind, cudaStream_t s) {
  bool contiguous = true;
  for (int l = 1; l < L && contiguous; ++l)
    if ((const char*)src[l] != (const char*)src[0] + sz * l ||
        (char*)dst[l] != (char*)dst[0] + sz * l)
      contiguous = false;
  if (contiguous) {
    cudaError_t e = cudaMemcpyAsync(dst[0], src[0], sz * L, kind, s);
    if (e != cudaErrorInvalidValue) return e;
    cudaGetLastError();   // not sticky; fall back to per-layer copies
  }
  for (int l = 0; l < L; ++l) {
    cudaError_t e = cudaMemcpyAsync(dst[l], src[l], sz, kind, s);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// The host-I/O pipeline of the first layer's handle, with staging slots of at
// least per_in / per_out bytes (grown on demand; growing syncs the handle).
static int pipe_ensure(bmc_t h0, size_t per_in, size_t per_out, Pipe** out) {
  Pipe* pp = h0->pipe;
  if (!pp || pp->in_bytes < per_in || pp->out_bytes < per_out) {
    if (pp) {
      cudaStreamSynchronize(h0->stream);
      per_in = std::max(per_in, pp->in_bytes);
      per_out = std::max(per_out, pp->out_bytes);
      pipe_destroy(pp);
    }
    pp = new Pipe();
    h0->pipe = pp;
    CK(h0, cudaStreamCreateWithFlags(&pp->copy, cudaStreamNonBlocking), "pipe stream");
    CK(h0, cudaStreamCreateWithFlags(&pp->down, cudaStreamNonBlocking), "pipe stream");
    for (int i = 0; i < 2; ++i) {
      CK(h0, cudaEventCreateWithFlags(&pp->in_ready[i], cudaEventDisableTiming), "pipe event");
      CK(h0, cudaEventCreateWithFlags(&pp->compute_done[i], cudaEventDisableTiming), "pipe event");
      CK(h0, cudaEventCreateWithFlags(&pp->out_done[i], cudaEventDisableTiming), "pipe event");
      CK(h0, cudaMalloc((void**)&pp->in_slot[i], per_in), "pipe staging");
      CK(h0, cudaMalloc((void**)&pp->out_slot[i], per_out), "pipe staging");
    }
    pp->in_bytes = per_in;
    pp->out_bytes = per_out;
  }
  *out = pp;
  return 0;
}

// Host-pointer decode step: stage every layer's K, V, Q on the copy stream
// into slot s%2, run the device-pointer step on the compute stream, and copy
// the outputs back on the copy stream.  Pinned host buffers make all copies
// asynchronous (outputs are readable after bmc_sync); inputs must stay
// unchanged until the copy stream has passed them.
static int decode_step_host(const bmc_t* hs, int L, const void* const* K, const void* const* V,
                            const void* const* Q, float* const* O, int n_valid) {
  bmc_t h0 = hs[0];
  int rc = enter(h0);
  if (rc) return rc;
  for (int l = 1; l < L; ++l)
    if (hs[l]->B != h0->B || hs[l]->H_kv != h0->H_kv || hs[l]->H_q != h0->H_q ||
        hs[l]->D != h0->D || hs[l]->dt != h0->dt || hs[l]->stream != h0->stream ||
        hs[l]->device != h0->device)
      return fail(BMC_ERR_ARG, "host-I/O decode step needs layers of one shape and stream");
  const size_t kv = (size_t)h0->U * h0->row_bytes;
  const size_t q = (size_t)h0->B * h0->H_q * h0->row_bytes;
  const size_t o = (size_t)h0->B * h0->H_q * h0->D * sizeof(float);
  // staging slot: [K of every layer][V ...][Q ...]; output slot [O ...]
  const size_t per_in = (2 * kv + q) * L, per_out = o * L;
  Pipe* pp = nullptr;
  rc = pipe_ensure(h0, per_in, per_out, &pp);
  if (rc) return rc;
  const int slot = (int)(pp->step & 1);
  std::vector<const void*> dK(L), dV(L), dQ(L);
  std::vector<float*> dO(L);
  char* kb = pp->in_slot[slot];
  char* vb = kb + kv * L;
  char* qb = vb + kv * L;
  char* ob = pp->out_slot[slot];
  for (int l = 0; l < L; ++l) {
    dK[l] = kb + kv * l;
    dV[l] = vb + kv * l;
    dQ[l] = qb + q * l;
    dO[l] = reinterpret_cast<float*>(ob + o * l);
  }
  // one copy per tensor when the caller's per-layer buffers are contiguous
  auto h2d = [&](char* dst, const void* const* src, size_t sz) -> int {
    std::vector<void*> d(L);
    for (int l = 0; l < L; ++l) d[l] = dst + sz * l;
    CK(h0, copy_layers(d.data(), src, sz, L, cudaMemcpyHostToDevice, pp->copy), "H2D");
    return 0;
  };
  if (pp->primed[slot]) CK(h0, cudaStreamWaitEvent(pp->copy, pp->compute_done[slot], 0), "wait");
  if ((rc = h2d(kb, K, kv)) || (rc = h2d(vb, V, kv)) || (rc = h2d(qb, Q, q))) return rc;
  CK(h0, cudaEventRecord(pp->in_ready[slot], pp->copy), "record");
  CK(h0, cudaStreamWaitEvent(h0->stream, pp->in_ready[slot], 0), "wait");
  if (pp->primed[slot]) CK(h0, cudaStreamWaitEvent(h0->stream, pp->out_done[slot], 0), "wait");
  rc = bmc_decode_step(hs, L, dK.data(), dV.data(), dQ.data(), dO.data(), n_valid);
  if (rc) return rc;
  CK(h0, cudaEventRecord(pp->compute_done[slot], h0->stream), "record");
  CK(h0, cudaStreamWaitEvent(pp->down, pp->compute_done[slot], 0), "wait");
  CK(h0, copy_layers((void* const*)O, (const void* const*)dO.data(), o, L, cudaMemcpyDeviceToHost,
                     pp->down), "D2H");
  CK(h0, cudaEventRecord(pp->out_done[slot], pp->down), "record");
  pp->primed[slot] = true;
  pp->step += 1;
  return 0;
}

// Host-pointer speculative step (the end-to-end form of bmc_spec_step): every
// layer's K, V, drafts and verify queries are staged on the copy stream into
// slot s%2, the device-pointer step runs on the compute stream, the outputs
// go back on the download stream (as decode_step_host).
static int spec_step_host(const bmc_t* hs, int L, const void* const* K, const void* const* V,
                          const void* const* Kd, const void* const* Vd, int k,
                          const void* const* Q, float* const* O) {
  bmc_t h0 = hs[0];
  int rc = enter(h0);
  if (rc) return rc;
  const int k_adm = bmc_admissible(h0, k);
  if (k_adm < 0) return k_adm;
  const int t = 1 + k_adm;
  const size_t kv = (size_t)h0->U * h0->row_bytes;
  const size_t kd = k_adm > 0 ? (size_t)h0->U * k * h0->row_bytes : 0;
  const size_t q = (size_t)h0->B * h0->H_q * t * h0->row_bytes;
  const size_t o = (size_t)h0->B * h0->H_q * t * h0->D * sizeof(float);
  Pipe* pp = nullptr;
  rc = pipe_ensure(h0, (2 * kv + 2 * kd + q) * L, o * L, &pp);
  if (rc) return rc;
  const int slot = (int)(pp->step & 1);
  std::vector<const void*> dK(L), dV(L), dKd(L), dVd(L), dQ(L);
  std::vector<float*> dO(L);
  char* base = pp->in_slot[slot];
  char* ob = pp->out_slot[slot];
  for (int l = 0; l < L; ++l) {
    dK[l] = base + kv * l;
    dV[l] = base + kv * (L + l);
    dKd[l] = base + kv * 2 * L + kd * l;
    dVd[l] = base + kv * 2 * L + kd * (L + l);
    dQ[l] = base + (kv + kd) * 2 * L + q * l;
    dO[l] = reinterpret_cast<float*>(ob + o * l);
  }
  if (pp->primed[slot]) CK(h0, cudaStreamWaitEvent(pp->copy, pp->compute_done[slot], 0), "wait");
  // one copy per tensor when the caller's per-layer buffers are contiguous
  // (the staging slot keeps every tensor's layers contiguous), else per layer
  auto h2d = [&](const std::vector<const void*>& dst, const void* const* src, size_t sz) -> int {
    CK(h0, copy_layers((void* const*)dst.data(), src, sz, L, cudaMemcpyHostToDevice, pp->copy),
       "H2D");
    return 0;
  };
  if ((rc = h2d(dK, K, kv)) || (rc = h2d(dV, V, kv)) || (kd && (rc = h2d(dKd, Kd, kd))) ||
      (kd && (rc = h2d(dVd, Vd, kd))) || (rc = h2d(dQ, Q, q)))
    return rc;
  CK(h0, cudaEventRecord(pp->in_ready[slot], pp->copy), "record");
  CK(h0, cudaStreamWaitEvent(h0->stream, pp->in_ready[slot], 0), "wait");
  if (pp->primed[slot]) CK(h0, cudaStreamWaitEvent(h0->stream, pp->out_done[slot], 0), "wait");
  rc = bmc_spec_step(hs, L, dK.data(), dV.data(), kd ? dKd.data() : dK.data(),
                     kd ? dVd.data() : dV.data(), kd ? k : 0, dQ.data(), dO.data());
  if (rc < 0) return rc;
  CK(h0, cudaEventRecord(pp->compute_done[slot], h0->stream), "record");
  CK(h0, cudaStreamWaitEvent(pp->down, pp->compute_done[slot], 0), "wait");
  CK(h0, copy_layers((void* const*)O, (const void* const*)dO.data(), o, L, cudaMemcpyDeviceToHost,
                     pp->down), "D2H");
  CK(h0, cudaEventRecord(pp->out_done[slot], pp->down), "record");
  pp->primed[slot] = true;
  pp->step += 1;
  return k_adm;
}

static int commit_impl(bmc_t h, const int* m) {
  if (h->n_app || h->n_draft) {
    int rc = flush_pending(h);
    if (rc) return rc;
  }
  bmc::ZeroArgs z;
  z.k[0] = h->kbuf.ptr;
  z.v[0] = h->vbuf.ptr;
  z.L = 1;
  z.B = h->B;
  z.H_kv = h->H_kv;
  z.cap = h->cap;
  z.row_bytes = h->row_bytes;
  z.max_rows = 0;
  for (int b = 0; b < h->B; ++b) {
    z.row_lo[b] = h->valid[b] + m[b];        // rejected drafts (reading R9)
    z.row_hi[b] = h->valid[b] + h->staged;
    z.max_rows = std::max(z.max_rows, h->staged - m[b]);
  }
  if (z.max_rows > 0) CK(h, bmc::launch_zero_rows(z, h->stream), "zero_rows");
  for (int b = 0; b < h->B; ++b) h->valid[b] += m[b];
  h->staged = 0;
  h->tree = 0;
  return 0;
}

// The accepted paths must be root-first, parent-linked node lists of the
// staged tree (or chain) of h.
static int check_path(bmc_t h, const int* path_host, const int* m_host, int max_depth) {
  if (!m_host || max_depth < 0) return fail(BMC_ERR_ARG, "null argument");
  for (int b = 0; b < h->B; ++b) {
    const int m = m_host[b];
    if (m < 0 || m > max_depth || m > h->staged || m > 32)
      return fail(BMC_ERR_ARG, "path length %d of row %d invalid (staged %d)", m, b, h->staged);
    if (m > 0 && !path_host) return fail(BMC_ERR_ARG, "null path");
    for (int i = 0; i < m; ++i) {
      const int x = path_host[b * max_depth + i];
      if (x < 0 || x >= h->staged) return fail(BMC_ERR_ARG, "path node %d out of range", x);
      const int par = h->tree ? (int)(31 - __builtin_clz(h->anc[x] & ~(1u << x) | 1u)) : x - 1;
      const int has_par = h->tree ? ((h->anc[x] & ~(1u << x)) != 0) : (x > 0);
      const int want = i == 0 ? -1 : path_host[b * max_depth + i - 1];
      if ((has_par ? par : -1) != want) return fail(BMC_ERR_ARG, "row %d: path is not parent-linked", b);
    }
  }
  return 0;
}

static void fill_path(bmc_t h, const int* path_host, const int* m_host, int max_depth,
                      bmc::PathArgs* a) {
  a->B = h->B;
  a->H_kv = h->H_kv;
  a->staged = h->staged;
  a->cap = h->cap;
  a->row_bytes = h->row_bytes;
  for (int b = 0; b < h->B; ++b) {
    a->valid[b] = h->valid[b];
    a->m[b] = (unsigned char)m_host[b];
    for (int i = 0; i < m_host[b]; ++i) a->path[b][i] = (unsigned char)path_host[b * max_depth + i];
  }
}

static void path_committed(bmc_t h, const int* m_host) {
  for (int b = 0; b < h->B; ++b) h->valid[b] += m_host[b];
  h->staged = 0;
  h->tree = 0;
}

int bmc_commit_path(bmc_t h, const int* path_host, const int* m_host, int max_depth) {
  int rc = enter(h);
  if (rc) return rc;
  rc = check_path(h, path_host, m_host, max_depth);
  if (rc) return rc;
  if (h->n_app || h->n_draft) {
    rc = flush_pending(h);
    if (rc) return rc;
  }
  bmc::PathArgs a;
  fill_path(h, path_host, m_host, max_depth, &a);
  a.L = 1;
  a.k[0] = h->kbuf.ptr;
  a.v[0] = h->vbuf.ptr;
  CK(h, bmc::launch_commit_path(a, h->stream), "commit_path");
  path_committed(h, m_host);
  return 0;
}

int bmc_commit_path_step(const bmc_t* hs, int L, const int* path_host, const int* m_host,
                         int max_depth) {
  if (!hs || L < 1) return fail(BMC_ERR_ARG, "null argument or L < 1");
  // validate every layer before enqueueing anything (as bmc_commit_path)
  for (int l = 0; l < L; ++l) {
    int rc = enter(hs[l]);
    if (rc) return rc;
    if (hs[l]->B != hs[0]->B) return fail(BMC_ERR_ARG, "layer %d: batch differs from layer 0", l);
    rc = check_path(hs[l], path_host, m_host, max_depth);
    if (rc) return rc;
  }
  const bmc_t h0 = hs[0];
  bool fused = true;
  for (int l = 0; l < L; ++l) {
    const bmc_t a = hs[l];
    if (a->n_app || a->n_draft || a->H_kv != h0->H_kv || a->stream != h0->stream ||
        a->device != h0->device || a->cap != h0->cap || a->row_bytes != h0->row_bytes ||
        a->staged != h0->staged || a->valid != h0->valid)
      fused = false;
  }
  if (!fused) {
    for (int l = 0; l < L; ++l) {
      int rc = bmc_commit_path(hs[l], path_host, m_host, max_depth);
      if (rc) return rc;
    }
    return 0;
  }
  // one launch per kMaxZeroLayers layers: accepted rows moved, the rest zeroed
  bmc::PathArgs a;
  fill_path(h0, path_host, m_host, max_depth, &a);
  for (int l0 = 0; l0 < L; l0 += bmc::kMaxZeroLayers) {
    a.L = std::min(bmc::kMaxZeroLayers, L - l0);
    for (int l = 0; l < a.L; ++l) {
      a.k[l] = hs[l0 + l]->kbuf.ptr;
      a.v[l] = hs[l0 + l]->vbuf.ptr;
    }
    CK(h0, bmc::launch_commit_path(a, h0->stream), "commit_path");
  }
  for (int l = 0; l < L; ++l) path_committed(hs[l], m_host);
  return 0;
}

int bmc_commit(bmc_t h, int n_accepted) {
  int rc = enter(h);
  if (rc) return rc;
  if (h->staged == 0 && n_accepted > 0) return fail(BMC_ERR_STATE, "nothing staged");
  if (n_accepted < 0 || n_accepted > h->staged)
    return fail(BMC_ERR_ARG, "n_accepted=%d outside [0, %d]", n_accepted, h->staged);
  if (h->tree && n_accepted > 0)
    return fail(BMC_ERR_STATE, "a staged token tree is committed with bmc_commit_path");
  std::vector<int> m(h->B, n_accepted);
  return commit_impl(h, m.data());
}

int bmc_commit_rows(bmc_t h, const int* n_accepted_host) {
  int rc = enter(h);
  if (rc) return rc;
  if (!n_accepted_host) return fail(BMC_ERR_ARG, "n_accepted is null");
  for (int b = 0; b < h->B; ++b) {
    if (h->staged == 0 && n_accepted_host[b] > 0) return fail(BMC_ERR_STATE, "nothing staged");
    if (n_accepted_host[b] < 0 || n_accepted_host[b] > h->staged)
      return fail(BMC_ERR_ARG, "n_accepted[%d]=%d outside [0, %d]", b, n_accepted_host[b],
                  h->staged);
    if (h->tree && n_accepted_host[b] > 0)
      return fail(BMC_ERR_STATE, "a staged token tree is committed with bmc_commit_path");
  }
  return commit_impl(h, n_accepted_host);
}

int bmc_commit_step(const bmc_t* hs, int L, const int* n_accepted_host) {
  if (!hs || L < 1 || !n_accepted_host) return fail(BMC_ERR_ARG, "null argument or L < 1");
  // validate every layer before enqueueing anything (as bmc_commit_rows)
  for (int l = 0; l < L; ++l) {
    const bmc_t h = hs[l];
    int rc = enter(h);
    if (rc) return rc;
    if (h->B != hs[0]->B) return fail(BMC_ERR_ARG, "layer %d: batch differs from layer 0", l);
    for (int b = 0; b < h->B; ++b) {
      const int m = n_accepted_host[b];
      if (h->staged == 0 && m > 0) return fail(BMC_ERR_STATE, "layer %d: nothing staged", l);
      if (m < 0 || m > h->staged)
        return fail(BMC_ERR_ARG, "n_accepted[%d]=%d outside [0, %d] (layer %d)", b, m, h->staged, l);
      if (h->tree && m > 0)
        return fail(BMC_ERR_STATE, "a staged token tree is committed with bmc_commit_path");
    }
  }
  const bmc_t h0 = hs[0];
  bool fused = true;
  for (int l = 0; l < L; ++l) {
    const bmc_t a = hs[l];
    if (a->n_app || a->n_draft || a->H_kv != h0->H_kv || a->stream != h0->stream ||
        a->device != h0->device || a->cap != h0->cap || a->row_bytes != h0->row_bytes ||
        a->staged != h0->staged || a->valid != h0->valid)
      fused = false;
  }
  if (!fused) {
    for (int l = 0; l < L; ++l) {
      int rc = enter(hs[l]);
      if (rc) return rc;
      rc = commit_impl(hs[l], n_accepted_host);
      if (rc) return rc;
    }
    return 0;
  }
  // one zero_rows launch per kMaxZeroLayers layers for the rejected drafts (reading R9)
  bmc::ZeroArgs z;
  z.B = h0->B;
  z.H_kv = h0->H_kv;
  z.cap = h0->cap;
  z.row_bytes = h0->row_bytes;
  z.max_rows = 0;
  for (int b = 0; b < h0->B; ++b) {
    z.row_lo[b] = h0->valid[b] + n_accepted_host[b];
    z.row_hi[b] = h0->valid[b] + h0->staged;
    z.max_rows = std::max(z.max_rows, h0->staged - n_accepted_host[b]);
  }
  if (z.max_rows > 0) {
    for (int l0 = 0; l0 < L; l0 += bmc::kMaxZeroLayers) {
      z.L = std::min(bmc::kMaxZeroLayers, L - l0);
      for (int l = 0; l < z.L; ++l) {
        z.k[l] = hs[l0 + l]->kbuf.ptr;
        z.v[l] = hs[l0 + l]->vbuf.ptr;
      }
      CK(h0, bmc::launch_zero_rows(z, h0->stream), "zero_rows");
    }
  }
  for (int l = 0; l < L; ++l) {
    const bmc_t h = hs[l];
    for (int b = 0; b < h->B; ++b) h->valid[b] += n_accepted_host[b];
    h->staged = 0;
    h->tree = 0;
  }
  return 0;
}

int bmc_destroy(bmc_t h) {
  if (!h) return fail(BMC_ERR_ARG, "null handle");
  cudaSetDevice(h->device);
  if (!h->sticky && h->cor) cor_materialize(h);
  if (!h->sticky && (h->n_app || h->n_draft)) flush_pending(h);
  cudaStreamSynchronize(h->stream);
  if (h->cor) {
    bmc::arena_release(h->arena, &h->cor_k, h->stream);
    bmc::arena_release(h->arena, &h->cor_v, h->stream);
  }
  pipe_destroy(h->pipe);
  h->pipe = nullptr;
  hio_destroy(h->hio);
  h->hio = nullptr;
  bmc::arena_release(h->arena, &h->kbuf, h->stream);
  bmc::arena_release(h->arena, &h->vbuf, h->stream);
  for (int i = 0; i < 3; ++i)
    if (h->stage_in[i]) cudaFreeAsync(h->stage_in[i], h->stream);
  if (h->stage_out) cudaFreeAsync(h->stage_out, h->stream);
  if (h->ws) cudaFreeAsync(h->ws, h->stream);
  if (h->counters) cudaFreeAsync(h->counters, h->stream);
  cudaStreamSynchronize(h->stream);
  bmc::arena_destroy(h->arena);
  cudaGetLastError();
  delete h;
  return 0;
}

int bmc_stats(bmc_t h, bmc_stats_t* out) {
  if (!h || !out) return fail(BMC_ERR_ARG, "null argument");
  *out = h->st;
  out->valid_min = min_valid(h);
  out->valid_max = max_valid(h);
  out->capacity = h->cap;
  out->staged = h->staged;
  return 0;
}

int bmc_kv_view(bmc_t h, void** K, void** V, int* cap) {
  int rc = enter(h);
  if (rc) return rc;
  if (h->n_app || h->n_draft) {
    rc = flush_pending(h);
    if (rc) return rc;
  }
  if (K) *K = h->kbuf.ptr;
  if (V) *V = h->vbuf.ptr;
  if (cap) *cap = (int)h->cap;
  return 0;
}

int bmc_read_cache(bmc_t h, void* K_dst, void* V_dst) {
  int rc = enter(h);
  if (rc) return rc;
  if (!K_dst || !V_dst) return fail(BMC_ERR_ARG, "null destination");
  if (h->n_app || h->n_draft) {
    rc = flush_pending(h);
    if (rc) return rc;
  }
  const size_t bytes = (size_t)h->U * h->cap * h->row_bytes;
  if (bytes == 0) return 0;
  CK(h, cudaMemcpyAsync(K_dst, h->kbuf.ptr, bytes, cudaMemcpyDefault, h->stream), "read K");
  CK(h, cudaMemcpyAsync(V_dst, h->vbuf.ptr, bytes, cudaMemcpyDefault, h->stream), "read V");
  if (!is_device_ptr(K_dst) || !is_device_ptr(V_dst))
    CK(h, cudaStreamSynchronize(h->stream), "sync");
  return 0;
}

int bmc_valid(bmc_t h, int* valid_host) {
  if (!h || !valid_host) return fail(BMC_ERR_ARG, "null argument");
  memcpy(valid_host, h->valid.data(), sizeof(int) * h->B);
  return 0;
}

int bmc_sync(bmc_t h) {
  int rc = enter(h);
  if (rc) return rc;
  if (h->n_app || h->n_draft) {
    rc = flush_pending(h);
    if (rc) return rc;
  }
  CK(h, cudaStreamSynchronize(h->stream), "sync");
  if (h->hio) {
    CK(h, cudaStreamSynchronize(h->hio->up), "sync upload stream");
    CK(h, cudaStreamSynchronize(h->hio->down), "sync download stream");
  }
  if (h->pipe) {
    CK(h, cudaStreamSynchronize(h->pipe->copy), "sync copy stream");
    CK(h, cudaStreamSynchronize(h->pipe->down), "sync copy stream");
  }
  return 0;
}

int bmc_set_option(bmc_t h, int key, long long value) {
  if (!h) return fail(BMC_ERR_ARG, "null handle");
  switch (key) {
    case BMC_OPT_ATTN_CTAS:
      if (value < 0) return fail(BMC_ERR_ARG, "ctas < 0");
      h->attn_ctas = (int)value;
      return 0;
    case BMC_OPT_ATTN_PATH:
      if (value < 0 || value > 4) return fail(BMC_ERR_ARG, "path");
      h->attn_path = (int)value;
      return 0;
    case BMC_OPT_ARENA:
      if (value < 0 || value > 2) return fail(BMC_ERR_ARG, "arena kind");
      h->arena_kind = (int)value;
      return 0;
    case BMC_OPT_SKIP_PADDING:
      if (value < 0 || value > 1) return fail(BMC_ERR_ARG, "skip padding");
      h->skip_padding = (int)value;
      return 0;
    case BMC_OPT_COPY_ON_READ:
      if (value < 0 || value > 1) return fail(BMC_ERR_ARG, "copy on read");
      h->copy_on_read = (int)value;
      return 0;
    case BMC_OPT_TCK_GROUPS:
      if (value != 0 && value != 2 && value != 3 && value != 4) return fail(BMC_ERR_ARG, "tck groups");
      h->tck_groups = (int)value;
      return 0;
    case BMC_OPT_TCK_PREFETCH:
      if (value < -1 || value > 64) return fail(BMC_ERR_ARG, "tck prefetch");
      h->tck_prefetch = (int)value;
      return 0;
    case BMC_OPT_FAULT_OOM:
      if (value < 0 || value > 1000000) return fail(BMC_ERR_ARG, "fault count");
      h->fault_oom = (int)value;
      return 0;
    default:
      return fail(BMC_ERR_ARG, "unknown option %d", key);
  }
}

int bmc_pool_reserve(int device, long long bytes) {
  if (bytes < 0) return fail(BMC_ERR_ARG, "bytes < 0");
  if (device < 0) {
    cudaError_t e = cudaGetDevice(&device);
    if (e != cudaSuccess) return cuda_fail(nullptr, e, "cudaGetDevice");
  }
  const int rc = bmc::pool_reserve(device, (size_t)bytes);
  if (rc) return fail(rc, "pool_reserve(%lld bytes) failed", bytes);
  return 0;
}

int bmc_region_reserve(int device, long long bytes) {
  if (bytes < 0) return fail(BMC_ERR_ARG, "bytes=%lld < 0", bytes);
  if (device < 0 && cudaGetDevice(&device) != cudaSuccess)
    return fail(BMC_ERR_CUDA, "cudaGetDevice failed");
  const int rc = bmc::region_reserve(device, (size_t)bytes);
  if (rc == BMC_ERR_STATE) return fail(rc, "growth region still holds live buffers");
  if (rc) return fail(rc, "region_reserve(%lld bytes) failed", bytes);
  return 0;
}

int bmc_pool_trim(int device) {
  if (device < 0) {
    cudaError_t e = cudaGetDevice(&device);
    if (e != cudaSuccess) return cuda_fail(nullptr, e, "cudaGetDevice");
  }
  const int rc = bmc::pool_trim(device);
  if (rc) return fail(rc, "pool_trim failed");
  return 0;
}

unsigned long long bmc_launch_count(void) { return bmc::launch_count(); }

int bmc_host_profile(long long* ns, long long* calls, int reset) {
  if (!ns || !calls) return fail(BMC_ERR_ARG, "null argument");
  bmc::host_time_read(ns, calls, reset != 0);
  return 0;
}

const char* bmc_last_error(void) { return g_err.c_str(); }

}  // extern "C"
