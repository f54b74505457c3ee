/*
 * bmc.h -- C ABI of the B200-native BMC decode hot path (libbmc.so).
 *
 * BMC = "Balancing Memory and Compute" (arXiv 2511.12031; PAPER.md is cited
 * as P:L<line>).  One handle holds ONE layer's K and V cache, each laid out
 * [B*H_kv][cap][D] row-major, contiguous per (batch, kv-head) unit, grown in
 * r-row chunks.  A model is L handles.
 *
 * Conventions for every call
 *   - Returns 0 (BMC_OK) or a negative bmc_status.  All argument/state
 *     validation happens BEFORE anything is enqueued, so an error leaves the
 *     handle unchanged.  bmc_last_error() gives a thread-local message.
 *   - Tensor pointers may be CUDA device pointers on the handle's device
 *     (the fast path) or host pointers (pageable or pinned).  Host inputs are
 *     copied to a device staging buffer inside the call (stream-ordered; a
 *     pinned input must not be modified until the stream has passed the
 *     call).  A pageable host output makes the call wait for its stream
 *     before returning; a pinned host output is written asynchronously (read
 *     it after bmc_sync or another stream synchronisation).
 *   - Work is stream-ordered on the handle's stream; device-pointer calls
 *     never synchronise the device.  The host tracks every length itself
 *     (no device->host reads on the hot path).
 *   - The caller owns K, V, K_draft, V_draft, Q, O and must keep device
 *     buffers alive until the stream has passed the call.  Rows given to
 *     bmc_append / bmc_spec_write are written into the cache by the NEXT
 *     call on the handle that touches it (normally bmc_sdpa, which fuses the
 *     write into the attention kernel): their device buffers must stay alive
 *     and unmodified until the stream has passed that call.  The library owns
 *     the cache memory (per-handle arena) and its workspace.
 *   - Single writer per handle.  Distinct handles are independent.
 *   - Inputs are stored bit-for-bit (no dtype conversion in append/spec);
 *     inputs must already be in the cache dtype.
 *   - Error codes:
 *       BMC_ERR_ARG        bad dims (<1, H_q % H_kv != 0, r outside [1,N_max]),
 *                          null pointers, k < 0, n_accepted outside [0, staged],
 *                          n_valid == 0 or any committed length == 0 at sdpa;
 *       BMC_ERR_STATE      append/spec_write while drafts are staged, n_valid
 *                          not equal to the committed length, commit of
 *                          n_accepted > 0 with nothing staged;
 *       BMC_ERR_CAPACITY   append when a row already holds N_max tokens;
 *       BMC_ERR_OOM        device memory exhausted;
 *       BMC_ERR_CUDA       CUDA error (sticky: the handle is usable only for
 *                          bmc_destroy);
 *       BMC_ERR_UNSUPPORTED D not in {64,128}, B > BMC_MAX_B, dtype not built.
 */
#ifndef BMC_H
#define BMC_H
#ifdef __cplusplus
extern "C" {
#endif

typedef struct bmc_ctx* bmc_t;

typedef enum {
  BMC_OK = 0,
  BMC_ERR_ARG = -1,
  BMC_ERR_STATE = -2,
  BMC_ERR_CAPACITY = -3,
  BMC_ERR_OOM = -4,
  BMC_ERR_CUDA = -5,
  BMC_ERR_UNSUPPORTED = -6
} bmc_status;

typedef enum { BMC_F32 = 0, BMC_BF16 = 1 } bmc_dtype;

/* Allocation policy.  BMC: grow by r rows when full.
   ITERATIVE: exact-size reallocation + copy for every new row block
   (the HuggingFace baseline).  UPFRONT: one N_max allocation,
   in-place writes, masked SDPA over all N_max rows. */
typedef enum { BMC_POLICY_BMC = 0, BMC_POLICY_ITERATIVE = 1, BMC_POLICY_UPFRONT = 2 } bmc_policy;

#define BMC_PER_ROW (-1) /* bmc_sdpa n_valid: use every batch row's own length */
#define BMC_MAX_B 256    /* batch rows per handle (per GPU shard) */

/* bmc_create: bf16 cache, BMC policy, current device, default stream.
   B batch rows, H_kv key/value heads, H_q query heads (GQA group
   G = H_q/H_kv; query head h reads kv head floor(h/G)),
   D head dim (64 or 128), r chunk rows (1 <= r <= N_max; T = N_max/r
   allocations), N_max maximum context.  The first allocation
   of min(r, N_max) zeroed rows happens here (UPFRONT: N_max rows;
   ITERATIVE: none). */
int bmc_create(int B, int H_kv, int H_q, int D, int r, int N_max, bmc_t* out);

/* As bmc_create with explicit dtype, policy, CUDA device ordinal (-1 =
   current) and stream (a cudaStream_t, NULL = the legacy default stream). */
int bmc_create_ex(int B, int H_kv, int H_q, int D, int r, int N_max, bmc_dtype dt,
                  bmc_policy pol, int device, void* cuda_stream, bmc_t* out);

/* bmc_append: KV cache update of one decode step.
   K, V: [B][H_kv][D] in the cache dtype.  Writes row valid_b of every unit
   of batch row b, then valid_b += 1.  BMC: if max_b valid_b == cap first
   grows to min(cap + r, N_max): new buffer, strided copy of the cap old rows
   of every unit, zero-fill of the new rows.  ITERATIVE: always
   reallocates to exactly max valid + 1 rows.  With BMC_OPT_COPY_ON_READ (the
   default) a BMC growth is left pending for the next bmc_sdpa, whose
   attention kernel copies the old rows while streaming them; any other call
   on the handle first carries the growth out with the realloc kernel.
   Contents and ledger are the same either way.  Errors: STATE if drafts are
   staged, CAPACITY if max valid == N_max. */
int bmc_append(bmc_t h, const void* K, const void* V);

/* The number of drafts an append followed by bmc_spec_write(k) would admit
   now (P:L867-869 admission after a possible growth): the t - 1
   of the next verify step.  Host-only, no device work.  Errors: STATE
   (drafts staged), CAPACITY (cache full), ARG (k < 0). */
int bmc_admissible(bmc_t h, int k);

/* One speculative-decoding iteration of L layers:
   for every layer bmc_append(K[l], V[l]) and bmc_spec_write(Kd[l], Vd[l], k),
   then the verify SDPA of all layers -- one persistent launch per 32 layers
   when the layers share shape, stream, lengths and capacity and the kernel
   takes several layers (the keys-on-lanes tcgen05 kernel for bf16, D = 128,
   M = G*t <= 80; CUDA cores for fp32 or D = 64), else one launch per layer.  K, V
   [B][H_kv][D], Kd, Vd [B][H_kv][k][D] (device or host, as bmc_append /
   bmc_spec_write); Q[l] DEVICE [B][H_q][t][D] and O[l] DEVICE
   [B][H_q][t][D] fp32 with t = 1 + bmc_admissible(hs[l], k) (every layer
   admits the same number).  Returns k_adm >= 0, or an error before anything
   is enqueued (ARG, STATE, CAPACITY, UNSUPPORTED; workspaces are allocated
   for every layer before any layer changes).  The 32-layer chunks are
   launched in layer order, or in reverse order when the layers' buffers sit
   at end 0 of the two-ended growth region (BMC_OPT_ARENA = 2: LIFO moves).
   OOM on a growth allocation: the layers of the chunks already launched
   have taken the step, every other layer is rolled back to its state before
   the call (a growth it completed stays: the retried step does not grow it
   again); bmc_valid tells the two apart.  Commit afterwards with bmc_commit_step
   (or per layer with bmc_commit / bmc_commit_rows).
   All-host form (the end-to-end call): when every K, V, Q, O (and Kd, Vd for
   k > 0) is a HOST pointer (pinned for asynchrony), the arguments are staged
   on the first layer's copy stream into double-buffered device slots, the
   step runs on the compute stream and O is copied back on a download stream;
   O is readable after bmc_sync(hs[0]), inputs reusable after the copy stream
   passed them (as bmc_decode_step's host form).  Mixed host / device
   arguments: K, V, Kd, Vd may be host (staged per call), Q and O must then be
   device pointers. */
int bmc_spec_step(const bmc_t* hs, int L, const void* const* K, const void* const* V,
                  const void* const* Kd, const void* const* Vd, int k,
                  const void* const* Q, float* const* O);

/* bmc_spec_step_tree: bmc_spec_step with the drafts placed as a token TREE
   (bmc_spec_write_tree's topology rules): for every layer
   bmc_append(K[l], V[l]) and bmc_spec_write_tree(Kd[l], Vd[l], k,
   parent_host), then the verify SDPA of all layers in one launch per 32
   layers (query row tau = 1 + i of node i sees the committed rows, its
   ancestors and itself).  parent_host[k]: one topology for every layer and
   batch row (host array).  Q, O DEVICE as bmc_spec_step (no all-host form).
   Returns k_adm (the admitted BFS prefix), errors and rollback as
   bmc_spec_step, plus ARG / UNSUPPORTED for an invalid topology or k > 32
   (checked before anything is enqueued).  Commit with bmc_commit_path_step. */
int bmc_spec_step_tree(const bmc_t* hs, int L, const void* const* K, const void* const* V,
                       const void* const* Kd, const void* const* Vd, int k,
                       const int* parent_host, const void* const* Q, float* const* O);

/* Bulk (prompt) append: n rows per unit, K and V [B][H_kv][n][D] in the
   cache dtype (device or host pointers).  Contents and lengths equal n
   bmc_append calls (P:L609 in-place writes); the allocation follows prompt
   ingestion (reading R19): at most ONE reallocation, to the
   capacity n appends would end at (BMC: cap + r*ceil((valid+n-cap)/r) capped
   at N_max; ITERATIVE: valid + n; UPFRONT: none), copying the valid rows.
   The rows are copied by a kernel this call enqueues (not deferred to the
   next call), so K and V must stay valid until the stream passes it.
   Errors: ARG (n < 0, null pointers), STATE (drafts staged), CAPACITY
   (valid + n > N_max); n == 0 is a no-op. */
int bmc_append_n(bmc_t h, const void* K, const void* V, int n);

/* bmc_spec_write: place k chain-draft rows in the padded rows.
   K_draft, V_draft: [B][H_kv][k][D].  Admits k_adm = min(k, cap - max valid)
   drafts (BMC, UPFRONT: never grows) or min(k, N_max - max valid)
   (ITERATIVE: exact-size reallocation).  Writes rows valid_b .. valid_b+k_adm-1,
   staged = k_adm.  Returns k_adm >= 0, or < 0 on error (STATE if drafts
   are already staged). */
int bmc_spec_write(bmc_t h, const void* K_draft, const void* V_draft, int k);

/* bmc_spec_write_tree: place a token TREE of k candidate rows (P:L863-866,
   Sequoia-style).  Nodes in breadth-first order; parent_host[i] in [-1, i)
   (-1: child of the last committed token); one topology for every batch row.
   Admitted like chain drafts (k_adm = min(k, free rows), a BFS prefix keeps
   parents before children, never grows).  Node i sits in row valid_b + i;
   at bmc_sdpa its query row tau = 1 + i sees the committed rows, its
   ancestors and itself only.  k <= 32 (else UNSUPPORTED).  Returns k_adm. */
int bmc_spec_write_tree(bmc_t h, const void* K_draft, const void* V_draft, int k,
                        const int* parent_host);

/* bmc_sdpa: masked scaled-dot-product attention over ALL cap rows of the
   padded cache (mask P:L846-853).
   Q: [B][H_q][t][D] in the cache dtype, t = 1 + staged (implicit).  Query
   row tau of batch row b attends keys [0, valid_b + tau) (row 0 = last
   committed token, rows >= 1 = chain drafts); every other row of the buffer
   is masked (it is still read).  O: [B][H_q][t][D] float32 =
   softmax(q K^T / sqrt(D) + mask) V with fp32 accumulation.
   n_valid: the committed length (must equal every valid_b), or BMC_PER_ROW. */
int bmc_sdpa(bmc_t h, const void* Q, int n_valid, float* O);

/* bmc_commit: accept the first n_accepted staged drafts of every row,
   valid_b += n_accepted; rejected staged rows are zeroed again; staged = 0. */
int bmc_commit(bmc_t h, int n_accepted);

/* bmc_commit_rows: per-row acceptance, n_accepted_host[B] (host array). */
int bmc_commit_rows(bmc_t h, const int* n_accepted_host);

/* bmc_commit_step: bmc_commit_rows(hs[l], n_accepted_host) for the L layers
   of one speculative iteration (the counterpart of bmc_spec_step).
   Every layer must accept the same n_accepted_host[B] (layers share the token
   sequence).  Layers that share stream, capacity, lengths and staged count
   get ONE zero-fill launch (rejected drafts, reading R9) per 32 layers; others
   are committed one by one.  Errors: as bmc_commit_rows, checked on every
   layer before anything is enqueued. */
int bmc_commit_step(const bmc_t* hs, int L, const int* n_accepted_host);

/* bmc_commit_path: commit one accepted root-to-node path per batch row
   (P:L447): path_host[b * max_depth + i], i < m_host[b], node
   indices of increasing depth (path[0] a root, path[i] a child of
   path[i-1]; for chain drafts the path 0..n-1).  The accepted rows are
   moved to valid_b .. valid_b + m_b - 1, every other staged row is zeroed,
   valid_b += m_b.  Chain commits (bmc_commit*) of a staged tree are a STATE
   error unless they reject everything. */
int bmc_commit_path(bmc_t h, const int* path_host, const int* m_host, int max_depth);

/* bmc_commit_path_step: bmc_commit_path(hs[l], path_host, m_host, max_depth)
   for the L layers of one token-tree iteration (the counterpart of
   bmc_spec_step_tree; every layer accepts the same paths, they share the
   token sequence).  Layers that share stream, capacity, lengths and staged
   count get ONE compaction launch per 32 layers, others are committed one by
   one.  Errors: as bmc_commit_path, checked on every layer before anything
   is enqueued. */
int bmc_commit_path_step(const bmc_t* hs, int L, const int* path_host, const int* m_host,
                         int max_depth);

/* bmc_decode_step: one plain decode step of a whole model, i.e. for every
   layer l = 0..L-1: bmc_append(hs[l], K[l], V[l]) then
   bmc_sdpa(hs[l], Q[l], n_valid, O[l]) (n_valid = the committed length AFTER
   the append, or BMC_PER_ROW).  Arrays of L pointers.  Every layer is
   validated before anything is enqueued.  One call instead of 2L.
   OOM on a growth allocation: as bmc_spec_step (the chunks already
   launched have stepped, the other layers are rolled back).
   When every K, V, Q and O is a HOST pointer the step is pipelined: the
   inputs are staged on an internal copy stream (double-buffered, so the copy
   of step s+1 overlaps the kernels of step s) and the outputs are copied back
   on it; with pinned buffers everything is asynchronous -- read O after
   bmc_sync(hs[0]) and keep inputs unchanged until then. */
int bmc_decode_step(const bmc_t* hs, int L, const void* const* K, const void* const* V,
                    const void* const* Q, float* const* O, int n_valid);

/* bmc_destroy: synchronises the handle's stream, frees the cache memory. */
int bmc_destroy(bmc_t h);

/* Host-side shadow state and cost ledger; no device synchronisation. */
typedef struct {
  long long valid_min, valid_max, capacity, staged;
  long long alloc_events, copy_events;
  long long copied_bytes;          /* payload moved by reallocation copies, K+V */
  long long init_written_bytes;    /* bytes written into new buffers (copy + zero) */
  long long append_written_bytes;  /* rows written by append / spec_write, K+V */
  long long kv_bytes_read;         /* K+V bytes read by SDPA (all cap rows) */
  long long macs;                  /* 2*B*H_q*t*cap*D per SDPA call */
  long long sdpa_calls;
} bmc_stats_t;
int bmc_stats(bmc_t h, bmc_stats_t* out);

/* Current cache buffers (device pointers, [B*H_kv][cap][D]) and capacity.
   Invalidated by the next growth. */
int bmc_kv_view(bmc_t h, void** K, void** V, int* cap);

/* Copy the whole cache [B*H_kv][cap][D] (cache dtype) into K_dst / V_dst
   (device or host buffers of bmc_stats().capacity rows); waits for the copy
   when a destination is host memory.  Inspection only (bit-exact checks). */
int bmc_read_cache(bmc_t h, void* K_dst, void* V_dst);

/* Committed length of every batch row, valid_host[B]. */
int bmc_valid(bmc_t h, int* valid_host);

/* Wait for all work enqueued on the handle's stream. */
int bmc_sync(bmc_t h);

/* Tuning / test options (key, value).  Keys:
     1 BMC_OPT_ATTN_CTAS      CTAs of the attention kernel (0 = auto)
     2 BMC_OPT_ATTN_PATH      0 auto, 1 CUDA-core split-K, 2 tcgen05 (keys on
                              the TMEM lanes for G*t <= 80, else queries on
                              the lanes), 3 tcgen05 with queries on the lanes,
                              4 tcgen05 with keys on the lanes (G*t <= 80)
     3 BMC_OPT_ARENA          0 VMM ping-pong slots, 1 stream-ordered pool,
                              2 the device's two-ended growth region
                              (bmc_region_reserve; the pool when the region is
                              absent or full).  Default: 2 when the device has
                              a region at bmc_create (the first buffer comes
                              from it too), else 1.  Takes effect at the next
                              growth
     4 BMC_OPT_SKIP_PADDING   1 = length-aware ABLATION: SDPA streams only the
                              rows some query sees instead of all cap rows
                              (not the method: P:L441, L853; results are
                              identical, bytes differ)
     5 BMC_OPT_COPY_ON_READ   1 (default) = a BMC growth inside bmc_decode_step
                              / bmc_spec_step, or between bmc_append and
                              bmc_sdpa, is copied by the attention kernel
                              while it streams the old buffer (SURVEY
                              NEXT-1: old rows read once, new buffer written
                              once, no separate realloc kernel; the
                              queries-on-lanes kernel, G*t > 80, still takes
                              the realloc kernel); 0 = separate
                              realloc_copy_zero launch.
                              Cache contents and ledger are identical.
     6 BMC_OPT_TCK_GROUPS     softmax column groups of the keys-on-lanes
                              tcgen05 kernel: 0 auto (4 for 16 < G*t <= 64,
                              else 2), 2 (384 threads), 4 (640 threads).  Tuning /
                              A/B only; results agree within the tolerance.
     8 BMC_OPT_TCK_PREFETCH   L2 prefetch distance of the keys-on-lanes kernel's
                              K / V producers, in 128-key tiles ahead of the
                              shared-memory ring (-1 auto = 0, off: measured
                              5-7% slower).  Tuning / A/B only; results are
                              identical.
     7 BMC_OPT_FAULT_OOM      fault injection for tests: the next `value`
                              growth allocations of this handle fail with
                              BMC_ERR_OOM (exercises the fused steps' OOM
                              fallback and rollback). */
#define BMC_OPT_ATTN_CTAS 1
#define BMC_OPT_ATTN_PATH 2
#define BMC_OPT_ARENA 3
#define BMC_OPT_SKIP_PADDING 4
#define BMC_OPT_COPY_ON_READ 5
#define BMC_OPT_TCK_GROUPS 6
#define BMC_OPT_FAULT_OOM 7
#define BMC_OPT_TCK_PREFETCH 8
int bmc_set_option(bmc_t h, int key, long long value);

/* bmc_pool_reserve: map `bytes` of device memory into the library's
   stream-ordered pool on `device` (-1 = current) now: one allocation and
   free (synchronous), kept by the pool (release threshold = max).  Growth
   allocations of every handle are then carved from it instead
   of waiting for the driver to grow the pool, which on B200 blocks the host
   for up to 0.6 s per growth step (profiles/r01_growth_cost_7b.txt).  Cache
   capacities and the ledger are unchanged; the memory is held by the
   process like a serving deployment's KV budget.  Errors: ARG (bytes < 0),
   OOM, CUDA. */
int bmc_pool_reserve(int device, long long bytes);

/* bmc_region_reserve: (re)create the two-ended growth region of `bytes` on
   `device` (-1 = current; 0 bytes frees it) for handles with BMC_OPT_ARENA =
   2.  All layers of a model grow in the same step,
   so a growth places each new buffer at the end of the region opposite to
   the buffer it replaces and pops the released old buffers off the other
   end: no fragmentation, no driver call and no host wait per growth (the
   stream-ordered pool stalled the host for up to ~1 s per growth step on the
   L3-8B workload, profiles/r02_growth_cost_l3.txt).  bmc_decode_step and
   bmc_spec_step move the layers chunk by chunk in LIFO order, so a copy
   growth's peak is the cache plus one 32-layer chunk of new buffers; size
   the region for that (per-layer calls: the cache plus the new buffers of
   the layers that grow before the first old buffer is released).  Space released on one stream is handed to
   another only after that stream passed the release (events).  Errors: ARG
   (bytes < 0), STATE (buffers of the current region are still live), OOM,
   CUDA. */
int bmc_region_reserve(int device, long long bytes);

/* bmc_pool_trim: wait for the device, then return the growth pool's unused
   memory (blocks no live buffer uses, e.g. a previous workload's or a
   reserve's) to the driver (-1 = current device).  Between workloads only.
   Errors: CUDA. */
int bmc_pool_trim(int device);

/* Kernels launched by this library in this process so far (all handles). */
unsigned long long bmc_launch_count(void);

/* Host-time diagnostics of the growth path, per category: 0 growth
   allocations (arena_alloc), 1 stream-ordered releases, 2 attention-launch
   calls of the fused steps, 3 helper-thread VMM pre-mapping, 4 VMM mappings
   done synchronously at a growth (the pre-map was late).  ns[5] and calls[5]
   (host arrays) receive nanoseconds and call counts since the last reset;
   reset != 0 zeroes them.  Errors: ARG (null arrays). */
int bmc_host_profile(long long* ns, long long* calls, int reset);

/* Thread-local message for the last error (empty string if none). */
const char* bmc_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
