/*
 * oracle.c -- plain, slow, fp64 CPU reference for the BMC decode hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Nothing here is used by the
 * product path; the product never links this file.
 *
 * Paper: arXiv 2511.12031, "BMC: Balancing Memory and Compute".  Citations
 * P:L<n> are PAPER.md line numbers.  Readings R<n> refer to DESIGN.md
 * section "Readings of the paper".
 *
 * Storage: one context = one layer's K and V cache, each laid out
 * [B*H_kv][cap][D] row-major with raw input element bits (4 B fp32 or
 * 2 B bf16).  Arithmetic is fp64, sums are sequential in index order.
 *
 * The three allocation policies are three separate functions
 * (append_iterative / append_upfront / append_bmc, and likewise for the
 * speculative write) so that the degeneracy checks BMC(r=1) == ITERATIVE
 * and BMC(r=N) == UPFRONT compare independent code.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_ERR_ARG (-1)
#define OR_ERR_STATE (-2)
#define OR_ERR_CAPACITY (-3)
#define OR_ERR_OOM (-4)
#define OR_ERR_UNSUPPORTED (-6)

/* Padded-row bias: "smallest representable value ...
   (approx -10^9)".  Applied in fp64 score space (reading R3). */
#define MASK_BIAS (-1.0e9)

struct oracle_ctx {
  int B, H_kv, H_q, D, r, N_max, dtype, policy;
  int eb;          /* bytes per element */
  long cap;        /* rows allocated per (b, h_kv) unit */
  int* valid;      /* [B] committed rows per batch row */
  int staged;      /* speculative rows written but not committed */
  int tree;        /* staged rows form a token tree (else a chain) */
  int parent[64];  /* tree topology of the staged nodes */
  unsigned char* K;
  unsigned char* V;
  oracle_stats_t st;
};

/* ---------------------------------------------------------------- helpers */

static long units(const struct oracle_ctx* h) { return (long)h->B * h->H_kv; }

static int max_valid(const struct oracle_ctx* h) {
  int m = 0;
  for (int b = 0; b < h->B; ++b)
    if (h->valid[b] > m) m = h->valid[b];
  return m;
}

static int min_valid(const struct oracle_ctx* h) {
  int m = h->valid[0];
  for (int b = 1; b < h->B; ++b)
    if (h->valid[b] < m) m = h->valid[b];
  return m;
}

/* Exact widening of one stored element to fp64. */
static double elem(const struct oracle_ctx* h, const unsigned char* p) {
  if (h->dtype == ORACLE_F32) {
    float f;
    memcpy(&f, p, 4);
    return (double)f;
  }
  /* bf16: the upper 16 bits of an IEEE binary32. */
  unsigned short b;
  memcpy(&b, p, 2);
  unsigned int u = ((unsigned int)b) << 16;
  float f;
  memcpy(&f, &u, 4);
  return (double)f;
}

static unsigned char* row_ptr(const struct oracle_ctx* h, unsigned char* base, long u,
                              long row) {
  return base + ((u * h->cap + row) * h->D) * (long)h->eb;
}

/* Replace the cache buffers by new zeroed [U][new_cap][D] buffers holding the
   first copy_rows rows of every unit ("allocate" + "concat";
   P:L676-678 "new tensors ... are allocated ... and the KV cache copy
   operation takes place"). */
static int reallocate(struct oracle_ctx* h, long new_cap, long copy_rows) {
  long U = units(h);
  size_t row_bytes = (size_t)h->D * h->eb;
  unsigned char* nk = (unsigned char*)calloc((size_t)(U * new_cap) + 1, row_bytes);
  unsigned char* nv = (unsigned char*)calloc((size_t)(U * new_cap) + 1, row_bytes);
  if (!nk || !nv) {
    free(nk);
    free(nv);
    return OR_ERR_OOM;
  }
  for (long u = 0; u < U; ++u) {
    for (long j = 0; j < copy_rows; ++j) {
      memcpy(nk + (u * new_cap + j) * row_bytes, row_ptr(h, h->K, u, j), row_bytes);
      memcpy(nv + (u * new_cap + j) * row_bytes, row_ptr(h, h->V, u, j), row_bytes);
    }
  }
  if (h->cap > 0) h->st.copy_events += 1;
  h->st.alloc_events += 1;
  h->st.copied_bytes += 2LL * U * copy_rows * (long long)row_bytes;
  h->st.init_written_bytes += 2LL * U * new_cap * (long long)row_bytes;
  free(h->K);
  free(h->V);
  h->K = nk;
  h->V = nv;
  h->cap = new_cap;
  return OR_OK;
}

/* Write one new row per unit at row valid[b] (+offset), from src laid out
   [B][H_kv][nrows][D] (row index i). */
static void write_row(struct oracle_ctx* h, const unsigned char* srcK,
                      const unsigned char* srcV, int nrows, int i, int offset) {
  size_t row_bytes = (size_t)h->D * h->eb;
  for (int b = 0; b < h->B; ++b) {
    for (int g = 0; g < h->H_kv; ++g) {
      long u = (long)b * h->H_kv + g;
      size_t src_off = (((size_t)u * nrows) + i) * row_bytes;
      long dst_row = (long)h->valid[b] + offset;
      memcpy(row_ptr(h, h->K, u, dst_row), srcK + src_off, row_bytes);
      memcpy(row_ptr(h, h->V, u, dst_row), srcV + src_off, row_bytes);
    }
  }
  h->st.append_written_bytes += 2LL * units(h) * (long long)row_bytes;
}

/* ------------------------------------------------------------------ create */

int oracle_create(int B, int H_kv, int H_q, int D, int r, int N_max, int dtype,
                  int policy, oracle_t* out) {
  if (!out) return OR_ERR_ARG;
  *out = NULL;
  if (B < 1 || H_kv < 1 || H_q < 1 || D < 1 || N_max < 1) return OR_ERR_ARG;
  if (H_q % H_kv != 0) return OR_ERR_ARG;
  if (dtype != ORACLE_F32 && dtype != ORACLE_BF16) return OR_ERR_UNSUPPORTED;
  if (policy == ORACLE_POLICY_BMC && (r < 1 || r > N_max)) return OR_ERR_ARG;
  if (policy < 0 || policy > 2) return OR_ERR_ARG;

  struct oracle_ctx* h = (struct oracle_ctx*)calloc(1, sizeof(*h));
  if (!h) return OR_ERR_OOM;
  h->B = B; h->H_kv = H_kv; h->H_q = H_q; h->D = D; h->r = r; h->N_max = N_max;
  h->dtype = dtype; h->policy = policy;
  h->eb = dtype == ORACLE_F32 ? 4 : 2;
  h->valid = (int*)calloc((size_t)B, sizeof(int));
  if (!h->valid) { free(h); return OR_ERR_OOM; }

  int rc = OR_OK;
  if (policy == ORACLE_POLICY_BMC) {
    /* first chunk of r rows (reading R1: cap = min(r, N_max)) */
    rc = reallocate(h, r < N_max ? r : N_max, 0);
  } else if (policy == ORACLE_POLICY_UPFRONT) {
    /* one allocation for the maximum context */
    rc = reallocate(h, N_max, 0);
  } /* ITERATIVE: nothing allocated until the first token */
  if (rc != OR_OK) { oracle_destroy(h); return rc; }
  *out = h;
  return OR_OK;
}

/* ------------------------------------------------------------------ append */

/* ITERATIVE (Fig. AttnBlkListing): allocate exactly the rows now
   needed, copy the valid rows, write the new one.  Reading R17: one
   reallocation per append and one per speculative write. */
static int append_iterative(struct oracle_ctx* h, const unsigned char* K,
                            const unsigned char* V) {
  int mv = max_valid(h);
  int rc = reallocate(h, (long)mv + 1, mv);
  if (rc) return rc;
  write_row(h, K, V, 1, 0, 0);
  for (int b = 0; b < h->B; ++b) h->valid[b] += 1;
  return OR_OK;
}

/* UPFRONT: "written in place in this larger KV cache". */
static int append_upfront(struct oracle_ctx* h, const unsigned char* K,
                          const unsigned char* V) {
  write_row(h, K, V, 1, 0, 0);
  for (int b = 0; b < h->B; ++b) h->valid[b] += 1;
  return OR_OK;
}

/* BMC: when the buffer is full, allocate r more
   rows (ragged last chunk capped at N_max, reading R12) and copy the old
   buffer; otherwise write in place. */
static int append_bmc(struct oracle_ctx* h, const unsigned char* K,
                      const unsigned char* V) {
  if (max_valid(h) == h->cap) {
    long nc = h->cap + h->r;
    if (nc > h->N_max) nc = h->N_max;
    int rc = reallocate(h, nc, h->cap);
    if (rc) return rc;
  }
  write_row(h, K, V, 1, 0, 0);
  for (int b = 0; b < h->B; ++b) h->valid[b] += 1;
  return OR_OK;
}

int oracle_append(oracle_t h, const void* K, const void* V) {
  if (!h || !K || !V) return OR_ERR_ARG;
  if (h->staged > 0) return OR_ERR_STATE;
  if (max_valid(h) >= h->N_max) return OR_ERR_CAPACITY;
  const unsigned char* k = (const unsigned char*)K;
  const unsigned char* v = (const unsigned char*)V;
  switch (h->policy) {
    case ORACLE_POLICY_ITERATIVE: return append_iterative(h, k, v);
    case ORACLE_POLICY_UPFRONT: return append_upfront(h, k, v);
    default: return append_bmc(h, k, v);
  }
}

/* ------------------------------------------------------------ bulk append */

/* Bulk (prompt) append of n rows per unit, K/V laid out [B][H_kv][n][D].
   Contents and valid lengths equal n single appends; the allocation ledger
   follows the prompt-ingestion rule ("one chunk covering the whole
   prompt (single alloc event), not token-by-token"; reading R19): at most
   one reallocation, to the capacity n single appends would end at --
   BMC: cap + r*ceil((mv + n - cap)/r) capped at N_max;
   ITERATIVE: exactly mv + n; UPFRONT: none --
   copying the mv rows that can hold data. */
int oracle_append_n(oracle_t h, const void* K, const void* V, int n) {
  if (!h || n < 0) return OR_ERR_ARG;
  if (n == 0) return OR_OK;
  if (!K || !V) return OR_ERR_ARG;
  if (h->staged > 0) return OR_ERR_STATE;
  int mv = max_valid(h);
  if ((long)mv + n > h->N_max) return OR_ERR_CAPACITY;
  long need = (long)mv + n;
  int rc = OR_OK;
  if (h->policy == ORACLE_POLICY_ITERATIVE) {
    rc = reallocate(h, need, mv);
  } else if (h->policy == ORACLE_POLICY_BMC && need > h->cap) {
    long chunks = (need - h->cap + h->r - 1) / h->r;
    long nc = h->cap + chunks * h->r;
    if (nc > h->N_max) nc = h->N_max;
    rc = reallocate(h, nc, mv);
  }
  if (rc) return rc;
  for (int i = 0; i < n; ++i) write_row(h, (const unsigned char*)K, (const unsigned char*)V, n, i, i);
  for (int b = 0; b < h->B; ++b) h->valid[b] += n;
  return OR_OK;
}

/* ------------------------------------------------------------- spec_write */

/* BMC / UPFRONT admission: "limit the number of speculated
   tokens (to the available rows)"; never reallocates. */
static int spec_write_in_place(struct oracle_ctx* h, const unsigned char* Kd,
                               const unsigned char* Vd, int k) {
  long free_rows = h->cap - max_valid(h);
  int k_adm = (long)k < free_rows ? k : (int)free_rows;
  for (int i = 0; i < k_adm; ++i) write_row(h, Kd, Vd, k, i, i);
  h->staged = k_adm;
  return k_adm;
}

/* ITERATIVE: the drafts are concatenated like any new rows,
   limited only by N_max (reading R17). */
static int spec_write_iterative(struct oracle_ctx* h, const unsigned char* Kd,
                                const unsigned char* Vd, int k) {
  int mv = max_valid(h);
  int k_adm = k < h->N_max - mv ? k : h->N_max - mv;
  if (k_adm > 0) {
    int rc = reallocate(h, (long)mv + k_adm, mv);
    if (rc) return rc;
  }
  for (int i = 0; i < k_adm; ++i) write_row(h, Kd, Vd, k, i, i);
  h->staged = k_adm;
  return k_adm;
}

int oracle_spec_write(oracle_t h, const void* Kd, const void* Vd, int k) {
  if (!h || k < 0) return OR_ERR_ARG;
  if (k > 0 && (!Kd || !Vd)) return OR_ERR_ARG;
  if (h->staged > 0) return OR_ERR_STATE;
  if (k == 0) return 0;
  const unsigned char* kd = (const unsigned char*)Kd;
  const unsigned char* vd = (const unsigned char*)Vd;
  if (h->policy == ORACLE_POLICY_ITERATIVE) return spec_write_iterative(h, kd, vd, k);
  return spec_write_in_place(h, kd, vd, k);
}

/* -------------------------------------------------------------------- sdpa */

/* Is key row j visible to query row tau of batch row b?  Chain drafts
   (reading R7): rows [0, valid_b + tau).  Token tree: the
   committed rows, plus node (tau-1) and its ancestors. */
static int visible(const struct oracle_ctx* h, int b, int tau, long j) {
  const long vb = h->valid[b];
  if (!h->tree) return j < vb + tau;
  if (j < vb) return 1;
  if (tau == 0) return 0;
  for (int x = tau - 1; x >= 0; x = h->parent[x])
    if (j - vb == x) return 1;
  return 0;
}

/* Masked SDPA over all cap rows of one unit for one query row
   (mask P:L853):
     s_j = (q . k_j) / sqrt(D) + bias_j,  bias_j = 0 (visible) else -1e9
     p_j = exp(s_j - max_j s_j),  o = (sum_j p_j v_j) / (sum_j p_j).        */
static void sdpa_row(const struct oracle_ctx* h, long u, const double* q, int b, int tau,
                     double* s, double* o) {
  const double scale = 1.0 / sqrt((double)h->D);   /* reading R4: d = head_dim */
  long cap = h->cap;
  for (long j = 0; j < cap; ++j) {
    const unsigned char* kr = row_ptr(h, h->K, u, j);
    double dot = 0.0;
    for (int x = 0; x < h->D; ++x) dot += q[x] * elem(h, kr + (size_t)x * h->eb);
    s[j] = dot * scale + (visible(h, b, tau, j) ? 0.0 : MASK_BIAS);
  }
  double mu = s[0];
  for (long j = 1; j < cap; ++j)
    if (s[j] > mu) mu = s[j];
  double l = 0.0;
  for (long j = 0; j < cap; ++j) {
    s[j] = exp(s[j] - mu);
    l += s[j];
  }
  for (int x = 0; x < h->D; ++x) o[x] = 0.0;
  for (long j = 0; j < cap; ++j) {
    const unsigned char* vr = row_ptr(h, h->V, u, j);
    for (int x = 0; x < h->D; ++x) o[x] += s[j] * elem(h, vr + (size_t)x * h->eb);
  }
  for (int x = 0; x < h->D; ++x) o[x] = o[x] / l;
}

int oracle_sdpa(oracle_t h, const void* Q, int n_valid, double* O) {
  if (!h || !Q || !O) return OR_ERR_ARG;
  if (n_valid == 0) return OR_ERR_ARG;                    /* reading R13 */
  if (n_valid != -1) {
    for (int b = 0; b < h->B; ++b)
      if (h->valid[b] != n_valid) return OR_ERR_STATE;
  }
  for (int b = 0; b < h->B; ++b)
    if (h->valid[b] == 0) return OR_ERR_ARG;
  const int t = 1 + h->staged;                            /* reading R7 */
  const int G = h->H_q / h->H_kv;                         /* reading R6 */
  const int D = h->D;
  const unsigned char* q_raw = (const unsigned char*)Q;
  int nthreads_err = 0;

#pragma omp parallel for collapse(2) schedule(dynamic)
  for (int b = 0; b < h->B; ++b) {
    for (int hq = 0; hq < h->H_q; ++hq) {
      double* s = (double*)malloc((size_t)(h->cap > 0 ? h->cap : 1) * sizeof(double));
      double* q = (double*)malloc((size_t)D * sizeof(double));
      if (!s || !q) {
        free(s); free(q);
#pragma omp atomic write
        nthreads_err = 1;
        continue;
      }
      long u = (long)b * h->H_kv + hq / G;                /* KV head floor(h/G) */
      for (int tau = 0; tau < t; ++tau) {
        size_t qi = (((size_t)b * h->H_q + hq) * t + tau) * D;
        for (int x = 0; x < D; ++x) q[x] = elem(h, q_raw + (qi + x) * h->eb);
        sdpa_row(h, u, q, b, tau, s, O + qi);
      }
      free(s);
      free(q);
    }
  }
  if (nthreads_err) return OR_ERR_OOM;
  h->st.sdpa_calls += 1;
  h->st.kv_bytes_read += 2LL * units(h) * h->cap * (long long)D * h->eb;
  h->st.macs += 2LL * h->B * h->H_q * t * h->cap * (long long)D;
  return OR_OK;
}

/* ------------------------------------------------------------------ commit */

/* "only the m accepted entries are used to update the KV cache".
   Chain drafts: the accepted ones are already a prefix of the staged rows.
   Rejected rows are re-zeroed (reading R9). */
static void commit_row(struct oracle_ctx* h, int b, int m) {
  size_t row_bytes = (size_t)h->D * h->eb;
  for (int g = 0; g < h->H_kv; ++g) {
    long u = (long)b * h->H_kv + g;
    for (int i = m; i < h->staged; ++i) {
      long row = (long)h->valid[b] + i;
      memset(row_ptr(h, h->K, u, row), 0, row_bytes);
      memset(row_ptr(h, h->V, u, row), 0, row_bytes);
    }
  }
  h->valid[b] += m;
}

int oracle_commit(oracle_t h, int n_accepted) {
  if (!h) return OR_ERR_ARG;
  if (h->staged == 0 && n_accepted > 0) return OR_ERR_STATE;
  if (n_accepted < 0 || n_accepted > h->staged) return OR_ERR_ARG;
  if (h->tree && n_accepted > 0) return OR_ERR_STATE;   /* trees commit paths */
  for (int b = 0; b < h->B; ++b) commit_row(h, b, n_accepted);
  h->staged = 0;
  h->tree = 0;
  return OR_OK;
}

int oracle_commit_rows(oracle_t h, const int* n_accepted) {
  if (!h || !n_accepted) return OR_ERR_ARG;
  for (int b = 0; b < h->B; ++b) {
    if (h->staged == 0 && n_accepted[b] > 0) return OR_ERR_STATE;
    if (n_accepted[b] < 0 || n_accepted[b] > h->staged) return OR_ERR_ARG;
    if (h->tree && n_accepted[b] > 0) return OR_ERR_STATE;
  }
  for (int b = 0; b < h->B; ++b) commit_row(h, b, n_accepted[b]);
  h->staged = 0;
  h->tree = 0;
  return OR_OK;
}

/* ------------------------------------------------------------ token tree */

int oracle_spec_write_tree(oracle_t h, const void* Kd, const void* Vd, int k,
                           const int* parent) {
  if (!h || k < 0 || k > 64) return OR_ERR_ARG;
  if (k > 0 && (!Kd || !Vd || !parent)) return OR_ERR_ARG;
  if (h->staged > 0) return OR_ERR_STATE;
  for (int i = 0; i < k; ++i)
    if (parent[i] < -1 || parent[i] >= i) return OR_ERR_ARG;   /* BFS order */
  int k_adm = oracle_spec_write(h, Kd, Vd, k);                  /* same placement */
  if (k_adm < 0) return k_adm;
  for (int i = 0; i < k_adm; ++i) h->parent[i] = parent[i];
  h->tree = k_adm > 0;
  return k_adm;
}

int oracle_commit_path(oracle_t h, const int* path, const int* m, int max_depth) {
  if (!h || !m || max_depth < 0) return OR_ERR_ARG;
  for (int b = 0; b < h->B; ++b) {
    if (m[b] < 0 || m[b] > max_depth || m[b] > h->staged) return OR_ERR_ARG;
    if (m[b] > 0 && !path) return OR_ERR_ARG;
    for (int i = 0; i < m[b]; ++i) {
      const int x = path[b * max_depth + i];
      if (x < 0 || x >= h->staged) return OR_ERR_ARG;
      const int want = i == 0 ? -1 : path[b * max_depth + i - 1];
      const int par = h->tree ? h->parent[x] : x - 1;          /* a chain's parents */
      if (par != want) return OR_ERR_ARG;
    }
  }
  size_t row_bytes = (size_t)h->D * h->eb;
  for (int b = 0; b < h->B; ++b) {
    for (int g = 0; g < h->H_kv; ++g) {
      long u = (long)b * h->H_kv + g;
      /* ascending moves are safe: path[i] >= i, so a destination never holds
         a row that a later step still has to read */
      for (int i = 0; i < m[b]; ++i) {
        long src = (long)h->valid[b] + path[b * max_depth + i];
        long dst = (long)h->valid[b] + i;
        if (src != dst) {
          memmove(row_ptr(h, h->K, u, dst), row_ptr(h, h->K, u, src), row_bytes);
          memmove(row_ptr(h, h->V, u, dst), row_ptr(h, h->V, u, src), row_bytes);
        }
      }
      for (int i = m[b]; i < h->staged; ++i) {
        long row = (long)h->valid[b] + i;
        memset(row_ptr(h, h->K, u, row), 0, row_bytes);
        memset(row_ptr(h, h->V, u, row), 0, row_bytes);
      }
    }
    h->valid[b] += m[b];
  }
  h->staged = 0;
  h->tree = 0;
  return OR_OK;
}

/* -------------------------------------------------------------- inspection */

int oracle_stats(oracle_t h, oracle_stats_t* out) {
  if (!h || !out) return OR_ERR_ARG;
  *out = h->st;
  out->valid_min = min_valid(h);
  out->valid_max = max_valid(h);
  out->capacity = h->cap;
  out->staged = h->staged;
  return OR_OK;
}

int oracle_valid(oracle_t h, int* valid) {
  if (!h || !valid) return OR_ERR_ARG;
  memcpy(valid, h->valid, (size_t)h->B * sizeof(int));
  return OR_OK;
}

int oracle_read_cache(oracle_t h, void* K, void* V) {
  if (!h) return OR_ERR_ARG;
  size_t bytes = (size_t)units(h) * h->cap * h->D * h->eb;
  if (bytes == 0) return OR_OK;
  if (!K || !V) return OR_ERR_ARG;
  memcpy(K, h->K, bytes);
  memcpy(V, h->V, bytes);
  return OR_OK;
}

int oracle_destroy(oracle_t h) {
  if (!h) return OR_ERR_ARG;
  free(h->K);
  free(h->V);
  free(h->valid);
  free(h);
  return OR_OK;
}

/* ------------------------------------------------------- textbook SDPA */

int oracle_exact_sdpa(const double* q, const double* K, const double* V, int n, int D,
                      double* o) {
  if (!q || !K || !V || !o || n < 1 || D < 1) return OR_ERR_ARG;
  double* s = (double*)malloc((size_t)n * sizeof(double));
  if (!s) return OR_ERR_OOM;
  const double scale = 1.0 / sqrt((double)D);
  for (int j = 0; j < n; ++j) {
    double dot = 0.0;
    for (int x = 0; x < D; ++x) dot += q[x] * K[(size_t)j * D + x];
    s[j] = dot * scale;
  }
  double mu = s[0];
  for (int j = 1; j < n; ++j)
    if (s[j] > mu) mu = s[j];
  double l = 0.0;
  for (int j = 0; j < n; ++j) {
    s[j] = exp(s[j] - mu);
    l += s[j];
  }
  for (int x = 0; x < D; ++x) o[x] = 0.0;
  for (int j = 0; j < n; ++j)
    for (int x = 0; x < D; ++x) o[x] += s[j] * V[(size_t)j * D + x];
  for (int x = 0; x < D; ++x) o[x] = o[x] / l;
  free(s);
  return OR_OK;
}
