/*
 * oracle.h -- CPU reference ("oracle") for the BMC decode hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (libbmc.so, paper_2511_12031_b200/) never includes,
 * links or calls anything under oracle/.  It shares no code, header, table
 * or helper with the CUDA path.
 *
 * What it computes (arXiv 2511.12031, PAPER.md = P:L<line>):
 *   - KV cache update under three allocation policies, each its own code path:
 *       ITERATIVE (Fig. AttnBlkListing): exact-size reallocation
 *         and copy on every append / speculative write;
 *       UPFRONT: one N_max allocation, in-place writes;
 *       BMC: allocate r more rows when full,
 *         copy the old rows, in-place writes in between.
 *   - SDPA over the padded cache with the additive -1e9 bias mask,
 *     softmax((Q K^T)/sqrt(d) + bias) V (MHA reshape P:L413-416),
 *     GQA head sharing, chain-speculative query rows.
 *   - speculative draft admission / commit / rollback.
 * All arithmetic is fp64 with sequential sums; element storage keeps the raw
 * input bits (fp32 or bf16) so cache contents are bit-comparable.
 * Readings of ambiguous passages are listed in DESIGN.md ("Readings").
 *
 * Status codes: 0 ok, -1 ARG, -2 STATE, -3 CAPACITY, -4 OOM, -6 UNSUPPORTED.
 */
#ifndef BMC_ORACLE_H
#define BMC_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct oracle_ctx* oracle_t;

enum { ORACLE_F32 = 0, ORACLE_BF16 = 1 };
enum { ORACLE_POLICY_BMC = 0, ORACLE_POLICY_ITERATIVE = 1, ORACLE_POLICY_UPFRONT = 2 };

typedef struct {
  long long valid_min, valid_max, capacity, staged;
  long long alloc_events, copy_events;
  long long copied_bytes;          /* payload rows moved by reallocations, K+V */
  long long init_written_bytes;    /* bytes written to initialise new buffers (copy + zero) */
  long long append_written_bytes;  /* rows written by append / spec_write, K+V */
  long long kv_bytes_read;         /* K+V bytes the SDPA reads (all cap rows) */
  long long macs;                  /* 2*B*H_q*t*cap*D per SDPA call */
  long long sdpa_calls;
} oracle_stats_t;

int oracle_create(int B, int H_kv, int H_q, int D, int r, int N_max, int dtype,
                  int policy, oracle_t* out);
int oracle_append(oracle_t h, const void* K, const void* V);          /* [B][H_kv][D] */
int oracle_append_n(oracle_t h, const void* K, const void* V, int n);   /* [B][H_kv][n][D] bulk (prompt) append */
int oracle_spec_write(oracle_t h, const void* Kd, const void* Vd, int k); /* [B][H_kv][k][D]; returns k_adm */
int oracle_sdpa(oracle_t h, const void* Q, int n_valid, double* O);   /* Q [B][H_q][t][D], O fp64 */
int oracle_commit(oracle_t h, int n_accepted);
int oracle_commit_rows(oracle_t h, const int* n_accepted);            /* [B] */

/* Token-tree speculation (Sequoia-style candidate tree).
   k nodes in breadth-first order, parent[i] in [-1, i) (-1: child of the last
   committed token), one topology for all batch rows.  Admission as for chain
   drafts (k_adm = min(k, free rows); a BFS prefix keeps every
   parent before its children).  Node i sits in row valid_b + i; query row
   tau = 1 + i sees the committed rows [0, valid_b) and the rows of node i's
   ancestors and of node i itself, nothing else (ancestor rule).
   Returns k_adm. */
int oracle_spec_write_tree(oracle_t h, const void* Kd, const void* Vd, int k,
                           const int* parent);
/* Commit an accepted root-to-node path per row:
   path[b*max_depth + i], i < m[b], node indices of increasing depth (path[0]
   a root, path[i] a child of path[i-1]).  The accepted rows are moved to
   valid_b .. valid_b + m_b - 1, all other staged rows are zeroed, valid_b +=
   m_b.  A chain commit of n (oracle_commit) is the path 0..n-1. */
int oracle_commit_path(oracle_t h, const int* path, const int* m, int max_depth);
int oracle_stats(oracle_t h, oracle_stats_t* out);
int oracle_valid(oracle_t h, int* valid);                              /* [B] */
int oracle_read_cache(oracle_t h, void* K, void* V);                   /* raw [B*H_kv][cap][D] */
int oracle_destroy(oracle_t h);

/* Textbook SDPA over exactly n rows (no padding, no mask), P:L274-276:
   o = softmax(q K^T / sqrt(D)) V, fp64 inputs.  Used by the mask pins. */
int oracle_exact_sdpa(const double* q, const double* K, const double* V, int n, int D,
                      double* o);

#ifdef __cplusplus
}
#endif
#endif
