"""Analytical model of BMC and the choice of r (host-side only).

Paper model (arXiv 2511.12031, Sec. 5.1), per-iteration
costs with C1 = B*L*D, copy efficiency alpha*BW and compute rate beta*C:
  copy time of chunk i   4*B*L*((i+1)*r)*D / (alpha*BW)          (eq;KVCacheUpdate)
  SDPA time per iter     2*B*L*((i+1)*r)*D / (beta*C)             (eq:SPDA)
  time for N iterations  2*C1*N*T/(aBW) + 2*C1*N/(aBW) + T*C0
                         + C1*N^2/(bC) + C1*N^2/(bC*T)            (eq:NiterFinal)
  optimum (C0 ignored)   T = sqrt(N * aBW / (2*bC))                (Opt-T-eq)
  rounded to the nearest power of 2
  with speculation (k drafts verified, m accepted on average)
                         ... + C1*k*(N^2/m)*(1 + 1/T)/(b'C)        (TimeNIter)
                         T = sqrt(k*N*aBW / (2*m*b'C))  (T ~ sqrt(N/m))

B200 form.  On B200 both the growth copy and the SDPA are HBM-bound, so the
natural cost unit is bytes: per layer, with row = 2*U*D*eb bytes (K+V of one
token for all U = B*H_kv units),
  SDPA reads   sum_n cap(n) * row      = row * N*(N + r)/2          (r | N)
  growth copy  sum_i (i*r + (i+1)*r) * row = row * r*T^2 = row * N^2/r
so  t(r) = row*N*(N + r)/(2*BW_read) + row*N^2/(r*BW_copy), minimised at
  r* = sqrt(2*N*BW_read/BW_copy)   (= sqrt(2N) at equal bandwidths),
i.e. T* = N/r* -- the paper's T = sqrt(N*aBW/(2bC)) with the compute rate of
the padded GEMV replaced by its read bandwidth.
"""
from __future__ import annotations

import math


def round_pow2(x: float) -> int:
    """Nearest power of two ('round it to the nearest power of 2');
    ties go to the larger power."""
    if x <= 1:
        return 1
    lo = 2 ** math.floor(math.log2(x))
    hi = lo * 2
    return lo if (x - lo) < (hi - x) else hi


# ------------------------------------------------------------- paper model

def chunk_copy_time(i: int, r: int, C1: float, alpha_bw: float, elem_bytes: int = 2,
                    G: float = 1.0, Q: float = 1.0) -> float:
    """eq;KVCacheUpdate, generalised to elem_bytes (the '4' is
    2 tensors x 2 bytes) and the GQA/quantisation divisor of
    eq:KVCacheUpdate_GQA."""
    return 2 * elem_bytes * C1 * ((i + 1) * r) / (alpha_bw * G * Q)


def sdpa_time(i: int, r: int, C1: float, beta_c: float) -> float:
    """eq:SPDA: one iteration of the i-th chunk."""
    return 2 * C1 * ((i + 1) * r) / beta_c


def time_r_iters(i: int, r: int, C1, alpha_bw, beta_c, c0=0.0) -> float:
    """eq:rIterTime, with the paper's 4-byte copy constant."""
    return chunk_copy_time(i, r, C1, alpha_bw) + c0 + r * sdpa_time(i, r, C1, beta_c)


def total_time_sum(T: int, N: int, C1, alpha_bw, beta_c, c0=0.0) -> float:
    """eq:NIterTime: the sum over the T chunks (r = N/T)."""
    r = N // T
    return sum(time_r_iters(i, r, C1, alpha_bw, beta_c, c0) for i in range(T))


def total_time(T: float, N: int, C1, alpha_bw, beta_c, c0=0.0) -> float:
    """eq:NiterFinal, closed form."""
    return (2 * C1 * N * T / alpha_bw + 2 * C1 * N / alpha_bw + T * c0
            + C1 * N * N / beta_c + C1 * N * N / (beta_c * T))


def optimal_T(N: int, alpha_bw: float, beta_c: float, C1: float = 1.0, c0: float = 0.0) -> float:
    """Opt-T-eq solved for T; with c0 = 0 this is
    T = sqrt(N * aBW / (2 bC))."""
    return math.sqrt(C1 * N * N / (beta_c * (2 * C1 * N / alpha_bw + c0)))


def optimal_T_cprime(N: int, cprime: float) -> float:
    """The validation form T = sqrt(C' * N) (C' = 0.1)."""
    return math.sqrt(cprime * N)


def total_time_sd(T: float, N: int, C1, alpha_bw, beta_prime_c, k: int, m: float,
                  c0=0.0) -> float:
    """TimeNIter."""
    return (2 * C1 * N * (T + 1) / alpha_bw + T * c0
            + C1 * k * (N * N / m) * (1 + 1 / T) / beta_prime_c)


def optimal_T_sd(N: int, alpha_bw, beta_prime_c, k: int, m: float) -> float:
    """Minimiser of TimeNIter with c0 = 0: T = sqrt(k N aBW / (2 m b'C))."""
    return math.sqrt(k * N * alpha_bw / (2 * m * beta_prime_c))


# ------------------------------------------------------------- B200 form

def bytes_per_layer(N: int, r: int, U: int, D: int, eb: int) -> dict:
    """Exact per-layer bytes of one decode 0 -> N (ragged last chunk allowed):
    SDPA reads all cap rows each step; each growth reads cap_old and writes
    cap_new rows."""
    row = 2 * U * D * eb
    sdpa = sum(min(r * -(-n // r), N) for n in range(1, N + 1)) * row
    copy, cap = 0, min(r, N)
    while cap < N:
        new = min(cap + r, N)
        copy += (cap + new) * row
        cap = new
    return {"sdpa": sdpa, "copy": copy}


def advise_r(N: int, bw_read: float = 1.0, bw_copy: float = 1.0, pow2: bool = True,
             copy_on_read: bool = False, tokens_per_iter: float = 1.0) -> int:
    """r* = sqrt(f N m BW_read / BW_copy), T* = N / r* rounded to a power of
    two as the paper does for T, r = N / T.
    f = 2 with a separate realloc copy (each growth reads cap_old and writes
    cap_new rows: ~N^2/r rows per decode); f = 1 with copy-on-read growth
    (the attention already streams the old rows, the growth adds the write of
    the new buffer: ~N^2/(2r) rows; BW_copy is then that write bandwidth).
    m = tokens per iteration under speculation: the verify reads cap rows
    once per iteration, N/m times per decode, while the T growths stay, so
    r* grows as sqrt(m) and T* ~ sqrt(N/m) (TimeNIter)."""
    f = 1.0 if copy_on_read else 2.0
    r = math.sqrt(f * N * tokens_per_iter * bw_read / bw_copy)
    if not pow2:
        return max(1, min(N, round(r)))
    T = round_pow2(N / r)
    return max(1, min(N, N // T))


def model_time_b200(N: int, r: int, U: int, D: int, eb: int, L: int, bw_read: float,
                    bw_copy: float) -> float:
    """Seconds of one full decode predicted by the byte model."""
    b = bytes_per_layer(N, r, U, D, eb)
    return L * (b["sdpa"] / bw_read + b["copy"] / bw_copy)
