"""Pins of the analytical model / r advisor against the paper."""
import math
import random

import pytest

from paper_2511_12031_b200 import advisor as A


def test_closed_form_equals_chunk_sum():
    """eq:NiterFinal is the sum of eq:rIterTime over the T chunks
     whenever r = N/T is an integer."""
    rng = random.Random(0)
    for _ in range(50):
        N = rng.choice([64, 256, 1024])
        T = rng.choice([t for t in (1, 2, 4, 8, 16, 32) if N % t == 0])
        C1, abw, bc, c0 = rng.uniform(1, 9), rng.uniform(1, 9), rng.uniform(1, 9), rng.uniform(0, 3)
        a = A.total_time_sum(T, N, C1, abw, bc, c0)
        b = A.total_time(T, N, C1, abw, bc, c0)
        assert abs(a - b) <= 1e-9 * b


def test_unit_constant_values():
    """Hand evaluation of eq:NiterFinal with C1 = aBW = bC = 1, C0 = 0, N = 16:
    f(T) = 32 T + 32 + 256 + 256/T -> f(2) = f(4) = 480, f(3) = 469.33."""
    f = lambda T: A.total_time(T, 16, 1, 1, 1)
    assert f(2) == 480 and f(4) == 480
    assert abs(f(3) - (96 + 32 + 256 + 256 / 3)) < 1e-12


def test_optimum_is_stationary_point():
    """Opt-T-eq: the derivative of eq:NiterFinal vanishes at T*."""
    N, C1, abw, bc, c0 = 2048, 3.0, 5.0, 0.7, 0.0
    T = A.optimal_T(N, abw, bc, C1, c0)
    assert abs(T - math.sqrt(N * abw / (2 * bc))) < 1e-9
    h = 1e-4
    d = (A.total_time(T + h, N, C1, abw, bc) - A.total_time(T - h, N, C1, abw, bc)) / (2 * h)
    assert abs(d) < 1e-5 * A.total_time(T, N, C1, abw, bc)


def test_paper_validation_points():
    """C' = 0.1, T = sqrt(0.1 N) gives T = 8 at N = 512 after the
    power-of-2 rounding of P:L820; N = 2048 -> 16."""
    assert A.round_pow2(A.optimal_T_cprime(512, 0.1)) == 8
    assert A.round_pow2(A.optimal_T_cprime(2048, 0.1)) == 16


def test_sqrt_scaling():
    """'T is proportional to sqrt(N)' and T ~ sqrt(N/m) with SD
    (P:L917)."""
    for N in (100, 777, 4096):
        assert abs(A.optimal_T(4 * N, 2.0, 3.0) - 2 * A.optimal_T(N, 2.0, 3.0)) < 1e-9
        assert abs(A.optimal_T_sd(N, 2.0, 3.0, k=26, m=4) -
                   2 * A.optimal_T_sd(N, 2.0, 3.0, k=26, m=16)) < 1e-9


def test_sd_optimum_is_stationary():
    N, abw, bpc, k, m = 4096, 4.0, 9.0, 26, 4
    T = A.optimal_T_sd(N, abw, bpc, k, m)
    h = 1e-4
    d = (A.total_time_sd(T + h, N, 1, abw, bpc, k, m) - A.total_time_sd(T - h, N, 1, abw, bpc, k, m))
    assert abs(d / (2 * h)) < 1e-6 * A.total_time_sd(T, N, 1, abw, bpc, k, m)


def test_byte_model_matches_ledger_closed_forms():
    """The B200 byte model uses the same counts as the ledger pins:
    SDPA rows sum N(N+r)/2 for r | N (P:L699-704 summed), growth copies
    r*T^2 rows (cap_old read + cap_new written per growth)."""
    N, r, U, D, eb = 256, 16, 3, 64, 2
    row = 2 * U * D * eb
    b = A.bytes_per_layer(N, r, U, D, eb)
    T = N // r
    assert b["sdpa"] == row * N * (N + r) // 2
    assert b["copy"] == row * r * (T * T - 1)       # growths 1..T-1: (2i+1) r rows each


def test_advise_r_minimises_byte_model():
    """r* = sqrt(2N) minimises SDPA + copy bytes at equal bandwidths."""
    N = 4096
    best = min(range(8, 1025, 8), key=lambda r: A.model_time_b200(N, r, 8, 128, 2, 1, 1.0, 1.0))
    r_star = math.sqrt(2 * N)
    assert abs(best - r_star) <= 8
    assert A.advise_r(N) in (64, 128)              # T* = 45.25 -> nearest power of 2 is 32
    assert A.advise_r(N) == 128


def test_advise_r_copy_on_read_and_speculation():
    """Byte model with copy-on-read growth (growth adds the write of cap_new
    rows, N^2/(2r) in total) is minimised at r* = sqrt(N BW_r/BW_w): at equal
    bandwidths the brute-force minimum of row*(N(N+r)/2 + N^2/(2r)) over r is
    sqrt(N).  Speculation with m tokens per iteration reads cap once per
    iteration: r* = sqrt(m N) (T ~ sqrt(N/m))."""
    import math
    from paper_2511_12031_b200 import advisor
    for N in (1024, 4096, 16384):
        cost = lambda r: N * (N + r) / 2 + N * N / (2 * r)
        best = min(range(1, N + 1), key=cost)
        assert abs(best - math.sqrt(N)) <= 1
        assert advisor.advise_r(N, copy_on_read=True, pow2=False) == round(math.sqrt(N))
        for m in (2.0, 4.0):
            cost_m = lambda r: (N / m) * (N + r) / 2 + N * N / (2 * r)
            best_m = min(range(1, N + 1), key=cost_m)
            assert abs(advisor.advise_r(N, copy_on_read=True, pow2=False, tokens_per_iter=m)
                       - best_m) <= 1
    # defaults unchanged (separate copy, no speculation): sqrt(2N), T rounded to 2^k
    assert advisor.advise_r(4096) == 128
