"""Pins for the CPU oracle against what the paper and mathematics fix.

Each test names the passage it checks.  None of them re-types the oracle's
formula: they use closed forms printed in the paper, the paper's worked
example, brute-force values on tiny inputs, a library routine (torch fp64
SDPA) on exact-size inputs, and invariants between independent code paths.
"""
import json
import math
import os

import numpy as np
import pytest
import torch

import oracle as O
from paper_2511_12031_b200 import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _f32(x):
    return np.ascontiguousarray(np.asarray(x, dtype=np.float32))


def _run_decode(policy, *, B, H_kv, H_q, D, N, r, dtype="f32", seed=1, sdpa=True, layer=0):
    """Decode N tokens from an empty cache: append, then SDPA."""
    dt = O.F32 if dtype == "f32" else O.BF16
    orc = O.Oracle(B, H_kv, H_q, D, r, N, dtype=dt, policy=policy)
    outs = []
    for n in range(1, N + 1):
        x = synth.step_inputs(seed, layer, n, B=B, H_kv=H_kv, H_q=H_q, D=D, dtype=dtype)
        orc.append(x["k"], x["v"])
        if sdpa:
            outs.append(orc.sdpa(x["q"], n))
    return orc, outs


# --------------------------------------------------------- closed forms (ledger)

@pytest.mark.parametrize("N", [4, 16, 64, 256])
def test_iterative_copy_closed_form(oracle_mod, N):
    """total elements moved by iterative allocation over N tokens,
    K and V, all L layers = B*L*N*(N+1)*D (copy of n-1 rows + the new row)."""
    B, H, d, L = 2, 3, 4, 2
    eb = 4
    total = 0
    for layer in range(L):
        orc, _ = _run_decode(O.POLICY_ITERATIVE, B=B, H_kv=H, H_q=H, D=d, N=N, r=1,
                             sdpa=False, layer=layer)
        s = orc.stats()
        total += (s["copied_bytes"] + s["append_written_bytes"]) // eb
        assert s["alloc_events"] == N                       # one allocation per token
    D = H * d
    assert total == B * L * N * (N + 1) * D


@pytest.mark.parametrize("N", [4, 16, 64])
def test_sdpa_mac_closed_forms(oracle_mod, N):
    """P:L405-410 iterative MACs L*B*N*(N+1)*D; P:L435-437 upfront 2L*B*N^2*D;
    BMC sums 2*B*L*((i+1)r)*D over r iterations per chunk
    = L*B*N*(N+r)*D for r | N."""
    B, H, d, L = 2, 2, 4, 1
    D = H * d
    it, _ = _run_decode(O.POLICY_ITERATIVE, B=B, H_kv=H, H_q=H, D=d, N=N, r=1)
    assert it.stats()["macs"] == L * B * N * (N + 1) * D
    up, _ = _run_decode(O.POLICY_UPFRONT, B=B, H_kv=H, H_q=H, D=d, N=N, r=N)
    assert up.stats()["macs"] == 2 * L * B * N * N * D
    for r in (1, 2, 4, N):
        bm, _ = _run_decode(O.POLICY_BMC, B=B, H_kv=H, H_q=H, D=d, N=N, r=r)
        assert bm.stats()["macs"] == L * B * N * (N + r) * D


@pytest.mark.parametrize("N,r", [(37, 5), (64, 8), (50, 50), (9, 1), (100, 7)])
def test_bmc_allocation_counts(oracle_mod, N, r):
    """P:L609-611 (allocate once every r iterations, T = N/r) with the ragged
    last chunk of reading R12: after n appends alloc_events = ceil(n/r), the
    i-th growth copies i*r rows, the capacity law cap - valid in [0, r-1]
     holds after every append."""
    B, H, d = 1, 2, 2
    orc = O.Oracle(B, H, H, d, r, N, dtype=O.F32, policy=O.POLICY_BMC)
    for n in range(1, N + 1):
        x = synth.step_inputs(3, 0, n, B=B, H_kv=H, H_q=H, D=d, dtype="f32")
        orc.append(x["k"], x["v"])
        s = orc.stats()
        assert s["alloc_events"] == math.ceil(n / r)
        assert 0 <= s["capacity"] - n <= r - 1 or s["capacity"] == N
        c = math.ceil(n / r)
        assert s["copied_bytes"] == 2 * B * H * d * 4 * r * (c - 1) * c // 2
        assert s["init_written_bytes"] == 2 * B * H * d * 4 * sum(
            min((i + 1) * r, N) for i in range(c))


def test_copy_ratio_T_minus_1_over_N_plus_1(oracle_mod):
    """S:L537 / P:L392: BMC realloc copies over iterative copies+writes
    = (T-1)/(N+1) exactly at N=1024, T=32."""
    N, T = 1024, 32
    r = N // T
    bm, _ = _run_decode(O.POLICY_BMC, B=1, H_kv=1, H_q=1, D=1, N=N, r=r, sdpa=False)
    it, _ = _run_decode(O.POLICY_ITERATIVE, B=1, H_kv=1, H_q=1, D=1, N=N, r=1, sdpa=False)
    sb, si = bm.stats(), it.stats()
    num = sb["copied_bytes"]
    den = si["copied_bytes"] + si["append_written_bytes"]
    assert num * (N + 1) == den * (T - 1)


def test_toy_config_counters(oracle_mod):
    """tests/golden/toy_counters.json (BASELINE configs[0]; closed forms)."""
    g = _gold("toy_counters.json")
    c = g["config"]
    kw = dict(B=c["B"], H_kv=c["H"], H_q=c["H"], D=c["d"], N=c["N"])
    s16 = _run_decode(O.POLICY_BMC, r=16, **kw)[0].stats()
    for key, val in g["bmc_r16"].items():
        assert s16[key] == val, key
    s1 = _run_decode(O.POLICY_BMC, r=1, sdpa=False, **kw)[0].stats()
    for key in ("alloc_events", "copy_events", "copied_bytes"):
        assert s1[key] == g["bmc_r1"][key], key
    assert s1["init_written_bytes"] // c["eb"] == g["bmc_r1"]["init_written_elems"]
    su = _run_decode(O.POLICY_UPFRONT, r=c["N"], **kw)[0].stats()
    for key, val in g["upfront"].items():
        assert su[key] == val, key


# ----------------------------------------------------------- worked example

def test_sd_worked_example(oracle_mod):
    """P:L863-866 (wasted rows 7 -> 3 -> 1 -> 0), admission P:L867-869, no
    reallocation during speculation P:L904."""
    g = _gold("sd_worked_example.json")
    B, H, d = 1, 1, 2
    r = 8
    orc = O.Oracle(B, H, H, d, r, 64, dtype=O.F32, policy=O.POLICY_BMC)
    x = synth.step_inputs(5, 0, 0, B=B, H_kv=H, H_q=H, D=d, dtype="f32")
    orc.append(x["k"], x["v"])                      # cap 8, valid 1 -> 7 free rows
    s = orc.stats()
    assert s["capacity"] - s["valid_max"] == g["initial_free_rows"]
    allocs = s["alloc_events"]
    for i, step in enumerate(g["iterations"]):
        k = step["k"]
        xd = synth.step_inputs(5, 0, 100 + i, B=B, H_kv=H, H_q=H, D=d, k_draft=k,
                               dtype="f32")
        k_adm = orc.spec_write(xd["kd"], xd["vd"], k)
        assert k_adm == k
        s = orc.stats()
        wasted = s["capacity"] - s["valid_max"] - s["staged"]
        assert wasted == step["wasted_after_place"]
        orc.commit(step["accept"])
    assert orc.stats()["alloc_events"] - allocs == g["extra_alloc_events_during_sd"]


def test_admission_limits_to_free_rows(oracle_mod):
    """fewer free rows than k -> admit only the free rows, no growth;
    zero free rows -> k_adm = 0 (plain decode iteration)."""
    B, H, d, r = 2, 1, 2, 4
    orc = O.Oracle(B, H, H, d, r, 64, dtype=O.F32, policy=O.POLICY_BMC)
    for n in range(1, 3):
        x = synth.step_inputs(6, 0, n, B=B, H_kv=H, H_q=H, D=d, dtype="f32")
        orc.append(x["k"], x["v"])
    xd = synth.step_inputs(6, 0, 50, B=B, H_kv=H, H_q=H, D=d, k_draft=5, dtype="f32")
    assert orc.spec_write(xd["kd"], xd["vd"], 5) == 2
    assert orc.stats()["alloc_events"] == 1
    orc.commit(2)
    assert orc.spec_write(xd["kd"], xd["vd"], 5) == 0


# -------------------------------------------------------- attention values

def _one_row_oracle(case):
    d = case["d"]
    K, V = np.asarray(case["K"]), np.asarray(case["V"])
    n = K.shape[0]
    orc = O.Oracle(1, 1, 1, d, 1, n, dtype=O.F32, policy=O.POLICY_UPFRONT)
    for j in range(n):
        orc.append(_f32(K[j]), _f32(V[j]))
    return orc.sdpa(_f32(case["q"]), n).reshape(d)


@pytest.mark.parametrize("name", ["d2_identity", "single_row", "equal_scores", "one_hot"])
def test_sdpa_brute_force_cases(oracle_mod, name):
    """tests/golden/sdpa_brute_force.json."""
    case = next(c for c in _gold("sdpa_brute_force.json")["cases"] if c["name"] == name)
    exp = np.asarray(case["expected"])
    got = _one_row_oracle(case)
    np.testing.assert_allclose(got, exp, rtol=0, atol=1e-15)
    got2 = O.exact_sdpa(case["q"], case["K"], case["V"])
    np.testing.assert_allclose(got2, exp, rtol=0, atol=1e-15)
    if name == "d2_identity":
        e = math.exp(1 / math.sqrt(2))
        np.testing.assert_allclose(got, [e / (e + 1), 1 / (e + 1)], rtol=0, atol=1e-15)


def test_scale_uses_head_dim(oracle_mod):
    """Reading R4: the 1/sqrt(D) of P:L275 is 1/sqrt(d), d = head dim, after
    the MHA reshape to [B*H, 1, d].  Two rows, scores q.k/sqrt(d)
    = (8/sqrt(4), 0) = (4, 0) -> p = (e^4, 1)/(e^4+1)."""
    d = 4
    K = [[2.0, 2.0, 2.0, 2.0], [0.0, 0.0, 0.0, 0.0]]
    V = [[1.0, 0.0, 0.0, 0.0], [0.0, 1.0, 0.0, 0.0]]
    got = _one_row_oracle({"d": d, "q": [1.0, 1.0, 1.0, 1.0], "K": K, "V": V})
    e = math.exp(4.0)
    np.testing.assert_allclose(got[:2], [e / (e + 1), 1 / (e + 1)], rtol=0, atol=1e-15)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_matches_torch_fp64_sdpa_with_drafts(oracle_mod, dtype):
    """Library special case: exact-size (no padding) SDPA with a chain-causal
    boolean mask = torch.nn.functional.scaled_dot_product_attention in fp64
    (SD query block P:L446; reading R7)."""
    B, H_kv, H_q, d, n0, k = 2, 2, 4, 8, 11, 3
    dt = O.F32 if dtype == "f32" else O.BF16
    orc = O.Oracle(B, H_kv, H_q, d, 1, 64, dtype=dt, policy=O.POLICY_ITERATIVE)
    Ks, Vs = [], []
    for n in range(n0):
        x = synth.step_inputs(7, 0, n, B=B, H_kv=H_kv, H_q=H_q, D=d, dtype=dtype)
        orc.append(x["k"], x["v"])
        Ks.append(x["k"]); Vs.append(x["v"])
    xd = synth.step_inputs(7, 0, 99, B=B, H_kv=H_kv, H_q=H_q, D=d, t=1 + k, k_draft=k,
                           dtype=dtype)
    assert orc.spec_write(xd["kd"], xd["vd"], k) == k
    got = orc.sdpa(xd["q"], n0)
    Kall = torch.cat([torch.stack(Ks, 2), xd["kd"]], 2).double()     # [B][H_kv][n0+k][d]
    Vall = torch.cat([torch.stack(Vs, 2), xd["vd"]], 2).double()
    G = H_q // H_kv
    Kq = Kall.repeat_interleave(G, dim=1)
    Vq = Vall.repeat_interleave(G, dim=1)
    t = 1 + k
    mask = torch.zeros(t, n0 + k, dtype=torch.bool)
    for tau in range(t):
        mask[tau, : n0 + tau] = True
    ref = torch.nn.functional.scaled_dot_product_attention(
        xd["q"].double(), Kq, Vq, attn_mask=mask)
    np.testing.assert_allclose(got, ref.numpy(), rtol=0, atol=1e-12)


@pytest.mark.parametrize("r", [1, 3, 8, 16, 40])
def test_mask_invariance_bit_exact(oracle_mod, r):
    """the -1e9 bias on padded rows leaves SDPA equal to exact-
    prefix SDPA.  In fp64 the masked p_j are exactly 0 and trail the sums, so
    the result is bit-identical for every r; padded mass < 1e-30."""
    B, H, d, N = 1, 2, 8, 40
    orc = O.Oracle(B, H, H, d, r, N, dtype=O.F32, policy=O.POLICY_BMC)
    Ks, Vs = [], []
    for n in range(1, N + 1):
        x = synth.step_inputs(11, 0, n, B=B, H_kv=H, H_q=H, D=d, dtype="f32",
                              variant="peaky" if n % 3 == 0 else "normal")
        orc.append(x["k"], x["v"])
        Ks.append(x["k"].numpy()); Vs.append(x["v"].numpy())
        if n % 5 != 0 and n != N:
            continue
        got = orc.sdpa(x["q"], n)
        for hh in range(H):
            K = np.stack([k[0, hh] for k in Ks]).astype(np.float64)
            V = np.stack([v[0, hh] for v in Vs]).astype(np.float64)
            ref = O.exact_sdpa(x["q"].numpy()[0, hh, 0], K, V)
            assert np.array_equal(got[0, hh, 0], ref)
    assert math.exp(-1e9 + 50.0) < 1e-30


def test_gqa_equals_replicated_mha(oracle_mod):
    """P:L834-844 / S:L173: GQA output equals MHA with every KV head
    replicated G times (query head h reads KV head floor(h/G), reading R6)."""
    B, H_kv, H_q, d, N, r = 2, 2, 8, 4, 13, 4
    G = H_q // H_kv
    gq = O.Oracle(B, H_kv, H_q, d, r, N, dtype=O.BF16, policy=O.POLICY_BMC)
    mh = O.Oracle(B, H_q, H_q, d, r, N, dtype=O.BF16, policy=O.POLICY_BMC)
    for n in range(1, N + 1):
        x = synth.step_inputs(13, 0, n, B=B, H_kv=H_kv, H_q=H_q, D=d, dtype="bf16")
        gq.append(x["k"], x["v"])
        mh.append(x["k"].repeat_interleave(G, 1), x["v"].repeat_interleave(G, 1))
        assert np.array_equal(gq.sdpa(x["q"], n), mh.sdpa(x["q"], n))


# ------------------------------------------------------- policy degeneracy

@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_bmc_r1_equals_iterative(oracle_mod, dtype):
    """T = N/r: r=1 reallocates every token like iterative
    allocation: same contents, allocation/copy counts and
    bit-identical fp64 outputs from independent code paths."""
    kw = dict(B=2, H_kv=2, H_q=4, D=8, N=24, dtype=dtype)
    bm, ob = _run_decode(O.POLICY_BMC, r=1, **kw)
    it, oi = _run_decode(O.POLICY_ITERATIVE, r=1, **kw)
    for a, b in zip(ob, oi):
        assert np.array_equal(a, b)
    sb, si = bm.stats(), it.stats()
    for key in ("alloc_events", "copy_events", "copied_bytes", "init_written_bytes",
                "append_written_bytes", "capacity", "macs"):
        assert sb[key] == si[key], key
    for x, y in zip(bm.read_cache(), it.read_cache()):
        assert np.array_equal(x, y)


def test_bmc_rN_equals_upfront(oracle_mod):
    """r = N gives T = 1 allocation, i.e. upfront."""
    kw = dict(B=2, H_kv=1, H_q=2, D=8, N=20, dtype="bf16")
    bm, ob = _run_decode(O.POLICY_BMC, r=20, **kw)
    up, ou = _run_decode(O.POLICY_UPFRONT, r=20, **kw)
    for a, b in zip(ob, ou):
        assert np.array_equal(a, b)
    sb, su = bm.stats(), up.stats()
    assert sb["alloc_events"] == su["alloc_events"] == 1
    assert sb["copied_bytes"] == su["copied_bytes"] == 0
    assert sb["macs"] == su["macs"]
    for x, y in zip(bm.read_cache(), up.read_cache()):
        assert np.array_equal(x, y)


def test_content_equivalence_across_policies(oracle_mod):
    """after identical appends the committed rows are bitwise identical
    across iterative, upfront and BMC(r); padded rows are zero."""
    kw = dict(B=2, H_kv=2, H_q=2, D=4, N=19, dtype="bf16", sdpa=False)
    caches = []
    for pol, r in ((O.POLICY_ITERATIVE, 1), (O.POLICY_UPFRONT, 19), (O.POLICY_BMC, 5),
                   (O.POLICY_BMC, 7)):
        orc, _ = _run_decode(pol, r=r, N=19, **{k: v for k, v in kw.items() if k != "N"})
        K, V = orc.read_cache()
        assert not K[:, 19:].any() and not V[:, 19:].any()
        caches.append((K[:, :19], V[:, :19]))
    for K, V in caches[1:]:
        assert np.array_equal(K, caches[0][0]) and np.array_equal(V, caches[0][1])


def test_unmasked_upfront_is_wrong(oracle_mod):
    """Negative test: without the mask the e^0 = 1 terms of zero rows
    change the output; with it the output matches the exact prefix."""
    d = 2
    q = np.array([1.0, 0.5]); K = np.array([[1.0, 0.0]]); V = np.array([[2.0, -1.0]])
    masked = _one_row_oracle({"d": d, "q": q, "K": K, "V": V})   # exact, 1 row
    Kpad = np.vstack([K, np.zeros((3, d))]); Vpad = np.vstack([V, np.zeros((3, d))])
    unmasked = O.exact_sdpa(q, Kpad, Vpad)                        # softmax over zeros too
    assert np.array_equal(masked, V[0])
    assert not np.allclose(unmasked, V[0])


# -------------------------------------------------------- speculative commit

def test_commit_equals_sequential_appends(oracle_mod):
    """S:L362-366 / P:L447: committing the m accepted chain drafts gives the
    cache that m plain appends of the same rows give; rejected rows are zero
    again (reading R9), capacity unchanged during speculation."""
    B, H, d, r, N = 2, 2, 4, 8, 64
    a = O.Oracle(B, H, H, d, r, N, dtype=O.BF16, policy=O.POLICY_BMC)
    b = O.Oracle(B, H, H, d, r, N, dtype=O.BF16, policy=O.POLICY_BMC)
    for n in range(3):
        x = synth.step_inputs(17, 0, n, B=B, H_kv=H, H_q=H, D=d, dtype="bf16")
        a.append(x["k"], x["v"]); b.append(x["k"], x["v"])
    k, m = 4, 2
    xd = synth.step_inputs(17, 0, 77, B=B, H_kv=H, H_q=H, D=d, k_draft=k, t=1 + k,
                           dtype="bf16")
    cap0 = a.stats()["capacity"]
    assert a.spec_write(xd["kd"], xd["vd"], k) == k
    a.sdpa(xd["q"], 3)
    a.commit(m)
    assert a.stats()["capacity"] == cap0
    for i in range(m):
        b.append(xd["kd"][:, :, i].contiguous(), xd["vd"][:, :, i].contiguous())
    for x, y in zip(a.read_cache(), b.read_cache()):
        assert np.array_equal(x, y)
    K, V = a.read_cache()
    assert not K[:, 3 + m:].any() and not V[:, 3 + m:].any()


def test_commit_rows_per_row_lengths(oracle_mod):
    """Reading R11: per-row acceptance at B > 1; masks use each row's length."""
    B, H, d, r, N = 3, 1, 4, 16, 64
    orc = O.Oracle(B, H, H, d, r, N, dtype=O.F32, policy=O.POLICY_BMC)
    x = synth.step_inputs(19, 0, 0, B=B, H_kv=H, H_q=H, D=d, dtype="f32")
    orc.append(x["k"], x["v"])
    xd = synth.step_inputs(19, 0, 1, B=B, H_kv=H, H_q=H, D=d, k_draft=3, t=4, dtype="f32")
    orc.spec_write(xd["kd"], xd["vd"], 3)
    orc.commit_rows([0, 3, 1])
    assert list(orc.valid()) == [1, 4, 2]
    q = synth.step_inputs(19, 0, 2, B=B, H_kv=H, H_q=H, D=d, dtype="f32")["q"]
    with pytest.raises(O.OracleError):
        orc.sdpa(q, 1)                                  # not uniform -> STATE
    out = orc.sdpa(q, -1)
    K, V = orc.read_cache()
    for b, n in enumerate([1, 4, 2]):
        ref = O.exact_sdpa(q.numpy()[b, 0, 0], K[b, :n].astype(np.float64),
                           V[b, :n].astype(np.float64))
        assert np.array_equal(out[b, 0, 0], ref)


def test_error_codes(oracle_mod):
    """Boundary errors: CAPACITY at N_max, STATE for a
    second spec_write / append while staged, ARG for bad commits and n_valid=0."""
    orc = O.Oracle(1, 1, 1, 2, 2, 2, dtype=O.F32, policy=O.POLICY_BMC)
    z = _f32([0.5, 0.5])
    orc.append(z, z); orc.append(z, z)
    with pytest.raises(O.OracleError) as e:
        orc.append(z, z)
    assert e.value.code == -3
    with pytest.raises(O.OracleError) as e:
        orc.commit(1)
    assert e.value.code == -2
    with pytest.raises(O.OracleError) as e:
        orc.sdpa(_f32([1, 1]), 0)
    assert e.value.code == -1
    with pytest.raises(O.OracleError) as e:
        O.Oracle(1, 3, 4, 2, 2, 2)
    assert e.value.code == -1
    o2 = O.Oracle(1, 1, 1, 2, 4, 8, dtype=O.F32, policy=O.POLICY_BMC)
    o2.append(z, z)
    kd = _f32([[1, 2], [3, 4]])
    assert o2.spec_write(kd, kd, 2) == 2
    with pytest.raises(O.OracleError) as e:
        o2.spec_write(kd, kd, 2)
    assert e.value.code == -2
    with pytest.raises(O.OracleError) as e:
        o2.append(z, z)
    assert e.value.code == -2
    with pytest.raises(O.OracleError) as e:
        o2.commit(3)
    assert e.value.code == -1


def test_footprint_example():
    """B=64, L=64, D=4096, N=2048 half precision K and V need ~137 GB
    (the layout's bytes per row x rows, 2 tensors)."""
    B, L, D, N, eb = 64, 64, 4096, 2048, 2
    assert abs(2 * B * L * N * D * eb / 1e9 - 137.4) < 0.1


# ------------------------------------------------------------ token trees

def _tree_ancestors(parent, i):
    out = []
    while i >= 0:
        out.append(i)
        i = parent[i]
    return sorted(out)


def test_tree_worked_example(oracle_mod):
    """P:L863-866 with the figure's 4-node tree: S11 (root), S21 and S22
    (children of S11), S31 (child of S21), BFS order [S11, S21, S22, S31];
    7 free rows -> 3 wasted; (S11, S22) accepted -> next tree leaves 1; S'11
    accepted -> next tree leaves 0; no reallocation."""
    B, H, d, r = 1, 1, 2, 8
    orc = O.Oracle(B, H, H, d, r, 64, dtype=O.F32, policy=O.POLICY_BMC)
    x = synth.step_inputs(5, 0, 0, B=B, H_kv=H, H_q=H, D=d, dtype="f32")
    orc.append(x["k"], x["v"])
    parent = [-1, 0, 0, 1]
    allocs = orc.stats()["alloc_events"]
    for i, (wasted, path) in enumerate([(3, [0, 2]), (1, [0]), (0, [])]):
        xd = synth.step_inputs(5, 0, 200 + i, B=B, H_kv=H, H_q=H, D=d, k_draft=4, dtype="f32")
        assert orc.spec_write_tree(xd["kd"], xd["vd"], 4, parent) == 4
        s = orc.stats()
        assert s["capacity"] - s["valid_max"] - s["staged"] == wasted
        orc.commit_path([path])
    assert orc.stats()["alloc_events"] == allocs


def test_tree_mask_is_ancestor_rule(oracle_mod):
    """Each node's output equals textbook SDPA over exactly the committed
    prefix, its ancestors and itself (S:L351-355 ancestor rule); siblings and
    cousins are invisible.  Bit-exact in fp64 (masked terms are exact zeros)."""
    rng = np.random.default_rng(3)
    B, H, d, n0 = 2, 2, 8, 9
    for trial in range(4):
        k = int(rng.integers(2, 12))
        parent = [-1] + [int(rng.integers(-1, i)) for i in range(1, k)]
        orc = O.Oracle(B, H, H, d, 32, 64, dtype=O.F32, policy=O.POLICY_BMC)
        Ks, Vs = [], []
        for n in range(n0):
            x = synth.step_inputs(11 + trial, 0, n, B=B, H_kv=H, H_q=H, D=d, dtype="f32")
            orc.append(x["k"], x["v"])
            Ks.append(x["k"].numpy()); Vs.append(x["v"].numpy())
        xd = synth.step_inputs(11 + trial, 0, 99, B=B, H_kv=H, H_q=H, D=d, t=1 + k,
                               k_draft=k, dtype="f32")
        k_adm = orc.spec_write_tree(xd["kd"], xd["vd"], k, parent)
        assert k_adm == k
        out = orc.sdpa(xd["q"], n0)
        for b in range(B):
            for h in range(H):
                pre_k = [Ks[n][b, h] for n in range(n0)]
                pre_v = [Vs[n][b, h] for n in range(n0)]
                q = xd["q"].numpy()[b, h]
                ref0 = O.exact_sdpa(q[0], np.array(pre_k, dtype=np.float64),
                                    np.array(pre_v, dtype=np.float64))
                assert np.array_equal(out[b, h, 0], ref0)
                for i in range(k):
                    rows = _tree_ancestors(parent, i)
                    Kg = np.array(pre_k + [xd["kd"].numpy()[b, h, j] for j in rows],
                                  dtype=np.float64)
                    Vg = np.array(pre_v + [xd["vd"].numpy()[b, h, j] for j in rows],
                                  dtype=np.float64)
                    assert np.array_equal(out[b, h, 1 + i], O.exact_sdpa(q[1 + i], Kg, Vg))


def test_chain_tree_equals_chain_drafts(oracle_mod):
    """A chain is the tree parent[i] = i-1: outputs, commit and cache equal
    the chain-draft calls (commit(n) == commit_path([0..n-1]))."""
    B, H, d = 2, 1, 4
    a = O.Oracle(B, H, H, d, 8, 64, dtype=O.BF16, policy=O.POLICY_BMC)
    b = O.Oracle(B, H, H, d, 8, 64, dtype=O.BF16, policy=O.POLICY_BMC)
    for n in range(3):
        x = synth.step_inputs(21, 0, n, B=B, H_kv=H, H_q=H, D=d, dtype="bf16")
        a.append(x["k"], x["v"]); b.append(x["k"], x["v"])
    xd = synth.step_inputs(21, 0, 50, B=B, H_kv=H, H_q=H, D=d, t=5, k_draft=4, dtype="bf16")
    assert a.spec_write(xd["kd"], xd["vd"], 4) == 4
    assert b.spec_write_tree(xd["kd"], xd["vd"], 4, [-1, 0, 1, 2]) == 4
    assert np.array_equal(a.sdpa(xd["q"], 3), b.sdpa(xd["q"], 3))
    a.commit_rows([2, 3])
    b.commit_path([[0, 1], [0, 1, 2]])
    for x, y in zip(a.read_cache(), b.read_cache()):
        assert np.array_equal(x, y)


def test_commit_path_equals_appending_the_path(oracle_mod):
    """Committing an accepted root-to-node path moves exactly those rows, in
    depth order, behind the committed prefix: the cache equals
    appending the path's K/V rows; other staged rows are zero again."""
    B, H, d = 1, 2, 4
    parent = [-1, -1, 0, 1, 1, 3, 2]
    path = [1, 3, 5]
    a = O.Oracle(B, H, H, d, 16, 64, dtype=O.F32, policy=O.POLICY_BMC)
    b = O.Oracle(B, H, H, d, 16, 64, dtype=O.F32, policy=O.POLICY_BMC)
    x = synth.step_inputs(23, 0, 0, B=B, H_kv=H, H_q=H, D=d, dtype="f32")
    a.append(x["k"], x["v"]); b.append(x["k"], x["v"])
    xd = synth.step_inputs(23, 0, 1, B=B, H_kv=H, H_q=H, D=d, k_draft=len(parent), dtype="f32")
    a.spec_write_tree(xd["kd"], xd["vd"], len(parent), parent)
    a.commit_path([path])
    for j in path:
        b.append(xd["kd"][:, :, j].contiguous(), xd["vd"][:, :, j].contiguous())
    for u, w in zip(a.read_cache(), b.read_cache()):
        assert np.array_equal(u, w)
    assert list(a.valid()) == [1 + len(path)]


def test_tree_errors(oracle_mod):
    orc = O.Oracle(1, 1, 1, 2, 8, 64, dtype=O.F32, policy=O.POLICY_BMC)
    z = _f32([0.5, 0.5])
    orc.append(z, z)
    kd = _f32(np.ones((3, 2)))
    with pytest.raises(O.OracleError) as e:
        orc.spec_write_tree(kd, kd, 3, [-1, 1, 0])         # parent not before child
    assert e.value.code == -1
    orc.spec_write_tree(kd, kd, 3, [-1, 0, 0])
    with pytest.raises(O.OracleError) as e:
        orc.commit(1)                                      # trees commit paths
    assert e.value.code == -2
    with pytest.raises(O.OracleError) as e:
        orc.commit_path([[0, 0]])                          # not parent-linked
    assert e.value.code == -1
    orc.commit_path([[0, 2]])
    assert list(orc.valid()) == [3]


# ------------------------------------------------------- bulk (prompt) append

def _prompt(seed, B, H_kv, D, n, dtype="bf16"):
    """[B][H_kv][n][D] prompt rows from the per-step streams of steps 1..n."""
    ks, vs = [], []
    for t in range(1, n + 1):
        x = synth.step_inputs(seed, 0, t, B=B, H_kv=H_kv, H_q=H_kv, D=D, dtype=dtype)
        ks.append(x["k"])
        vs.append(x["v"])
    return torch.stack(ks, dim=2).contiguous(), torch.stack(vs, dim=2).contiguous()


@pytest.mark.parametrize("policy,r", [(O.POLICY_BMC, 4), (O.POLICY_BMC, 16),
                                      (O.POLICY_ITERATIVE, 1), (O.POLICY_UPFRONT, 40)])
def test_append_n_equals_single_appends(oracle_mod, policy, r):
    """A bulk append of n rows leaves the cache contents and lengths that n
    single appends leave (P:L609 in-place writes; S:L104 prompt ingestion),
    including after earlier decode rows; padded rows stay zero."""
    B, H, D, N = 2, 3, 8, 40
    a = O.Oracle(B, H, H, D, r, N, dtype=O.BF16, policy=policy)
    b = O.Oracle(B, H, H, D, r, N, dtype=O.BF16, policy=policy)
    K1, V1 = _prompt(5, B, H, D, 13)
    K2, V2 = _prompt(6, B, H, D, 9)
    a.append_n(K1, V1, 13)
    a.append_n(K2, V2, 9)
    for K, V, n in ((K1, V1, 13), (K2, V2, 9)):
        for i in range(n):
            b.append(K[:, :, i].contiguous(), V[:, :, i].contiguous())
    assert list(a.valid()) == list(b.valid()) == [22, 22]
    Ka, Va = a.read_cache()
    Kb, Vb = b.read_cache()
    assert np.array_equal(Ka[:, :22], Kb[:, :22]) and np.array_equal(Va[:, :22], Vb[:, :22])
    assert not Ka[:, 22:].any() and not Va[:, 22:].any()
    assert a.stats()["append_written_bytes"] == b.stats()["append_written_bytes"]


@pytest.mark.parametrize("P", [1, 15, 16, 17, 100, 128])
def test_prefill_ledger_closed_form(oracle_mod, P):
    """Prompt ingestion is one allocation: from an empty BMC cache
    with r=16 a prompt of P rows ends at cap = r*ceil(P/r) (min r, max N_max)
    after one growth beyond the first chunk, copying nothing; ITERATIVE
    allocates exactly P rows; UPFRONT allocates nothing more."""
    B, H, D, N, r = 1, 2, 4, 128, 16
    K, V = _prompt(7, B, H, D, P, dtype="f32")
    U, rb = B * H, D * 4
    bm = O.Oracle(B, H, H, D, r, N, dtype=O.F32, policy=O.POLICY_BMC)
    bm.append_n(K, V, P)
    s = bm.stats()
    cap = min(N, max(r, r * math.ceil(P / r)))
    assert s["capacity"] == cap and s["valid_max"] == P
    assert s["alloc_events"] == (1 if P <= r else 2)
    assert s["copy_events"] == (0 if P <= r else 1) and s["copied_bytes"] == 0
    assert s["init_written_bytes"] == 2 * U * rb * (r + (cap if P > r else 0))
    it = O.Oracle(B, H, H, D, 1, N, dtype=O.F32, policy=O.POLICY_ITERATIVE)
    it.append_n(K, V, P)
    s = it.stats()
    assert s["capacity"] == P and s["alloc_events"] == 1 and s["copied_bytes"] == 0
    up = O.Oracle(B, H, H, D, N, N, dtype=O.F32, policy=O.POLICY_UPFRONT)
    up.append_n(K, V, P)
    assert up.stats()["alloc_events"] == 1 and up.stats()["capacity"] == N


def test_prefill_then_decode_sdpa_is_exact(oracle_mod):
    """After a bulk prompt the masked SDPA over the padded cache equals the
    textbook SDPA over exactly the prompt rows."""
    B, H, D, N, r, P = 1, 1, 8, 64, 16, 21
    K, V = _prompt(8, B, H, D, P, dtype="f32")
    orc = O.Oracle(B, H, H, D, r, N, dtype=O.F32, policy=O.POLICY_BMC)
    orc.append_n(K, V, P)
    q = synth.step_inputs(8, 0, P + 1, B=B, H_kv=H, H_q=H, D=D, dtype="f32")["q"]
    got = orc.sdpa(q, P).reshape(D)
    ref = O.exact_sdpa(q.numpy().reshape(D).astype(np.float64),
                       K.numpy().reshape(P, D).astype(np.float64),
                       V.numpy().reshape(P, D).astype(np.float64))
    assert np.abs(got - ref).max() <= 1e-12


def test_append_n_errors(oracle_mod):
    """CAPACITY past N_max, STATE with staged drafts, n = 0 is a no-op."""
    B, H, D, N = 1, 1, 4, 10
    orc = O.Oracle(B, H, H, D, 4, N, dtype=O.F32, policy=O.POLICY_BMC)
    K, V = _prompt(9, B, H, D, 11, dtype="f32")
    with pytest.raises(O.OracleError) as e:
        orc.append_n(K, V, 11)
    assert e.value.code == -3
    orc.append_n(K[:, :, :0], V[:, :, :0], 0)
    assert orc.stats()["valid_max"] == 0
    K3, V3 = _prompt(9, B, H, D, 3, dtype="f32")
    orc.append_n(K3, V3, 3)
    kd = torch.zeros(B, H, 1, D)
    orc.spec_write(kd, kd, 1)
    with pytest.raises(O.OracleError) as e:
        orc.append_n(K3, V3, 3)
    assert e.value.code == -2


# ------------------------------------------- ITERATIVE with speculation (R17)

def _iter_sd_run(P, I, k, m, *, B=2, H=2, d=4, N=256, sdpa=False, check=None):
    """Prompt of P single appends, then I speculative iterations under the
    ITERATIVE policy: append x_last, spec_write k drafts, (SDPA), commit m."""
    orc = O.Oracle(B, H, H, d, 1, N, dtype=O.F32, policy=O.POLICY_ITERATIVE)
    for n in range(P):
        x = synth.step_inputs(41, 0, n, B=B, H_kv=H, H_q=H, D=d, dtype="f32")
        orc.append(x["k"], x["v"])
        if check:
            check("append", orc.stats())
    for i in range(I):
        x = synth.step_inputs(41, 0, 1000 + i, B=B, H_kv=H, H_q=H, D=d, dtype="f32")
        orc.append(x["k"], x["v"])
        if check:
            check("append", orc.stats())
        xd = synth.step_inputs(41, 0, 2000 + i, B=B, H_kv=H, H_q=H, D=d, k_draft=k,
                               t=1 + k, dtype="f32")
        ka = orc.spec_write(xd["kd"], xd["vd"], k)
        if check:
            check("spec", orc.stats())
        if sdpa:
            orc.sdpa(xd["q"][:, :, :1 + ka].contiguous(), orc.stats()["valid_max"])
        orc.commit(min(m, ka))
        if check:
            check("commit", orc.stats())
    return orc


def test_iterative_sd_buffers_are_exact_size(oracle_mod):
    """P:L340 ("copies them into the new K and V matrices (size increased by one
    additional row)") and the update_cache listing P:L352-359 (allocate, then
    concat the new block): an iterative buffer never holds a padded row.  So
    after an append the capacity is the committed length, after a speculative
    write it is the committed length plus the drafts, and a commit that
    rejects drafts leaves them as zero rows that the next append drops
    (reading R17).  Each reallocation copies exactly the rows that hold data
    (valid_max before the call)."""
    prev = {}

    def check(what, s):
        if what == "append":
            assert s["capacity"] == s["valid_max"], s
        elif what == "spec":
            assert s["capacity"] == s["valid_max"] + s["staged"], s
        else:
            assert s["staged"] == 0 and s["capacity"] == prev["capacity"], s
        if what != "commit":
            # one new allocation per call; it copies the rows that held data
            assert s["alloc_events"] == prev.get("alloc_events", 0) + 1
            moved = (s["copied_bytes"] - prev.get("copied_bytes", 0)) // (2 * 2 * 2 * 4 * 4)
            assert moved == prev.get("valid_max", 0), (what, moved, prev)
        prev.update(s)

    _iter_sd_run(P=5, I=9, k=4, m=2, check=check)
    prev.clear()
    _iter_sd_run(P=1, I=6, k=3, m=0, check=check)


@pytest.mark.parametrize("P,I,k,m", [(5, 9, 4, 2), (1, 7, 3, 3), (12, 4, 8, 0), (3, 10, 1, 1)])
def test_iterative_sd_ledger_closed_form(oracle_mod, P, I, k, m):
    """HF-concat growth under speculation (reading R17), summed by
    hand.  Prompt: P appends copy sum_{n<P} n = P(P-1)/2 rows and write
    sum_{n<=P} n = P(P+1)/2 rows per unit.  Iteration i starts at
    v_i = P + i(1+m): the append copies v_i rows into v_i+1, the speculative
    write copies v_i+1 rows into v_i+1+k, so over I iterations the copies are
    I(2P+1) + (1+m)I(I-1) rows and the initialised rows I(2P+2+k) + (1+m)I(I-1);
    2 allocations per iteration; the final capacity is v_{I-1}+1+k and the
    valid length P + I(1+m).  Each iteration's verify SDPA streams all
    v_i+1+k rows (S 8(d)): sum = I(P+1+k) + (1+m)I(I-1)/2 rows.
    MACs: 2*B*H_q*t*cap*D per call with t = 1+k."""
    B, H, d = 2, 2, 4
    orc = _iter_sd_run(P, I, k, m, B=B, H=H, d=d, sdpa=True)
    s = orc.stats()
    row = 2 * B * H * d * 4                       # K and V, all units, fp32
    assert s["alloc_events"] == P + 2 * I
    assert s["copy_events"] == (P - 1) + 2 * I
    assert s["copied_bytes"] == row * (P * (P - 1) // 2 + I * (2 * P + 1) + (1 + m) * I * (I - 1))
    assert s["init_written_bytes"] == row * (P * (P + 1) // 2 + I * (2 * P + 2 + k)
                                             + (1 + m) * I * (I - 1))
    assert s["valid_max"] == s["valid_min"] == P + I * (1 + m)
    assert s["capacity"] == P + (I - 1) * (1 + m) + 1 + k
    rows_read = I * (P + 1 + k) + (1 + m) * I * (I - 1) // 2
    assert s["kv_bytes_read"] == row * rows_read
    assert s["macs"] == 2 * B * H * (1 + k) * rows_read * d


def test_iterative_sd_matches_bmc_sd(oracle_mod):
    """Reading R17 vs P:L864-869: with room for every draft, ITERATIVE and
    BMC speculation hold the same committed rows and give bit-identical fp64
    outputs (mask invariance); only the ledger differs."""
    B, H, d, k = 2, 2, 4, 3
    it = O.Oracle(B, H, H, d, 1, 128, dtype=O.BF16, policy=O.POLICY_ITERATIVE)
    bm = O.Oracle(B, H, H, d, 64, 128, dtype=O.BF16, policy=O.POLICY_BMC)
    for i, m in enumerate([2, 0, 3, 1, 3]):
        x = synth.step_inputs(43, 0, i, B=B, H_kv=H, H_q=H, D=d, dtype="bf16")
        xd = synth.step_inputs(43, 0, 100 + i, B=B, H_kv=H, H_q=H, D=d, k_draft=k, t=1 + k,
                               dtype="bf16")
        outs = []
        for orc in (it, bm):
            orc.append(x["k"], x["v"])
            assert orc.spec_write(xd["kd"], xd["vd"], k) == k
            outs.append(orc.sdpa(xd["q"], orc.stats()["valid_max"]))
            orc.commit(m)
        assert np.array_equal(outs[0], outs[1])
    n = it.stats()["valid_max"]
    assert bm.stats()["valid_max"] == n
    Ki, Vi = it.read_cache()
    Kb, Vb = bm.read_cache()
    assert np.array_equal(Ki[:, :n], Kb[:, :n]) and np.array_equal(Vi[:, :n], Vb[:, :n])


@pytest.mark.parametrize("N,r", [(32, 4), (40, 8), (30, 7)])
def test_kv_bytes_read_closed_form(oracle_mod, N, r):
    """SURVEY 8(d) algorithmic bytes: every SDPA streams K and V over all cap
    rows, padding included ("wasteful computation" of the zero rows).
    Decoding N tokens reads 2*U*D*eb * sum_n cap(n) bytes with
    cap(n) = min(r*ceil(n/r), N) (BMC), n (ITERATIVE), N (UPFRONT); for r | N the
    BMC sum is N(N+r)/2 rows."""
    B, H, d = 1, 2, 2
    row = 2 * B * H * d * 4
    bm, _ = _run_decode(O.POLICY_BMC, B=B, H_kv=H, H_q=H, D=d, N=N, r=r)
    assert bm.stats()["kv_bytes_read"] == row * sum(min(r * math.ceil(n / r), N)
                                                    for n in range(1, N + 1))
    if N % r == 0:
        assert bm.stats()["kv_bytes_read"] == row * N * (N + r) // 2
    it, _ = _run_decode(O.POLICY_ITERATIVE, B=B, H_kv=H, H_q=H, D=d, N=N, r=1)
    assert it.stats()["kv_bytes_read"] == row * N * (N + 1) // 2
    up, _ = _run_decode(O.POLICY_UPFRONT, B=B, H_kv=H, H_q=H, D=d, N=N, r=N)
    assert up.stats()["kv_bytes_read"] == row * N * N
    assert bm.stats()["sdpa_calls"] == it.stats()["sdpa_calls"] == N
