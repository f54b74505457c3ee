"""GPU parity: libbmc (sm_100a kernels, called through the C ABI) against the
CPU oracle, element by element, on the same seeded inputs.

Sizes span several 16 KiB tiles, ragged tails (r not dividing N, caps not a
multiple of the tile rows), multi-CTA split-K segments and every policy.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from harness import Pair  # noqa: E402
from paper_2511_12031_b200 import bmc, synth  # noqa: E402


@pytest.fixture(autouse=True, scope="module")
def _built():
    import __graft_entry__
    __graft_entry__.build()
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"


def _decode(p: Pair, steps: int, check_every: int = 1, state_every: int = 0):
    for i in range(steps):
        p.append()
        if (i + 1) % check_every == 0 or i + 1 == steps:
            p.sdpa()
        if state_every and (i + 1) % state_every == 0:
            p.check_state()
    p.check_state()


def test_toy_config_full_run():
    """BASELINE configs[0]: B=1, 2 heads, head_dim 64, N_max=128, r=16, fp32,
    128 decode steps, every SDPA output and the final state checked."""
    p = Pair(1, 2, 2, 64, 16, 128, dtype="f32")
    _decode(p, 128, check_every=1, state_every=16)
    s = p.gpu.stats()
    assert s["alloc_events"] == 8 and s["copy_events"] == 7
    p.close()


@pytest.mark.parametrize("policy,r", [("bmc", 1), ("bmc", 7), ("bmc", 32), ("bmc", 300),
                                      ("iterative", 1), ("upfront", 300)])
def test_policies_bf16_d128(policy, r):
    """Every policy, bf16 head_dim 128, ragged N=300 (r does not divide N)."""
    p = Pair(3, 4, 4, 128, r, 300, dtype="bf16", policy=policy, seed=3)
    _decode(p, 300, check_every=13, state_every=97)
    p.close()


@pytest.mark.parametrize("dtype,D", [("bf16", 64), ("f32", 128), ("f32", 64)])
def test_dtypes_and_head_dims(dtype, D):
    p = Pair(2, 3, 3, D, 24, 200, dtype=dtype, seed=5)
    _decode(p, 200, check_every=9, state_every=50)
    p.close()


@pytest.mark.parametrize("H_kv,H_q", [(2, 8), (8, 32), (1, 4)])
def test_gqa(H_kv, H_q):
    """GQA: G = H_q/H_kv query heads share one KV head."""
    p = Pair(2, H_kv, H_q, 128, 64, 256, dtype="bf16", seed=7)
    _decode(p, 256, check_every=17)
    p.close()


@pytest.mark.parametrize("variant", ["peaky", "outlier"])
def test_structured_inputs(variant):
    """Near one-hot softmax (Q x 8) and +large-score outliers (max subtraction)."""
    p = Pair(2, 4, 4, 128, 32, 160, dtype="bf16", seed=9, variant=variant)
    _decode(p, 160, check_every=5)
    p.close()


def test_pool_reserve_then_decode():
    """bmc_pool_reserve maps memory into the growth pool up front; growths
    afterwards are carved from it and the decode matches the oracle."""
    assert bmc.bmc_pool_reserve(-1, 256 << 20) == 0
    assert bmc.bmc_pool_reserve(0, 0) == 0
    p = Pair(2, 2, 4, 128, 16, 120, dtype="bf16", seed=41)
    _decode(p, 120, check_every=7)
    p.close()


@pytest.mark.parametrize("path", [1, 0])
@pytest.mark.parametrize("ctas", [1, 2, 3, 7, 64, 500])
def test_split_k_segments(ctas, path):
    """Force the number of persistent CTAs so units split across many / few
    CTAs (split-K combine) and CTAs span many units; CUDA-core kernel (path
    1) and the auto tcgen05 kernel (CTAs capped at the SM count)."""
    p = Pair(2, 4, 8, 128, 50, 700, dtype="bf16", seed=11, ctas=ctas)
    p.gpu.set_option(bmc.BMC_OPT_ATTN_PATH, path)
    _decode(p, 700, check_every=37)
    p.close()


@pytest.mark.parametrize("B,H_kv,H_q,k", [(1, 1, 1, 4), (4, 2, 2, 4), (3, 2, 4, 3),
                                          (2, 2, 16, 8)])
def test_speculative_chain(B, H_kv, H_q, k):
    """SD in the padded rows: append x_last, place k chain drafts
    (admission-limited), verify with t = 1 + k_adm query rows, per-row commit
    with rollback of rejected rows.  (2,2,16,8) gives M = 8*9 = 72
    query rows per KV head (the 70B-shaped verify)."""
    p = Pair(B, H_kv, H_q, 128, 16, 400, dtype="bf16", seed=13)
    for _ in range(5):
        p.append()
    p.sdpa()
    it = 0
    while p.orc.stats()["valid_max"] < 380:
        p.append()
        k_adm = p.spec_write(k)
        p.sdpa(n_valid=-1)
        m = synth.acceptance(13, it, B, k_adm)
        p.commit_rows(m)
        it += 1
        if it % 10 == 0:
            p.check_state()
    p.check_state()
    p.close()


def test_sd_admission_and_allocs():
    """Admission never grows the cache; the allocation count is the plain-BMC
    one."""
    p = Pair(2, 2, 2, 128, 8, 64, dtype="bf16", seed=15)
    p.append()
    allocs = p.gpu.stats()["alloc_events"]
    assert p.spec_write(20) == 7
    p.sdpa()
    p.commit(3)
    assert p.gpu.stats()["alloc_events"] == allocs
    p.check_state()
    p.close()


@pytest.mark.parametrize("host_io", [True, "pinned"])
def test_host_pointer_io(host_io):
    """The end-to-end path: host inputs staged inside the call (pageable: on
    the compute stream; pinned: on the handle's upload stream, event-ordered),
    host output (pinned: downloaded on the handle's download stream)."""
    p = Pair(2, 2, 4, 128, 16, 110, dtype="bf16", seed=17, host_io=host_io)
    _decode(p, 100, check_every=7)
    p.append()
    p.spec_write(3)
    p.sdpa()
    p.commit(1)
    p.check_state()
    p.close()


def test_single_row_and_tiny():
    """n_valid = 1 (single visible row -> O = v exactly up to rounding), B*H = 1."""
    p = Pair(1, 1, 1, 128, 4, 9, dtype="f32", seed=19)
    p.append()
    og, ref = p.sdpa()
    _decode(p, 8, check_every=1)
    p.close()


def test_error_codes_gpu():
    g = bmc.KVCache(1, 1, 1, 64, 2, 2, dtype="f32")
    z = torch.zeros(1, 1, 64, device="cuda")
    g.append(z, z)
    g.append(z, z)
    with pytest.raises(bmc.BMCError) as e:
        g.append(z, z)
    assert e.value.code == bmc.BMC_ERR_CAPACITY
    with pytest.raises(bmc.BMCError) as e:
        g.commit(1)
    assert e.value.code == bmc.BMC_ERR_STATE
    q = torch.zeros(1, 1, 1, 64, device="cuda")
    with pytest.raises(bmc.BMCError) as e:
        g.sdpa(q, 1)
    assert e.value.code == bmc.BMC_ERR_STATE
    g.close()


def test_arena_kinds_agree():
    """VMM arena and stream-ordered pool give identical results."""
    for kind in (0, 1):
        p = Pair(2, 2, 2, 128, 8, 120, dtype="bf16", seed=21)
        p.gpu.set_option(bmc.BMC_OPT_ARENA, kind)
        _decode(p, 120, check_every=11, state_every=40)
        p.close()


def test_growth_region_two_ended():
    """BMC_OPT_ARENA = 2 (two-ended growth region, bmc_region_reserve): a
    3-layer model (one stream) and a separate handle on its own stream share
    the region; caches, ledgers and outputs match the oracle; a region too
    small for the late growths falls back to the pool mid-run; the region
    cannot be replaced while buffers live in it, and is freed at the end."""
    import torch
    from harness import Model
    row = 4 * 128 * 2            # one row of all 4 units (B=2 x H_kv=2) of one tensor, bf16
    # ample (both ends hold every buffer), then ~0.7 MB: the later growths
    # no longer fit and come from the pool
    for size in (64 << 20, 6 * 120 * row):
        assert bmc.bmc_region_reserve(-1, size) == 0
        m = Model(3, 2, 2, 8, 128, 16, 200, seed=23, options=((bmc.BMC_OPT_ARENA, 2),))
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):          # the side handle lives on stream s
            side = Pair(2, 2, 2, 128, 8, 120, dtype="bf16", seed=21)
            side.gpu.set_option(bmc.BMC_OPT_ARENA, 2)
        for n in range(1, 201):
            m.decode_step(check=(n % 17 == 0 or n in (16, 17, 200)))
            if n <= 120:
                with torch.cuda.stream(s):
                    side.append()
                    if n % 11 == 0:
                        side.sdpa()
        m.check_state()
        with torch.cuda.stream(s):
            side.check_state()
        with pytest.raises(bmc.BMCError):
            bmc.bmc_region_reserve(-1, 1 << 20)     # live buffers
        m.close()
        side.close()
        torch.cuda.synchronize()
        assert bmc.bmc_region_reserve(-1, 0) == 0
        del s


def test_launch_count_increments():
    n0 = bmc.bmc_launch_count()
    p = Pair(1, 2, 2, 128, 4, 16, dtype="bf16")
    _decode(p, 16, check_every=4)
    assert bmc.bmc_launch_count() - n0 >= 16 + 4
    p.close()


@pytest.mark.parametrize("path", [2, 3, 4])
@pytest.mark.parametrize("H_kv,H_q,k,ctas", [(2, 2, 0, 0), (2, 8, 0, 0), (2, 16, 0, 0),
                                             (1, 8, 8, 0), (2, 16, 8, 5), (1, 16, 7, 0),
                                             (2, 2, 4, 7), (3, 3, 4, 11), (1, 8, 3, 0),
                                             (2, 8, 4, 9), (1, 16, 3, 6), (2, 4, 12, 0),
                                             (1, 8, 9, 4), (2, 6, 7, 0)])
def test_tcgen05_verify_path(path, H_kv, H_q, k, ctas):
    """The tensor-core kernels (BMC_OPT_ATTN_PATH=2: auto, 3: queries on the
    TMEM lanes, 4: keys on the lanes, M <= 80) against the oracle: M = G*(1+k_adm)
    from 1 to 128 query rows per KV head (M = 1, 4, 5, 8, 24, 32, 40, 52, 64,
    72, 80, 128), ragged caps (r=24 divides neither tile), split units."""
    if path == 4 and (H_q // H_kv) * (1 + k) > 80:
        pytest.skip("keys-on-lanes kernel covers G*t <= 80")
    p = Pair(2, H_kv, H_q, 128, 24, 300, dtype="bf16", seed=23, ctas=ctas)
    p.gpu.set_option(bmc.BMC_OPT_ATTN_PATH, path)
    for _ in range(3):
        p.append()
    p.sdpa()
    it = 0
    while p.orc.stats()["valid_max"] < 280:
        p.append()
        k_adm = p.spec_write(k) if k else 0
        p.sdpa(n_valid=-1)
        if k_adm:
            p.commit_rows(synth.acceptance(23, it, 2, k_adm))
        it += 1
    p.check_state()
    p.close()


@pytest.mark.parametrize("groups", [0, 2, 4])
@pytest.mark.parametrize("H_kv,H_q,k,ctas", [(2, 2, 4, 7), (2, 6, 7, 0), (1, 8, 3, 0),
                                             (2, 16, 4, 5), (1, 8, 7, 0), (1, 8, 8, 3),
                                             (1, 16, 4, 0)])
def test_tcgen05_softmax_groups(groups, H_kv, H_q, k, ctas):
    """Keys-on-lanes kernel with 2 or 4 softmax column groups (384 / 640
    threads; BMC_OPT_TCK_GROUPS) against the oracle for N = 16 ... 80 query
    columns (M = 5, 24, 32, 40, 64, 72, 80): 4 groups of N/4 columns exercise
    the 4-column TMEM loads and 8-byte P stores (N/4 = 4, 12, 20)."""
    p = Pair(2, H_kv, H_q, 128, 24, 300, dtype="bf16", seed=31, ctas=ctas)
    p.gpu.set_option(bmc.BMC_OPT_ATTN_PATH, 4)
    p.gpu.set_option(bmc.BMC_OPT_TCK_GROUPS, groups)
    for _ in range(3):
        p.append()
    p.sdpa()
    it = 0
    while p.orc.stats()["valid_max"] < 280:
        p.append()
        k_adm = p.spec_write(k) if k else 0
        p.sdpa(n_valid=-1)
        if k_adm:
            p.commit_rows(synth.acceptance(31, it, 2, k_adm))
        it += 1
    p.check_state()
    p.close()


@pytest.mark.parametrize("path", [3, 4])
def test_tcgen05_peaky_long(path):
    """Near one-hot rows through the tensor-core paths: P is split into
    bf16 hi + lo so its rounding stays far inside the 2e-3 budget."""
    p = Pair(2, 2, 16, 128, 64, 1500, dtype="bf16", seed=29, variant="peaky")
    p.gpu.set_option(bmc.BMC_OPT_ATTN_PATH, path)
    _decode(p, 1500, check_every=61)
    p.close()


@pytest.mark.parametrize("path,policy", [(1, "bmc"), (2, "bmc"), (1, "upfront")])
def test_length_aware_ablation(path, policy):
    """BMC_OPT_SKIP_PADDING (SURVEY NEXT-4 ablation): streaming only visible
    rows leaves every output and the cache unchanged."""
    p = Pair(2, 2, 8, 128, 40, 260, dtype="bf16", policy=policy, seed=31)
    p.gpu.set_option(bmc.BMC_OPT_SKIP_PADDING, 1)
    p.gpu.set_option(bmc.BMC_OPT_ATTN_PATH, path)
    for it in range(60):
        p.append()
        k = p.spec_write(3)
        p.sdpa(n_valid=-1)
        p.commit_rows(synth.acceptance(31, it, 2, k))
    p.check_state()
    p.close()


def _random_tree(rng, k):
    return [-1] + [int(rng.integers(-1, i)) for i in range(1, k)]


def _random_path(rng, parent, k_adm):
    """A root-to-node path among the admitted nodes (possibly empty)."""
    if k_adm == 0 or rng.random() < 0.15:
        return []
    node = int(rng.integers(0, k_adm))
    path = []
    while node >= 0:
        path.append(node)
        node = parent[node]
    return path[::-1][: int(rng.integers(1, len(path) + 1))]


@pytest.mark.parametrize("path,H_kv,H_q,k", [(1, 2, 2, 6), (2, 2, 2, 6), (2, 2, 8, 12),
                                             (1, 1, 4, 26), (2, 1, 4, 26), (3, 2, 8, 12),
                                             (3, 1, 4, 26), (4, 1, 8, 9)])
def test_token_tree_speculation(path, H_kv, H_q, k):
    """Token-tree speculation: nodes in BFS order in the padded
    rows, ancestor-rule mask in both attention kernels (CUDA cores: path 1,
    tcgen05: path 2), per-row accepted paths compacted on commit; every
    output row and the final cache against the oracle."""
    rng = np.random.default_rng(7 * k + path)
    p = Pair(3, H_kv, H_q, 128, 32, 600, dtype="bf16", seed=37 + k)
    p.gpu.set_option(bmc.BMC_OPT_ATTN_PATH, path)
    for _ in range(4):
        p.append()
    p.sdpa()
    it = 0
    while p.orc.stats()["valid_max"] < 560 and it < 45:
        p.append()
        parent = _random_tree(rng, k)
        k_adm = p.spec_write_tree(k, parent)
        p.sdpa(n_valid=-1)
        p.commit_path([_random_path(rng, parent, k_adm) for _ in range(3)])
        it += 1
        if it % 15 == 0:
            p.check_state()
    p.check_state()
    p.close()


def test_token_tree_paper_example_gpu():
    """The figure's 4-node tree on the GPU: 7 -> 3 -> 1 -> 0 wasted rows."""
    p = Pair(1, 1, 1, 128, 8, 64, dtype="bf16", seed=41)
    p.append()
    for wasted, pth in [(3, [0, 2]), (1, [0]), (0, [])]:
        assert p.spec_write_tree(4, [-1, 0, 0, 1]) == 4
        s = p.gpu.stats()
        assert s["capacity"] - s["valid_max"] - s["staged"] == wasted
        p.sdpa()
        p.commit_path([pth])
    p.check_state()
    p.close()


@pytest.mark.parametrize("policy,r,prompt", [("bmc", 16, 1), ("bmc", 16, 16), ("bmc", 16, 17),
                                             ("bmc", 24, 130), ("iterative", 1, 45),
                                             ("upfront", 300, 77)])
@pytest.mark.parametrize("host_io", [False, True])
def test_bulk_prefill_then_decode(policy, r, prompt, host_io):
    """bmc_append_n (prompt ingestion, one allocation: S:L104, reading R19)
    then decode and a second bulk append mid-stream: cache bytes, lengths and
    ledger bit-exact vs the oracle, every output within 2e-3."""
    p = Pair(2, 2, 8, 128, r, 300, dtype="bf16", policy=policy, seed=41, host_io=host_io)
    p.append_n(prompt)
    p.check_state()
    for _ in range(20):
        p.append()
        p.sdpa()
    p.append_n(33)
    p.sdpa()
    p.check_state()
    p.close()


def test_pinned_per_layer_loop_overlaps_correctly():
    """Two layers driven call by call with pinned host buffers, as the
    speculative bench loop does: every upload of layer l+1 may overlap layer
    l's kernel, every download the next layer's; all outputs and caches
    against the oracle."""
    ps = [Pair(2, 2, 4, 128, 16, 140, dtype="bf16", seed=50 + l, layer=l, host_io="pinned")
          for l in range(2)]
    for it in range(40):
        for p in ps:
            p.append()
            k = p.spec_write(3)
            p.sdpa(n_valid=-1)
            p.commit_rows(synth.acceptance(50, it, 2, k))
    for p in ps:
        p.check_state()
        p.close()
