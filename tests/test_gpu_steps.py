"""Oracle parity of the fused whole-model calls bench.py times
(bmc_decode_step, bmc_spec_step, bmc_commit_step): every layer of a full-depth
model against its own oracle, the ITERATIVE and UPFRONT baselines under
speculation, and the OOM fallback / rollback of the fused steps.

Tolerances as tests/harness.py (bf16 max-abs 2e-3); caches, lengths and the
ledger bit-exact / equal.
"""
import pytest
import torch

pytestmark = pytest.mark.gpu

from harness import Model  # noqa: E402
from paper_2511_12031_b200 import bmc, synth  # noqa: E402


@pytest.fixture(autouse=True, scope="module")
def _built():
    import __graft_entry__
    __graft_entry__.build()


@pytest.mark.parametrize("H_kv,H_q,r,N", [(32, 32, 64, 200), (8, 32, 48, 150)])
def test_full_depth_decode_step(H_kv, H_q, r, N):
    """BASELINE configs[1] / [3] head shapes at full depth (L = 32 layers in
    ONE fused launch per token, the bench's launch configuration) with a
    reduced batch and context: every layer's output at every checked step,
    then every layer's cache and ledger, against per-layer oracles.  Growths
    happen inside the fused launch (copy-on-read)."""
    m = Model(32, 2, H_kv, H_q, 128, r, N, seed=32)
    for n in range(1, N + 1):
        m.decode_step(check=(n % 23 == 0 or n in (1, r, r + 1, N)))
        if n in (r + 1, N):
            m.check_state()
    m.close()


def test_full_depth_spec_step_70b_heads():
    """70B-long head shape (64 q / 8 kv heads, k = 8 chain drafts: M = 72 at
    full admission) over 34 layers (two fused verify launches: 32 + 2) with
    per-row acceptance and bmc_commit_step; every layer against its oracle."""
    B, k = 2, 8
    m = Model(34, B, 8, 64, 128, 40, 160, seed=70)
    it = 0
    while m.orc[0].stats()["valid_max"] < 150:
        k_adm = m.spec_step(k, check=(it % 3 == 0))
        m.commit_step([min(x, k_adm) for x in synth.acceptance(3, it, B, k)])
        it += 1
        if it % 9 == 0:
            m.check_state(layers=(0, 31, 33))
    m.check_state()
    m.close()


def _bfs_tree(k, seed):
    import numpy as np
    rng = np.random.default_rng(seed)
    return [-1] + [int(rng.integers(-1, i)) for i in range(1, k)]


def _tree_path(parent, k_adm, salt):
    """A root-to-node path among the admitted nodes (empty every 5th call)."""
    if k_adm == 0 or salt % 5 == 4:
        return []
    node = (salt * 7 + 3) % k_adm
    path = []
    while node >= 0:
        path.append(node)
        node = parent[node]
    return path[::-1]


@pytest.mark.parametrize("L,B,H_kv,H_q,k,r", [(32, 2, 32, 32, 26, 40),   # E8 heads, full depth
                                              (3, 3, 2, 8, 9, 24),      # GQA, M = 40
                                              (34, 1, 1, 2, 26, 64),    # 32 + 2 layers
                                              (3, 2, 2, 2, 32, 48)])    # largest tree
def test_tree_step_fused(L, B, H_kv, H_q, k, r):
    _tree_run(L, B, H_kv, H_q, k, r, "bmc")


@pytest.mark.parametrize("policy", ["iterative", "upfront"])
def test_tree_step_fused_baselines(policy):
    """The fused token-tree step under the two baselines (ITERATIVE grows
    exactly for the appended row and again for the admitted tree, reading
    R17; UPFRONT never grows): outputs, caches and the whole ledger against
    per-layer oracles."""
    _tree_run(3, 2, 2, 8, 9, 1 if policy == "iterative" else 200, policy)


def _tree_run(L, B, H_kv, H_q, k, r, policy):
    """bmc_spec_step_tree + bmc_commit_path_step (the token-tree bench
    mode's calls: every layer's append and k-node tree, one verify launch per
    32 layers, one path-compaction launch per 32 layers) against per-layer
    oracles: every output row (ancestor mask), then caches,
    lengths and ledgers bit-exact; per-row accepted paths of different
    lengths; topologies change every iteration."""
    m = Model(L, B, H_kv, H_q, 128, r, 200, seed=26 + k, policy=policy)
    it = 0
    while m.orc[0].stats()["valid_max"] < 200 - k - 2:
        parent = _bfs_tree(k, 100 + it)
        k_adm = m.spec_step_tree(k, parent, check=(it % 2 == 0))
        m.commit_path_step([_tree_path(parent, k_adm, it + 3 * b) for b in range(B)])
        it += 1
        if it % 7 == 0:
            m.check_state(layers=(0, L - 1))
    m.check_state()
    m.close()


def test_tree_step_errors_leave_state():
    """Invalid topologies, k > 32 and paths that are not parent-linked fail
    before anything is enqueued (every layer unchanged)."""
    m = Model(3, 2, 2, 2, 128, 16, 64, seed=3)
    m.decode_step()
    before = [(g.stats(), g.valid()) for g in m.gpu]
    p = m.plan
    z = [torch.zeros(2, 2, 128, dtype=torch.bfloat16, device="cuda") for _ in range(3)]
    zd = [torch.zeros(2, 2, 33, 128, dtype=torch.bfloat16, device="cuda") for _ in range(3)]
    q = [torch.zeros(2, 2, 34, 128, dtype=torch.bfloat16, device="cuda") for _ in range(3)]
    o = [torch.empty(2, 2, 34, 128, device="cuda") for _ in range(3)]
    args = (p.ptrs(z), p.ptrs(z), p.ptrs(zd), p.ptrs(zd))
    with pytest.raises(bmc.BMCError):
        bmc.bmc_spec_step_tree(p, *args, 3, [-1, 1, 0], p.ptrs(q), p.ptrs(o))   # parent >= i
    with pytest.raises(bmc.BMCError):
        bmc.bmc_spec_step_tree(p, *args, 33, [-1] * 33, p.ptrs(q), p.ptrs(o))   # k > 32
    assert [(g.stats(), g.valid()) for g in m.gpu] == before
    k_adm = m.spec_step_tree(4, [-1, 0, 0, 1])
    assert k_adm == 4
    with pytest.raises(bmc.BMCError):
        bmc.bmc_commit_path_step(p, [[0, 2, 1], [0]])   # node 1 does not hang off node 2
    m.commit_path_step([[0, 1, 3], []])
    m.check_state()
    m.close()


@pytest.mark.parametrize("spec", [False, True])
def test_region_lifo_chunks(spec):
    """34 layers (two fused chunks: 32 + 2) in a two-ended growth region of
    only the final cache plus one 32-layer chunk: the fused steps move the
    chunks in LIFO order (the chunk whose old buffers are on top first), so
    every growth fits without the pool -- all buffers end inside one
    region-sized span -- and outputs, caches and ledgers match the oracle."""
    B, H_kv, L, N, r = 2, 4, 34, 96, 16
    per_layer = 2 * B * H_kv * N * 128 * 2
    size = (L + 32) * per_layer + (1 << 20)
    assert bmc.bmc_region_reserve(-1, size) == 0
    m = Model(L, B, H_kv, 8, 128, r, N, seed=34, options=((bmc.BMC_OPT_ARENA, 2),))
    it = 0
    while m.orc[0].stats()["valid_max"] < N - 6:
        if spec:
            k_adm = m.spec_step(4, check=(it % 4 == 0))
            m.commit_step(synth.acceptance(5, it, B, k_adm))
        else:
            m.decode_step(check=(it % 9 == 0))
        it += 1
    m.check_state()
    ptrs = []
    for g in m.gpu:
        k, v, cap = bmc.bmc_kv_view(g.h)
        ptrs += [k, v]
    assert max(ptrs) - min(ptrs) < size, "a growth fell back to the pool"
    m.close()
    torch.cuda.synchronize()
    assert bmc.bmc_region_reserve(-1, 0) == 0


@pytest.mark.parametrize("policy", ["iterative", "upfront"])
def test_region_baseline_policies(policy):
    """The two baselines in the growth region (handles created after
    bmc_region_reserve take every buffer from it): ITERATIVE moves every
    layer to the other end each step, UPFRONT holds its N_max buffers;
    outputs, caches and ledgers against the oracle."""
    assert bmc.bmc_region_reserve(-1, 32 << 20) == 0
    m = Model(3, 2, 2, 8, 128, 1 if policy == "iterative" else 90, 90, policy=policy, seed=12)
    for n in range(1, 91):
        m.decode_step(check=(n % 13 == 0 or n == 90))
    m.check_state()
    m.close()
    torch.cuda.synchronize()
    assert bmc.bmc_region_reserve(-1, 0) == 0


@pytest.mark.parametrize("policy", ["iterative", "upfront"])
@pytest.mark.parametrize("H_kv,H_q,k", [(2, 2, 4), (2, 16, 4), (1, 8, 8)])
def test_baselines_under_speculation(policy, H_kv, H_q, k):
    """The two baselines with speculative decoding (SURVEY 8(d) ITERATIVE-SD
    and UPFRONT-SD; reading R17: ITERATIVE reallocates exactly for the
    appended row and again for the drafts, copying the valid rows), through
    bmc_spec_step + bmc_commit_step with per-row acceptance: outputs, caches,
    capacities and the whole ledger (alloc_events, copied_bytes, ...) equal
    the oracle's after every iteration."""
    B, L, N = 3, 3, 90
    m = Model(L, B, H_kv, H_q, 128, 1, N, policy=policy, seed=17)
    it = 0
    while m.orc[0].stats()["valid_max"] < N - k - 2:
        k_adm = m.spec_step(k)
        m.check_state()
        m.commit_step(synth.acceptance(19, it, B, k_adm))
        m.check_state()
        it += 1
    m.close()


@pytest.mark.parametrize("policy", ["iterative", "upfront"])
def test_baselines_speculative_7b_fullsize(policy):
    """BASELINE configs[2] (7B shape, B = 32, k = 4 chain drafts, context to
    4096) for the two baselines through the fused bmc_spec_step: ledger
    against the oracle's closed-form behaviour (ITERATIVE: two exact
    reallocations per iteration; UPFRONT: none), sampled units of the layer
    against per-unit oracles at sampled iterations, cache bit-exact at the end."""
    import numpy as np
    import oracle as O
    from harness import TOL_BF16
    B, H, D, N, k = 32, 32, 128, 4096, 4
    dev = torch.device("cuda")
    c = bmc.KVCache(B, H, H, D, 1, N, dtype="bf16", policy=policy)
    plan = bmc.StepPlan([c])
    g = torch.Generator(device=dev)
    g.manual_seed(41)
    units = [(0, 0), (31, 31), (9, 20)]
    hist = {u: [] for u in units}
    rows_k = torch.zeros(B, H, N, D, dtype=torch.bfloat16, device=dev)
    rows_v = torch.zeros_like(rows_k)
    it, allocs = 0, c.stats()["alloc_events"]
    while max(c.valid()) < N - 1:
        kk = min(k, N - max(c.valid()) - 1)
        k_adm = bmc.bmc_admissible(c.h, kk)
        t = 1 + k_adm
        kn = torch.randn(B, H, D, generator=g, device=dev).to(torch.bfloat16)
        vn = torch.randn(B, H, D, generator=g, device=dev).to(torch.bfloat16)
        kd = torch.randn(B, H, max(kk, 1), D, generator=g, device=dev).to(torch.bfloat16)
        vd = torch.randn(B, H, max(kk, 1), D, generator=g, device=dev).to(torch.bfloat16)
        q = torch.randn(B, H, t, D, generator=g, device=dev).to(torch.bfloat16)
        o = torch.empty(B, H, t, D, device=dev)
        v0 = c.valid()
        got = bmc.bmc_spec_step(plan, plan.ptrs([kn]), plan.ptrs([vn]), plan.ptrs([kd]),
                                plan.ptrs([vd]), kk, plan.ptrs([q]), plan.ptrs([o]))
        assert got == k_adm
        if policy == "iterative":
            s = c.stats()
            assert s["alloc_events"] - allocs == (2 if k_adm else 1)
            assert s["capacity"] == max(v0) + 1 + k_adm
            allocs = s["alloc_events"]
        m = synth.acceptance(23, it, B, k_adm)
        for b in range(B):
            rows_k[b, :, v0[b]] = kn[b]
            rows_v[b, :, v0[b]] = vn[b]
            rows_k[b, :, v0[b] + 1:v0[b] + 1 + m[b]] = kd[b, :, :m[b]]
            rows_v[b, :, v0[b] + 1:v0[b] + 1 + m[b]] = vd[b, :, :m[b]]
        sample = it % 150 == 0 or max(c.valid()) > N - 10
        for (b, h) in units:
            hist[(b, h)].append((kn[b, h].cpu(), vn[b, h].cpu(), kd[b, h, :k_adm].cpu(),
                                 vd[b, h, :k_adm].cpu(), q[b, h].cpu() if sample else None,
                                 o[b, h].cpu().numpy() if sample else None, m[b]))
        if k_adm:
            bmc.bmc_commit_step(plan, m)
        it += 1
    worst, checks = 0.0, 0
    for (b, h), ops in hist.items():
        orc = O.Oracle(1, 1, 1, D, 1, N, dtype=O.BF16,
                       policy=O.POLICY_ITERATIVE if policy == "iterative" else O.POLICY_UPFRONT)
        for (kn_, vn_, kd_, vd_, q_, o_, mb) in ops:
            orc.append(kn_.reshape(1, 1, D), vn_.reshape(1, 1, D))
            ka = kd_.shape[0]
            if ka:
                assert orc.spec_write(kd_.reshape(1, 1, ka, D).contiguous(),
                                      vd_.reshape(1, 1, ka, D).contiguous(), ka) == ka
            if q_ is not None:
                ref = orc.sdpa(q_.reshape(1, 1, 1 + ka, D).contiguous(), -1)
                worst = max(worst, float(np.abs(o_.reshape(ref.shape) - ref).max()))
                checks += 1
            if ka:
                orc.commit(min(mb, ka))
        orc.close()
    assert checks > 20 and worst <= TOL_BF16, (checks, worst)
    torch.cuda.synchronize()
    Kc, Vc = c.kv()
    U = B * H
    vmax = max(c.valid())
    assert Kc.shape[1] >= vmax
    exp_k = rows_k.reshape(U, N, D)[:, :Kc.shape[1]]
    exp_v = rows_v.reshape(U, N, D)[:, :Kc.shape[1]]
    assert torch.equal(Kc.view(torch.int16), exp_k.view(torch.int16))
    assert torch.equal(Vc.view(torch.int16), exp_v.view(torch.int16))
    c.close()


@pytest.mark.parametrize("kind", ["decode", "spec"])
def test_fused_step_oom_fallback(kind):
    """when deferring layer l's copy-on-read growth runs out
    of memory (injected, BMC_OPT_FAULT_OOM), the deferred growths of the
    chunk's earlier layers are carried out by the realloc kernel and layer l
    grows without deferral; the launch then sees mixed layers and must still
    produce the oracle's outputs and caches (no stale old-buffer pointers)."""
    B, L, r = 2, 6, 16
    m = Model(L, B, 2, 8, 128, r, 120, seed=9)
    for n in range(1, r + 1):
        m.decode_step(check=False) if kind == "decode" else m.spec_step(0, check=False)
    m.check_state()
    m.gpu[3].set_option(bmc.BMC_OPT_FAULT_OOM, 1)      # the next growth of layer 3 fails once
    if kind == "decode":
        m.decode_step()                                 # grows every layer
    else:
        k_adm = m.spec_step(4)
        m.commit_step([2, 1])
        assert k_adm == 4
    m.check_state()
    for _ in range(3):
        m.decode_step() if kind == "decode" else m.spec_step(0)
    m.check_state()
    m.close()


@pytest.mark.parametrize("kind", ["decode", "spec"])
def test_fused_step_oom_rollback(kind):
    """an OOM that the fallback cannot absorb (layer 3's
    growth fails twice) returns BMC_ERR_OOM with every layer of the chunk
    rolled back to its lengths before the call; the retried step then gives
    the oracle's outputs, caches and ledger totals."""
    B, L, r = 2, 5, 16
    m = Model(L, B, 2, 8, 128, r, 120, seed=11)
    for n in range(1, r + 1):
        m.decode_step(check=False)
    m.check_state()
    before = [c.valid() for c in m.gpu]
    m.gpu[3].set_option(bmc.BMC_OPT_FAULT_OOM, 2)
    xs = [synth.step_inputs(1234, l, 0, B=B, H_kv=2, H_q=8, D=128, t=5, k_draft=4)
          for l in range(L)]
    dev = [{k: v.cuda() for k, v in x.items()} for x in xs]
    p = m.plan
    with pytest.raises(bmc.BMCError) as ei:
        if kind == "decode":
            outs = [torch.empty(B, 8, 1, 128, device="cuda") for _ in range(L)]
            bmc.bmc_decode_step(p, p.ptrs([d["k"] for d in dev]), p.ptrs([d["v"] for d in dev]),
                                p.ptrs([d["q"][:, :, :1].contiguous() for d in dev]),
                                p.ptrs(outs), r + 1)
        else:
            outs = [torch.empty(B, 8, 5, 128, device="cuda") for _ in range(L)]
            bmc.bmc_spec_step(p, p.ptrs([d["k"] for d in dev]), p.ptrs([d["v"] for d in dev]),
                              p.ptrs([d["kd"] for d in dev]), p.ptrs([d["vd"] for d in dev]), 4,
                              p.ptrs([d["q"] for d in dev]), p.ptrs(outs))
    assert ei.value.code == bmc.BMC_ERR_OOM
    assert [c.valid() for c in m.gpu] == before
    assert all(c.stats()["staged"] == 0 for c in m.gpu)
    # the retried step (fresh inputs through the harness) matches the oracle
    if kind == "decode":
        m.decode_step()
    else:
        k_adm = m.spec_step(4)
        m.commit_step([1, 3])
        assert k_adm == 4
    m.check_state()
    m.decode_step()
    m.check_state()
    m.close()
