"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (bmc_decode_step: all layers of a step in one persistent launch).

Inputs are seeded N(0,1) draws (torch generator on the device for speed,
RNE-rounded to bf16); the oracle receives the same rounded bits of the
sampled units.  Checked: SDPA outputs of sampled (batch, kv-head) units at
sampled steps against per-unit oracles (element by element, max-abs 2e-3),
the whole cache against the appended rows (bit-exact, zero padding), and the
allocation / copy ledger against the paper's closed forms.
"""
import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import oracle as O  # noqa: E402
from harness import TOL_BF16  # noqa: E402
from paper_2511_12031_b200 import bmc, synth  # noqa: E402


@pytest.fixture(autouse=True, scope="module")
def _built():
    import __graft_entry__
    __graft_entry__.build()


def _bits(x: torch.Tensor) -> torch.Tensor:
    return x.view(torch.int16)


def _run_decode_fullsize(B, H_kv, H_q, D, N, r, L, sample_steps, sample_units, seed):
    dev = torch.device("cuda")
    caches = [bmc.KVCache(B, H_kv, H_q, D, r, N, dtype="bf16") for _ in range(L)]
    plan = bmc.StepPlan(caches)
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    U = B * H_kv
    G = H_q // H_kv
    Kall = [torch.empty(N, B, H_kv, D, dtype=torch.bfloat16, device=dev) for _ in range(L)]
    Vall = [torch.empty_like(Kall[0]) for _ in range(L)]
    outs = [torch.empty(B, H_q, 1, D, device=dev) for _ in range(L)]
    Optr = plan.ptrs(outs)
    saved = {}
    for n in range(1, N + 1):
        ks, vs, qs = [], [], []
        for l in range(L):
            Kall[l][n - 1] = torch.randn(B, H_kv, D, generator=g, device=dev).to(torch.bfloat16)
            Vall[l][n - 1] = torch.randn(B, H_kv, D, generator=g, device=dev).to(torch.bfloat16)
            qs.append(torch.randn(B, H_q, 1, D, generator=g, device=dev).to(torch.bfloat16))
            ks.append(Kall[l][n - 1])
            vs.append(Vall[l][n - 1])
        bmc.bmc_decode_step(plan, plan.ptrs(ks), plan.ptrs(vs), plan.ptrs(qs), Optr, n)
        if n in sample_steps:
            for l in range(L):
                saved[(n, l)] = (qs[l].clone(), outs[l].clone())
    torch.cuda.synchronize()
    return caches, Kall, Vall, saved


@pytest.mark.parametrize("cfg", [
    # BASELINE configs[1]: Llama-2-7B shape, B=16, context 4096, r = 128 (bench default)
    dict(B=16, H_kv=32, H_q=32, D=128, N=4096, r=128, L=2),
    # BASELINE configs[3] per GPU: Llama-3-8B GQA (32 q / 8 kv heads), B=64, context 8192
    # (two layers: the fused multi-layer tcgen05 launch of the GQA decode step)
    dict(B=64, H_kv=8, H_q=32, D=128, N=8192, r=128, L=2),
])
def test_fullsize_decode(cfg):
    B, H_kv, H_q, D, N, r, L = (cfg[k] for k in ("B", "H_kv", "H_q", "D", "N", "r", "L"))
    steps = sorted({1, r - 1, r, r + 1, 1000, N // 2, N - 1, N})
    units = [(0, 0), (B - 1, H_kv - 1), (B // 2, H_kv // 3), (3 % B, (5 * H_kv) // 7)]
    caches, Kall, Vall, saved = _run_decode_fullsize(B, H_kv, H_q, D, N, r, L, set(steps),
                                                     units, seed=2511)
    G = H_q // H_kv
    U = B * H_kv
    # 1) cache contents: committed rows == appended rows (bit-exact), no padding at N
    for l in range(L):
        Kc, Vc = caches[l].kv()
        assert Kc.shape == (U, N, D)
        expK = Kall[l].permute(1, 2, 0, 3).reshape(U, N, D)
        expV = Vall[l].permute(1, 2, 0, 3).reshape(U, N, D)
        assert torch.equal(_bits(Kc), _bits(expK)) and torch.equal(_bits(Vc), _bits(expV))
    # 2) ledger against the closed forms (P:L609-611 T = N/r, one copy per growth)
    s = caches[0].stats()
    T = math.ceil(N / r)
    assert s["alloc_events"] == T and s["copy_events"] == T - 1
    assert s["copied_bytes"] == 2 * U * D * 2 * r * (T - 1) * T // 2
    assert s["macs"] == sum(2 * B * H_q * min(r * math.ceil(n / r), N) * D
                            for n in range(1, N + 1))
    # 3) SDPA outputs of sampled units vs per-unit oracles
    worst = 0.0
    for l in range(L):
        Kl = Kall[l].cpu()
        Vl = Vall[l].cpu()
        for (b, g) in units:
            orc = O.Oracle(1, 1, G, D, r, N, dtype=O.BF16, policy=O.POLICY_BMC)
            for n in range(1, N + 1):
                orc.append(Kl[n - 1, b, g].reshape(1, 1, D).contiguous(),
                           Vl[n - 1, b, g].reshape(1, 1, D).contiguous())
                if n in saved and (n, l) in saved:
                    q, o = saved[(n, l)]
                    qu = q[b, g * G:(g + 1) * G].cpu().reshape(1, G, 1, D).contiguous()
                    ref = orc.sdpa(qu, n)
                    got = o[b, g * G:(g + 1) * G].cpu().numpy().reshape(ref.shape)
                    worst = max(worst, float(np.abs(got - ref).max()))
            orc.close()
    assert worst <= TOL_BF16, worst
    for c in caches:
        c.close()


def test_fullsize_speculative_7b():
    """BASELINE configs[2]: 7B shape, B=32, k=4 chain drafts in the padded
    rows, per-row acceptance (Bernoulli 0.7 leading successes), one layer to
    N=4096; sampled units checked against per-unit oracles replaying the same
    row sequence."""
    B, H, D, N, r, k = 32, 32, 128, 4096, 64, 4
    dev = torch.device("cuda")
    c = bmc.KVCache(B, H, H, D, r, N, dtype="bf16")
    g = torch.Generator(device=dev)
    g.manual_seed(7)
    units = [(0, 0), (31, 31), (17, 5)]
    hist = {u: [] for u in units}          # per unit: list of ("app"|"spec"|"sdpa"|"commit", data)
    it = 0
    worst = 0.0
    checks = 0
    while max(c.valid()) < N - 1:
        kn = torch.randn(B, H, D, generator=g, device=dev).to(torch.bfloat16)
        vn = torch.randn(B, H, D, generator=g, device=dev).to(torch.bfloat16)
        c.append(kn, vn)
        kk = min(k, N - max(c.valid()))
        kd = torch.randn(B, H, max(kk, 1), D, generator=g, device=dev).to(torch.bfloat16)
        vd = torch.randn(B, H, max(kk, 1), D, generator=g, device=dev).to(torch.bfloat16)
        k_adm = c.spec_write(kd, vd, kk) if kk > 0 else 0
        t = 1 + k_adm
        q = torch.randn(B, H, t, D, generator=g, device=dev).to(torch.bfloat16)
        o = c.sdpa(q, -1)
        m = synth.acceptance(11, it, B, k_adm)
        sample = it % 97 == 0 or max(c.valid()) > N - 12
        for (b, h) in units:
            hist[(b, h)].append((kn[b, h].cpu(), vn[b, h].cpu(), kd[b, h, :k_adm].cpu(),
                                 vd[b, h, :k_adm].cpu(), q[b, h].cpu() if sample else None,
                                 o[b, h].cpu().numpy() if sample else None, m[b]))
        c.commit_rows(m)
        it += 1
    for (b, h), ops in hist.items():
        # One unit alone cannot reproduce the batch's shared growth schedule
        # (admission uses max_b valid_b), so it is replayed with the GPU's
        # admitted counts in an UPFRONT oracle: SDPA is independent of the
        # padding (mask invariance, tests/test_oracle_pins.py).
        orc = O.Oracle(1, 1, 1, D, r, N, dtype=O.BF16, policy=O.POLICY_UPFRONT)
        for (kn, vn, kd, vd, q, o, mb) in ops:
            orc.append(kn.reshape(1, 1, D), vn.reshape(1, 1, D))
            ka = kd.shape[0]
            if ka:
                assert orc.spec_write(kd.reshape(1, 1, ka, D).contiguous(),
                                      vd.reshape(1, 1, ka, D).contiguous(), ka) == ka
            if q is not None:
                ref = orc.sdpa(q.reshape(1, 1, 1 + ka, D).contiguous(), -1)
                worst = max(worst, float(np.abs(o.reshape(ref.shape) - ref).max()))
                checks += 1
            if ka:
                orc.commit(min(mb, ka))
        orc.close()
    assert checks > 10 and worst <= TOL_BF16, (checks, worst)
    s = c.stats()
    assert s["alloc_events"] == math.ceil(s["valid_max"] / r) or s["capacity"] == N
    c.close()


def test_fullsize_speculative_70b_long():
    """BASELINE configs[4] (70B-long shape: B=8, 64 q / 8 kv heads, k=8 chain
    drafts, r=256, context to 32768) through the fused bmc_spec_step the bench
    times (keys-on-lanes tcgen05 verify, M = 8*(1+k_adm) up to 72, copy-on-read
    growth) and bmc_commit_step, two layers; sampled (batch row, kv head)
    units of layer 1 replayed in per-unit oracles (UPFRONT, with the GPU's
    admitted counts: mask invariance makes the padding irrelevant)."""
    B, Hk, Hq, D, N, r, k, L = 8, 8, 64, 128, 32768, 256, 8, 2
    G = Hq // Hk
    dev = torch.device("cuda")
    cs = [bmc.KVCache(B, Hk, Hq, D, r, N, dtype="bf16") for _ in range(L)]
    plan = bmc.StepPlan(cs)
    g = torch.Generator(device=dev)
    g.manual_seed(70)
    units = [(0, 0), (7, 7), (3, 5)]
    hist = {u: [] for u in units}
    it = 0
    while max(cs[0].valid()) < N - 1:
        kk = min(k, N - max(cs[0].valid()) - 1)
        k_adm = bmc.bmc_admissible(cs[0].h, kk)
        t = 1 + k_adm
        kn = [torch.randn(B, Hk, D, generator=g, device=dev).to(torch.bfloat16) for _ in range(L)]
        vn = [torch.randn(B, Hk, D, generator=g, device=dev).to(torch.bfloat16) for _ in range(L)]
        # drafts [B][H_kv][kk][D]: the library reads the k it is given
        kd = [torch.randn(B, Hk, max(kk, 1), D, generator=g, device=dev).to(torch.bfloat16)
              for _ in range(L)]
        vd = [torch.randn(B, Hk, max(kk, 1), D, generator=g, device=dev).to(torch.bfloat16)
              for _ in range(L)]
        q = [torch.randn(B, Hq, t, D, generator=g, device=dev).to(torch.bfloat16)
             for _ in range(L)]
        o = [torch.empty(B, Hq, t, D, device=dev) for _ in range(L)]
        got = bmc.bmc_spec_step(plan, plan.ptrs(kn), plan.ptrs(vn), plan.ptrs(kd), plan.ptrs(vd),
                                kk, plan.ptrs(q), plan.ptrs(o))
        assert got == k_adm
        m = [min(x, k_adm) for x in synth.acceptance(13, it, B, k)]
        sample = it % 700 == 0 or max(cs[0].valid()) > N - 20
        for (b, h) in units:
            hist[(b, h)].append((kn[1][b, h].cpu(), vn[1][b, h].cpu(), kd[1][b, h, :k_adm].cpu(),
                                 vd[1][b, h, :k_adm].cpu(),
                                 q[1][b, h * G:(h + 1) * G].cpu() if sample else None,
                                 o[1][b, h * G:(h + 1) * G].cpu().numpy() if sample else None,
                                 m[b]))
        if k_adm:
            bmc.bmc_commit_step(plan, m)
        it += 1
    worst, checks = 0.0, 0
    for (b, h), ops in hist.items():
        orc = O.Oracle(1, 1, G, D, r, N, dtype=O.BF16, policy=O.POLICY_UPFRONT)
        for (kn_, vn_, kd_, vd_, q_, o_, mb) in ops:
            orc.append(kn_.reshape(1, 1, D), vn_.reshape(1, 1, D))
            ka = kd_.shape[0]
            if ka:
                assert orc.spec_write(kd_.reshape(1, 1, ka, D).contiguous(),
                                      vd_.reshape(1, 1, ka, D).contiguous(), ka) == ka
            if q_ is not None:
                ref = orc.sdpa(q_.reshape(1, G, 1 + ka, D).contiguous(), -1)
                worst = max(worst, float(np.abs(o_.reshape(ref.shape) - ref).max()))
                checks += 1
            if ka:
                orc.commit(min(mb, ka))
        orc.close()
    assert checks > 20 and worst <= TOL_BF16, (checks, worst)
    for c in cs:
        s = c.stats()
        assert s["alloc_events"] == math.ceil(s["valid_max"] / r) or s["capacity"] == N
        c.close()


@pytest.mark.parametrize("H_q,path_b", [(4, 1), (8, 0)])
def test_decode_step_matches_per_layer_calls(H_q, path_b):
    """bmc_decode_step (fused multi-layer launch, >32 layers -> 2 launches)
    matches per-layer append + sdpa calls: caches and ledgers bit-identical,
    outputs equal up to the split-K summation order (the CTA partition of the
    tile stream differs).  G = 2: CUDA-core step kernel; G = 4: the
    keys-on-lanes tcgen05 kernel, fused over layers, vs its per-layer launches."""
    B, H_kv, D, N, r, L = 2, 2, 128, 200, 24, 40
    dev = torch.device("cuda")
    a = [bmc.KVCache(B, H_kv, H_q, D, r, N, dtype="bf16") for _ in range(L)]
    b = [bmc.KVCache(B, H_kv, H_q, D, r, N, dtype="bf16") for _ in range(L)]
    for x in a + b:  # same algorithm on both sides
        x.set_option(bmc.BMC_OPT_ATTN_PATH, path_b)
    plan = bmc.StepPlan(a)
    g = torch.Generator(device=dev)
    g.manual_seed(3)
    oa = [torch.empty(B, H_q, 1, D, device=dev) for _ in range(L)]
    ob = [torch.empty(B, H_q, 1, D, device=dev) for _ in range(L)]
    for n in range(1, N + 1):
        ks = [torch.randn(B, H_kv, D, generator=g, device=dev).to(torch.bfloat16) for _ in range(L)]
        vs = [torch.randn(B, H_kv, D, generator=g, device=dev).to(torch.bfloat16) for _ in range(L)]
        qs = [torch.randn(B, H_q, 1, D, generator=g, device=dev).to(torch.bfloat16)
              for _ in range(L)]
        bmc.bmc_decode_step(plan, plan.ptrs(ks), plan.ptrs(vs), plan.ptrs(qs), plan.ptrs(oa), n)
        for l in range(L):
            b[l].append(ks[l], vs[l])
            b[l].sdpa(qs[l], n, ob[l])
        torch.cuda.synchronize()   # keep ks/vs alive until consumed
        if n % 37 == 0 or n == N:
            for l in range(L):
                torch.testing.assert_close(oa[l], ob[l], rtol=0, atol=1e-5)
    for l in range(L):
        ka, va = a[l].kv()
        kb, vb = b[l].kv()
        assert torch.equal(_bits(ka), _bits(kb)) and torch.equal(_bits(va), _bits(vb))
        assert a[l].stats() == b[l].stats()
    for x in a + b:
        x.close()


@pytest.mark.parametrize("dtype,D,r,B,N,H_q,path", [("bf16", 128, 24, 3, 170, 2, 1),
                                                    ("bf16", 128, 64, 2, 200, 2, 1),
                                                    ("f32", 64, 5, 2, 60, 2, 0),
                                                    ("bf16", 64, 1, 1, 40, 2, 0),
                                                    ("f32", 128, 37, 2, 120, 2, 0),
                                                    ("bf16", 128, 24, 3, 170, 2, 0),
                                                    ("bf16", 128, 24, 3, 300, 8, 0),
                                                    ("bf16", 128, 128, 2, 300, 16, 0),
                                                    ("bf16", 128, 1, 2, 40, 16, 0)])
def test_copy_on_read_growth(dtype, D, r, B, N, H_q, path):
    """a BMC growth inside bmc_decode_step is copied by the
    attention kernel while it streams the old buffer (old rows + zero page ->
    new buffer, appended row patched in).  Against the separate realloc
    kernel (BMC_OPT_COPY_ON_READ = 0): outputs identical at every step
    (same kernel, same partition), caches bit-identical right after every
    growth (copied rows, zero rows, appended row), ledgers equal.  r not a
    multiple of the tile's rows makes tiles straddle the old / new boundary;
    r = 1 grows every step.  CUDA-core kernel (path 1 or fp32 / D = 64: bulk
    copies, zero page); keys-on-lanes tcgen05 kernel (auto for bf16, D = 128:
    3D tensor maps, out-of-bounds zero fill, patched tile, tensor-map store)."""
    H_kv, L = 2, 3
    dev = torch.device("cuda")
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    a = [bmc.KVCache(B, H_kv, H_q, D, r, N, dtype=dtype) for _ in range(L)]
    b = [bmc.KVCache(B, H_kv, H_q, D, r, N, dtype=dtype) for _ in range(L)]
    for x in b:
        x.set_option(bmc.BMC_OPT_COPY_ON_READ, 0)
    for x in a + b:
        x.set_option(bmc.BMC_OPT_ATTN_PATH, path)
    pa, pb = bmc.StepPlan(a), bmc.StepPlan(b)
    g = torch.Generator(device=dev)
    g.manual_seed(17)
    oa = [torch.empty(B, H_q, 1, D, device=dev) for _ in range(L)]
    ob = [torch.empty(B, H_q, 1, D, device=dev) for _ in range(L)]
    l0 = bmc.bmc_launch_count()
    for n in range(1, N + 1):
        ks = [torch.randn(B, H_kv, D, generator=g, device=dev).to(tdt) for _ in range(L)]
        vs = [torch.randn(B, H_kv, D, generator=g, device=dev).to(tdt) for _ in range(L)]
        qs = [torch.randn(B, H_q, 1, D, generator=g, device=dev).to(tdt) for _ in range(L)]
        bmc.bmc_decode_step(pa, pa.ptrs(ks), pa.ptrs(vs), pa.ptrs(qs), pa.ptrs(oa), n)
        bmc.bmc_decode_step(pb, pb.ptrs(ks), pb.ptrs(vs), pb.ptrs(qs), pb.ptrs(ob), n)
        torch.cuda.synchronize()
        for l in range(L):
            assert torch.equal(oa[l], ob[l]), (n, l)
        if (n - 1) % r == 0 or n == N:        # growth steps (and the end)
            for l in range(L):
                ka, va = a[l].kv()
                kb, vb = b[l].kv()
                assert torch.equal(_bits(ka), _bits(kb)) and torch.equal(_bits(va), _bits(vb)), n
    for l in range(L):
        assert a[l].stats() == b[l].stats()
    grows = a[0].stats()["copy_events"]
    for x in a + b:
        x.close()
    assert grows == math.ceil(N / r) - 1


@pytest.mark.parametrize("contiguous", [False, True])
def test_spec_step_host_io_pipeline(contiguous):
    """bmc_spec_step with pinned host K/V/drafts/Q/O (staged on the library's
    copy stream, outputs downloaded on its download stream; one copy per
    tensor when the layers' buffers are contiguous) equals the device-pointer
    step: outputs bit-identical, caches bit-identical."""
    B, H_kv, H_q, D, N, r, L, k = 2, 2, 8, 128, 120, 16, 3, 4
    dev = torch.device("cuda")
    a = [bmc.KVCache(B, H_kv, H_q, D, r, N, dtype="bf16") for _ in range(L)]
    b = [bmc.KVCache(B, H_kv, H_q, D, r, N, dtype="bf16") for _ in range(L)]
    pa, pb = bmc.StepPlan(a), bmc.StepPlan(b)
    g = torch.Generator().manual_seed(5)
    it = 0
    while max(a[0].valid()) < N - 1 - k:
        kad = bmc.bmc_admissible(a[0].h, k)
        t = 1 + kad
        if contiguous:
            mk = lambda *shape: list(torch.randn(L, *shape, generator=g).to(torch.bfloat16)
                                     .pin_memory().unbind(0))
        else:
            mk = lambda *shape: [torch.randn(*shape, generator=g).to(torch.bfloat16).pin_memory()
                                 for _ in range(L)]
        ks, vs, kd, vd = mk(B, H_kv, D), mk(B, H_kv, D), mk(B, H_kv, k, D), mk(B, H_kv, k, D)
        qs = mk(B, H_q, t, D)
        oa = (list(torch.empty(L, B, H_q, t, D).pin_memory().unbind(0)) if contiguous
              else [torch.empty(B, H_q, t, D).pin_memory() for _ in range(L)])
        ob = [torch.empty(B, H_q, t, D, device=dev) for _ in range(L)]
        got = bmc.bmc_spec_step(pa, pa.ptrs(ks), pa.ptrs(vs), pa.ptrs(kd), pa.ptrs(vd), k,
                                pa.ptrs(qs), pa.ptrs(oa))
        assert got == kad
        dv = lambda xs: [x.to(dev) for x in xs]
        kk, vv, kdd, vdd, qq = dv(ks), dv(vs), dv(kd), dv(vd), dv(qs)
        assert bmc.bmc_spec_step(pb, pb.ptrs(kk), pb.ptrs(vv), pb.ptrs(kdd), pb.ptrs(vdd), k,
                                 pb.ptrs(qq), pb.ptrs(ob)) == kad
        a[0].sync()
        torch.cuda.synchronize()
        for l in range(L):
            assert torch.equal(oa[l], ob[l].cpu()), (it, l)
        acc = [int((it * 5 + 2 * bb) % (kad + 1)) for bb in range(B)]
        if kad:
            bmc.bmc_commit_step(pa, acc)
            bmc.bmc_commit_step(pb, acc)
        it += 1
    for x, y in zip(a, b):
        kx, vx = x.kv()
        ky, vy = y.kv()
        assert torch.equal(_bits(kx), _bits(ky)) and torch.equal(_bits(vx), _bits(vy))
        assert x.stats() == y.stats()
    for x in a + b:
        x.close()


def test_decode_step_host_io_pipeline():
    """bmc_decode_step with pinned host K/V/Q/O (the pipelined end-to-end path:
    copy stream, double-buffered staging) equals the device-pointer step."""
    B, H_kv, H_q, D, N, r, L = 3, 2, 2, 128, 150, 16, 4
    dev = torch.device("cuda")
    a = [bmc.KVCache(B, H_kv, H_q, D, r, N, dtype="bf16") for _ in range(L)]
    b = [bmc.KVCache(B, H_kv, H_q, D, r, N, dtype="bf16") for _ in range(L)]
    pa, pb = bmc.StepPlan(a), bmc.StepPlan(b)
    g = torch.Generator().manual_seed(9)
    oa = [torch.empty(B, H_q, 1, D).pin_memory() for _ in range(L)]
    ob = [torch.empty(B, H_q, 1, D, device=dev) for _ in range(L)]
    for n in range(1, N + 1):
        ks = [torch.randn(B, H_kv, D, generator=g).to(torch.bfloat16).pin_memory() for _ in range(L)]
        vs = [torch.randn(B, H_kv, D, generator=g).to(torch.bfloat16).pin_memory() for _ in range(L)]
        qs = [torch.randn(B, H_q, 1, D, generator=g).to(torch.bfloat16).pin_memory()
              for _ in range(L)]
        bmc.bmc_decode_step(pa, pa.ptrs(ks), pa.ptrs(vs), pa.ptrs(qs), pa.ptrs(oa), n)
        kd = [x.to(dev) for x in ks]
        vd = [x.to(dev) for x in vs]
        qd = [x.to(dev) for x in qs]
        bmc.bmc_decode_step(pb, pb.ptrs(kd), pb.ptrs(vd), pb.ptrs(qd), pb.ptrs(ob), n)
        a[0].sync()                      # host outputs readable; inputs reusable
        torch.cuda.synchronize()
        for l in range(L):
            assert torch.equal(oa[l], ob[l].cpu()), (n, l)
    for x, y in zip(a, b):
        kx, vx = x.kv()
        ky, vy = y.kv()
        assert torch.equal(_bits(kx), _bits(ky)) and torch.equal(_bits(vx), _bits(vy))
    for x in a + b:
        x.close()


@pytest.mark.parametrize("H_kv,H_q,k,L", [(2, 2, 1, 3), (2, 2, 4, 3), (2, 8, 3, 3),
                                          (1, 8, 8, 3), (2, 4, 4, 34), (1, 16, 8, 2)])
def test_spec_step_matches_per_layer_calls(H_kv, H_q, k, L):
    """bmc_spec_step (append + spec_write of every layer, then one verify
    launch per 32 layers: CUDA cores for M <= 2, keys-on-lanes tcgen05 up to
    M = 80, per-layer launches above) matches per-layer append / spec_write /
    sdpa calls: admissions, caches and ledgers identical, outputs equal up to
    the split-K summation order; per-row commits in between (bmc_commit_step
    against per-layer bmc_commit_rows)."""
    B, D, N, r = 2, 128, 160, 24
    dev = torch.device("cuda")
    a = [bmc.KVCache(B, H_kv, H_q, D, r, N, dtype="bf16") for _ in range(L)]
    b = [bmc.KVCache(B, H_kv, H_q, D, r, N, dtype="bf16") for _ in range(L)]
    plan = bmc.StepPlan(a)
    g = torch.Generator(device=dev)
    g.manual_seed(11)
    it = 0
    while max(a[0].valid()) < N - 1 - k:
        kad = bmc.bmc_admissible(a[0].h, k)
        t = 1 + kad
        ks = [torch.randn(B, H_kv, D, generator=g, device=dev).to(torch.bfloat16) for _ in range(L)]
        vs = [torch.randn(B, H_kv, D, generator=g, device=dev).to(torch.bfloat16) for _ in range(L)]
        kd = [torch.randn(B, H_kv, k, D, generator=g, device=dev).to(torch.bfloat16)
              for _ in range(L)]
        vd = [torch.randn(B, H_kv, k, D, generator=g, device=dev).to(torch.bfloat16)
              for _ in range(L)]
        qs = [torch.randn(B, H_q, t, D, generator=g, device=dev).to(torch.bfloat16)
              for _ in range(L)]
        oa = [torch.empty(B, H_q, t, D, device=dev) for _ in range(L)]
        got = bmc.bmc_spec_step(plan, plan.ptrs(ks), plan.ptrs(vs), plan.ptrs(kd), plan.ptrs(vd),
                                k, plan.ptrs(qs), plan.ptrs(oa))
        assert got == kad
        ob = []
        for l in range(L):
            b[l].append(ks[l], vs[l])
            assert b[l].spec_write(kd[l], vd[l], k) == kad
            ob.append(b[l].sdpa(qs[l], -1))
        torch.cuda.synchronize()
        for l in range(L):
            torch.testing.assert_close(oa[l], ob[l], rtol=0, atol=2e-5)
        acc = [int((it * 7 + 3 * bb) % (kad + 1)) for bb in range(B)]
        if kad:   # bmc_commit_step: one zero-fill launch per 32 layers; errors before any work
            with pytest.raises(bmc.BMCError):
                bmc.bmc_commit_step(plan, [kad + 1] * B)
            bmc.bmc_commit_step(plan, acc)
        for l in range(L):
            if not kad:
                a[l].commit_rows(acc)
            b[l].commit_rows(acc)
        it += 1
    for l in range(L):
        ka, va = a[l].kv()
        kb, vb = b[l].kv()
        assert torch.equal(_bits(ka), _bits(kb)) and torch.equal(_bits(va), _bits(vb))
        assert a[l].stats() == b[l].stats()
    for x in a + b:
        x.close()
