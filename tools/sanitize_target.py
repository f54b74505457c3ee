"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck):
the toy config through every kernel: growth copies, fused appends, the CUDA-
core attention (single layer and multi-layer step), SD with rollback, both
tcgen05 kernels (keys on the TMEM lanes incl. N=80, a token tree and the fused
GQA decode step; queries on the lanes), the bulk append; outputs checked
against the oracle."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

from harness import Pair  # noqa: E402
from paper_2511_12031_b200 import bmc, synth  # noqa: E402

# toy config (BASELINE configs[0]), fp32, CUDA cores
p = Pair(1, 2, 2, 64, 16, 128, dtype="f32")
for _ in range(40):
    p.append()
    p.sdpa()
p.check_state()
p.close()
# SD with per-row commits, bf16, tensor cores (M = 4 * (1 + 3))
p = Pair(2, 1, 4, 128, 16, 96, dtype="bf16", seed=3, ctas=3)
p.gpu.set_option(bmc.BMC_OPT_ATTN_PATH, 2)
for it in range(12):
    p.append()
    k = p.spec_write(3)
    p.sdpa(n_valid=-1)
    p.commit_rows(synth.acceptance(3, it, 2, k))
p.check_state()
p.close()
# the queries-on-lanes tcgen05 kernel, split units
p = Pair(2, 1, 4, 128, 16, 96, dtype="bf16", seed=4, ctas=5)
p.gpu.set_option(bmc.BMC_OPT_ATTN_PATH, 3)
for it in range(8):
    p.append()
    k = p.spec_write(3)
    p.sdpa(n_valid=-1)
    p.commit_rows(synth.acceptance(4, it, 2, k))
p.check_state()
p.close()
# keys on the lanes at N = 80 (M = 8 * 9), bulk prompt first
p = Pair(1, 1, 8, 128, 32, 200, dtype="bf16", seed=5, ctas=3)
p.gpu.set_option(bmc.BMC_OPT_ATTN_PATH, 4)
p.append_n(70)
for it in range(6):
    p.append()
    k = p.spec_write(8)
    p.sdpa(n_valid=-1)
    p.commit_rows(synth.acceptance(5, it, 1, k))
p.check_state()
p.close()
# token tree through the keys-on-lanes kernel
p = Pair(2, 1, 4, 128, 32, 160, dtype="bf16", seed=6)
p.gpu.set_option(bmc.BMC_OPT_ATTN_PATH, 2)
for _ in range(3):
    p.append()
for it in range(5):
    p.append()
    k = p.spec_write_tree(6, [-1, 0, 0, 1, 1, 2])
    p.sdpa(n_valid=-1)
    p.commit_path([[0, 1, 3][: it % 4], [0, 2][: (it + 1) % 3]])
p.check_state()
p.close()
# fused GQA decode step (G = 4, keys-on-lanes kernel over 3 layers)
caches = [bmc.KVCache(2, 2, 8, 128, 16, 64, dtype="bf16") for _ in range(3)]
plan = bmc.StepPlan(caches)
ks = [torch.randn(2, 2, 128, device="cuda").to(torch.bfloat16) for _ in range(3)]
qs = [torch.randn(2, 8, 1, 128, device="cuda").to(torch.bfloat16) for _ in range(3)]
os_ = [torch.empty(2, 8, 1, 128, device="cuda") for _ in range(3)]
for n in range(1, 40):
    bmc.bmc_decode_step(plan, plan.ptrs(ks), plan.ptrs(ks), plan.ptrs(qs), plan.ptrs(os_), n)
torch.cuda.synchronize()
for c in caches:
    c.close()
# multi-layer step
caches = [bmc.KVCache(1, 2, 2, 128, 8, 32, dtype="bf16") for _ in range(3)]
plan = bmc.StepPlan(caches)
ks = [torch.randn(1, 2, 128, device="cuda").to(torch.bfloat16) for _ in range(3)]
qs = [torch.randn(1, 2, 1, 128, device="cuda").to(torch.bfloat16) for _ in range(3)]
os_ = [torch.empty(1, 2, 1, 128, device="cuda") for _ in range(3)]
for n in range(1, 20):
    bmc.bmc_decode_step(plan, plan.ptrs(ks), plan.ptrs(ks), plan.ptrs(qs), plan.ptrs(os_), n)
torch.cuda.synchronize()
for c in caches:
    c.close()
# copy-on-read growth in the CUDA-core kernel (path 1) over a multi-layer step
caches = [bmc.KVCache(1, 2, 2, 128, 8, 32, dtype="bf16") for _ in range(3)]
for c in caches:
    c.set_option(bmc.BMC_OPT_ATTN_PATH, 1)
plan = bmc.StepPlan(caches)
for n in range(1, 20):
    bmc.bmc_decode_step(plan, plan.ptrs(ks), plan.ptrs(ks), plan.ptrs(qs), plan.ptrs(os_), n)
torch.cuda.synchronize()
for c in caches:
    c.close()
# speculative step (G = 8, k = 8: M up to 72) with copy-on-read growth and
# bmc_commit_step; then 4 softmax column groups (M = 32)
for groups, Hq, k in ((0, 16, 8), (4, 8, 3)):
    caches = [bmc.KVCache(1, 2, Hq, 128, 16, 64, dtype="bf16") for _ in range(2)]
    for c in caches:
        c.set_option(bmc.BMC_OPT_TCK_GROUPS, groups)
    plan = bmc.StepPlan(caches)
    kn = [torch.randn(1, 2, 128, device="cuda").to(torch.bfloat16) for _ in range(2)]
    kd = [torch.randn(1, 2, k, 128, device="cuda").to(torch.bfloat16) for _ in range(2)]
    it = 0
    while max(caches[0].valid()) < 64 - 1 - k:
        kad = bmc.bmc_admissible(caches[0].h, k)
        q = [torch.randn(1, Hq, 1 + kad, 128, device="cuda").to(torch.bfloat16) for _ in range(2)]
        o = [torch.empty(1, Hq, 1 + kad, 128, device="cuda") for _ in range(2)]
        bmc.bmc_spec_step(plan, plan.ptrs(kn), plan.ptrs(kn), plan.ptrs(kd), plan.ptrs(kd), k,
                          plan.ptrs(q), plan.ptrs(o))
        if kad:
            bmc.bmc_commit_step(plan, [it % (kad + 1)])
        torch.cuda.synchronize()
        it += 1
    for c in caches:
        c.close()
# round 2: the fused token-tree step (bmc_spec_step_tree + bmc_commit_path_step,
# 34 layers = two verify launches, k = 9 tree) in the two-ended growth region
# (LIFO chunk moves, copy-on-read growth), checked against per-layer oracles
from harness import Model  # noqa: E402
bmc.bmc_region_reserve(-1, 64 << 20)
m = Model(34, 2, 1, 4, 128, 16, 64, seed=9, options=((bmc.BMC_OPT_ARENA, 2),))
parent = [-1, 0, 0, 1, 1, 2, 3, 3, 5]
it = 0
while m.orc[0].stats()["valid_max"] < 50:
    k_adm = m.spec_step_tree(9, parent, check=(it % 3 == 0))
    acc = [x for x in (0, 1, 3, 6) if x < k_adm]
    m.commit_path_step([acc[: it % 4], acc[: (it + 2) % 4]])
    it += 1
m.check_state()
m.close()
torch.cuda.synchronize()
bmc.bmc_region_reserve(-1, 0)
print("sanitize target ok")
