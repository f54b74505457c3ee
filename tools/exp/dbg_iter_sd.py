"""Debug: ITERATIVE + SD at the 7B-SD shape, per-check errors vs the oracle."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import oracle as O
from paper_2511_12031_b200 import bmc, synth
policy = sys.argv[1] if len(sys.argv) > 1 else "iterative"
path = int(sys.argv[2]) if len(sys.argv) > 2 else 0
N = int(sys.argv[3]) if len(sys.argv) > 3 else 4096
B, H, D, k = 32, 32, 128, 4
dev = torch.device("cuda")
c = bmc.KVCache(B, H, H, D, 1 if policy != "bmc" else 64, N, dtype="bf16", policy=policy)
c.set_option(bmc.BMC_OPT_ATTN_PATH, path)
plan = bmc.StepPlan([c])
g = torch.Generator(device=dev); g.manual_seed(41)
units = [(0, 0), (31, 31), (9, 20)]
hist = {u: [] for u in units}
it = 0
while max(c.valid()) < N - 1:
    kk = min(k, N - max(c.valid()) - 1)
    k_adm = bmc.bmc_admissible(c.h, kk); t = 1 + k_adm
    kn = torch.randn(B, H, D, generator=g, device=dev).to(torch.bfloat16)
    vn = torch.randn(B, H, D, generator=g, device=dev).to(torch.bfloat16)
    kd = torch.randn(B, H, max(kk, 1), D, generator=g, device=dev).to(torch.bfloat16)
    vd = torch.randn(B, H, max(kk, 1), D, generator=g, device=dev).to(torch.bfloat16)
    q = torch.randn(B, H, t, D, generator=g, device=dev).to(torch.bfloat16)
    o = torch.empty(B, H, t, D, device=dev)
    v0 = c.valid()
    bmc.bmc_spec_step(plan, plan.ptrs([kn]), plan.ptrs([vn]), plan.ptrs([kd]), plan.ptrs([vd]), kk,
                      plan.ptrs([q]), plan.ptrs([o]))
    cap = c.stats()["capacity"]
    m = synth.acceptance(23, it, B, k_adm)
    sample = it % 150 == 0 or max(c.valid()) > N - 10
    for (b, h) in units:
        hist[(b, h)].append((kn[b, h].cpu(), vn[b, h].cpu(), kd[b, h, :k_adm].cpu(), vd[b, h, :k_adm].cpu(),
                             q[b, h].cpu() if sample else None, o[b, h].cpu().numpy() if sample else None,
                             m[b], it, v0[b], cap))
    if k_adm:
        bmc.bmc_commit_step(plan, m)
    it += 1
for (b, h), ops in hist.items():
    orc = O.Oracle(1, 1, 1, D, 1, N, dtype=O.BF16, policy=O.POLICY_UPFRONT)
    for (kn_, vn_, kd_, vd_, q_, o_, mb, it_, v0_, cap_) in ops:
        orc.append(kn_.reshape(1, 1, D), vn_.reshape(1, 1, D))
        ka = kd_.shape[0]
        if ka:
            orc.spec_write(kd_.reshape(1, 1, ka, D).contiguous(), vd_.reshape(1, 1, ka, D).contiguous(), ka)
        if q_ is not None:
            ref = orc.sdpa(q_.reshape(1, 1, 1 + ka, D).contiguous(), -1)
            d = np.abs(o_.reshape(ref.shape) - ref)
            i = np.unravel_index(d.argmax(), d.shape)
            print(f"unit {b},{h} it {it_} valid {v0_} cap {cap_} k_adm {ka} err {d.max():.2e} at tau {i[2]} dim {i[3]} o {o_.reshape(ref.shape)[i]:.5f} ref {ref[i]:.5f} |ref|max {np.abs(ref).max():.3f}")
        if ka:
            orc.commit(min(mb, ka))
    orc.close()
