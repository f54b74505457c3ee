"""Where a 7B-shaped generation (32 layers, B=16, 0 -> 4096, r=128) spends
its time: host time of each bmc_decode_step call and GPU time between events,
growth steps vs the other steps, for three generations in a row (the first
one fills the stream-ordered pool)."""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

from paper_2511_12031_b200 import bmc  # noqa: E402

L, B, H, D, N, r = 32, 16, 32, 128, 4096, 128
HQ = H
if "--l3" in sys.argv:      # BASELINE configs[3]: Llama-3-8B GQA, B=64, 0 -> 8192
    B, H, HQ, N = 64, 8, 32, 8192
ARENA = 0 if "--vmm" in sys.argv else 1   # BMC_OPT_ARENA: 0 VMM slots (premapped), 1 pool
if "--region" in sys.argv:                 # 2: two-ended growth region of twice the final cache
    ARENA = 2
    bmc.load()
    bmc.bmc_region_reserve(0, 2 * (2 * B * H * N * D * 2) * L + (256 << 20))
if "--reserve" in sys.argv:                # map the peak footprint into the pool up front
    bmc.load()
    bmc.bmc_pool_reserve(0, 2 * B * H * N * D * 2 * (L + L))
k = [torch.randn(B, H, D, device="cuda").to(torch.bfloat16) for _ in range(L)]
q = [torch.randn(B, HQ, 1, D, device="cuda").to(torch.bfloat16) for _ in range(L)]
o = [torch.empty(B, HQ, 1, D, device="cuda") for _ in range(L)]


def gen(tag):
    hs = [bmc.KVCache(B, H, HQ, D, r, N, dtype="bf16") for _ in range(L)]
    for h in hs:
        h.set_option(bmc.BMC_OPT_ARENA, ARENA)
    plan = bmc.StepPlan(hs)
    K, Q, O = plan.ptrs(k), plan.ptrs(q), plan.ptrs(o)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(N + 1)]
    host = [0.0] * (N + 1)
    T0 = time.perf_counter()
    ev[0].record()
    for n in range(1, N + 1):
        t0 = time.perf_counter()
        bmc.bmc_decode_step(plan, K, K, Q, O, n)
        host[n] = time.perf_counter() - t0
        ev[n].record()
    torch.cuda.synchronize()
    T1 = time.perf_counter()
    g = [ev[n - 1].elapsed_time(ev[n]) for n in range(1, N + 1)]
    grow = [n for n in range(2, N + 1) if (n - 1) % r == 0]
    gs = sum(g[n - 1] for n in grow)
    hg = sum(host[n] for n in grow) * 1e3
    gb = sum(2 * B * H * D * 2 * L * ((n - 1) + (n - 1 + r)) for n in grow) / 1e9
    print(f"{tag}: growth launches {gb / (gs / 1e3) :.0f} GB/s algorithmic (incl. host gaps)")
    print(f"{tag}: wall {1e3 * (T1 - T0):.0f} ms, gpu {sum(g):.0f} ms; {len(grow)} growth steps: "
          f"gpu {gs:.0f} ms, host {hg:.0f} ms; other steps: host {1e3 * sum(host) - hg:.0f} ms; "
          f"max growth host {max(host[n] for n in grow) * 1e3:.1f} ms", flush=True)
    prof = bmc.bmc_host_profile(reset=True)
    print("   host ms (calls):", {k: (round(v[0], 1), v[1]) for k, v in prof.items()}, flush=True)
    for h in hs:
        h.close()


print("arena:", {0: "vmm (helper-thread premap)", 1: "pool", 2: "two-ended region"}[ARENA])
for i in range(3):
    gen(f"gen{i}")
