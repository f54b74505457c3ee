"""Per-kernel microbenchmarks through the C ABI (CUDA events, warm, L2-cold
inputs): decode attention at fixed capacity, the realloc copy, and the host
cost of an append+sdpa layer-step."""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2511_12031_b200 import bmc  # noqa: E402


def attn_at(B, H_kv, H_q, D, cap, t=1, reps=50, dtype="bf16", ctas=0, layers=8, path=0,
            groups=0, prefetch=-1):
    """SDPA over `layers` independent handles filled to `cap` rows (upfront
    policy so the buffer is exactly cap rows), round-robin so each launch reads
    an L2-cold cache."""
    eb = 2 if dtype == "bf16" else 4
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    hs = []
    for _ in range(layers):
        h = bmc.KVCache(B, H_kv, H_q, D, cap, cap, dtype=dtype, policy="upfront")
        if ctas:
            h.set_option(bmc.BMC_OPT_ATTN_CTAS, ctas)
        h.set_option(bmc.BMC_OPT_ATTN_PATH, path)
        if groups:
            h.set_option(bmc.BMC_OPT_TCK_GROUPS, groups)
        if prefetch >= 0:
            h.set_option(bmc.BMC_OPT_TCK_PREFETCH, prefetch)
        hs.append(h)
    k = torch.randn(B, H_kv, D, device="cuda").to(tdt)
    for h in hs:
        for _ in range(cap - (t - 1)):
            h.append(k, k)
        if t > 1:
            kd = torch.randn(B, H_kv, t - 1, D, device="cuda").to(tdt)
            h.spec_write(kd, kd, t - 1)
    q = torch.randn(B, H_q, t, D, device="cuda").to(tdt)
    o = torch.empty(B, H_q, t, D, device="cuda")
    n = cap - (t - 1)
    for i in range(layers):
        hs[i].sdpa(q, n, o)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(reps):
        hs[i % layers].sdpa(q, n, o)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    by = 2.0 * B * H_kv * cap * D * eb + B * H_q * t * D * (eb + 4)
    for h in hs:
        h.close()
    return {"cap": cap, "t": t, "M": (H_q // H_kv) * t, "path": path, "groups": groups,
            "us": ms * 1e3,
            "GBps": by / ms / 1e6}


def copy_at(B, H_kv, D, cap_old, r, reps=20, arena=0):
    """Realloc growth cap_old -> cap_old + r (BMC append at a full cache)."""
    res = []
    for _ in range(reps):
        h = bmc.KVCache(B, H_kv, H_kv, D, cap_old, cap_old + r, dtype="bf16", policy="bmc")
        h.set_option(bmc.BMC_OPT_ARENA, arena)
        k = torch.zeros(B, H_kv, D, device="cuda", dtype=torch.bfloat16)
        for _ in range(cap_old):
            h.append(k, k)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        h.append(k, k)             # growth: map + copy + zero + row write
        e1.record()
        torch.cuda.synchronize()
        res.append(e0.elapsed_time(e1))
        h.close()
    ms = sorted(res)[len(res) // 2]
    by = 2.0 * B * H_kv * D * 2 * (cap_old + cap_old + r)
    return {"cap_old": cap_old, "r": r, "arena": arena, "us": ms * 1e3, "GBps": by / ms / 1e6}


def host_cost_step(layers=32, steps=12):
    """Same through bmc_decode_step (one C call per token for all layers)."""
    hs = [bmc.KVCache(1, 1, 1, 128, 16, 16, dtype="bf16") for _ in range(layers)]
    plan = bmc.StepPlan(hs)
    k = [torch.zeros(1, 1, 128, device="cuda", dtype=torch.bfloat16) for _ in range(layers)]
    q = [torch.zeros(1, 1, 1, 128, device="cuda", dtype=torch.bfloat16) for _ in range(layers)]
    o = [torch.empty(1, 1, 1, 128, device="cuda") for _ in range(layers)]
    K, Q, O = plan.ptrs(k), plan.ptrs(q), plan.ptrs(o)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for n in range(1, steps + 1):
        bmc.bmc_decode_step(plan, K, K, Q, O, n)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    for h in hs:
        h.close()
    return {"step_host_us_per_layer_step": (t1 - t0) / (layers * steps) * 1e6,
            "step_wall_us_per_layer_step": (t2 - t0) / (layers * steps) * 1e6}


def host_cost(layers=32, steps=12):
    """Host time per layer-step (append + sdpa) with a tiny cache (GPU idle)."""
    hs = [bmc.KVCache(1, 1, 1, 128, 16, 16, dtype="bf16") for _ in range(layers)]
    k = torch.zeros(1, 1, 128, device="cuda", dtype=torch.bfloat16)
    q = torch.zeros(1, 1, 1, 128, device="cuda", dtype=torch.bfloat16)
    o = torch.empty(1, 1, 1, 128, device="cuda")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for n in range(1, steps + 1):
        for h in hs:
            h.append(k, k)
            h.sdpa(q, n, o)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    for h in hs:
        h.close()
    return {"host_us_per_layer_step": (t1 - t0) / (layers * steps) * 1e6,
            "wall_us_per_layer_step": (t2 - t0) / (layers * steps) * 1e6}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--what", default="all")
    args = ap.parse_args()
    bmc.load()
    out = {}
    if args.what in ("all", "attn"):
        out["attn_7b"] = [attn_at(16, 32, 32, 128, c) for c in (64, 256, 1024, 2048, 4096)]
        out["attn_l3"] = [attn_at(64, 8, 32, 128, c) for c in (1024, 8192)]
        out["attn_sd5"] = [attn_at(32, 32, 32, 128, c, t=5) for c in (1024, 4096)]
    if args.what in ("all", "tc"):
        # verify shapes: 70B (G=8, t=1+k), L3-8B GQA (G=4), 7B-SD (t=5): CUDA cores vs tcgen05
        out["verify"] = []
        for (B, Hk, Hq, cap, t) in [(8, 8, 64, 8192, 9), (8, 8, 64, 8192, 1),
                                    (64, 8, 32, 4096, 1), (32, 32, 32, 2048, 5),
                                    (8, 8, 64, 8192, 4), (8, 8, 64, 8192, 8)]:
            for pa in ((2, 3, 4) if (Hq // Hk) * t > 64 else (1, 2, 3)):
                print("config", B, Hk, Hq, cap, t, pa, file=sys.stderr, flush=True)
                out["verify"].append(attn_at(B, Hk, Hq, 128, cap, t=t, path=pa, reps=20,
                                             layers=4))
                print(out["verify"][-1], file=sys.stderr, flush=True)
    if args.what == "tc72":           # ncu target: 70B-shaped verify, M = 72
        out["verify"] = [attn_at(8, 8, 64, 128, 8192, t=9, path=2, reps=6, layers=2)]
    if args.what == "tc8":            # ncu target: 70B-shaped decode on tensor cores, M = 8
        out["verify"] = [attn_at(8, 8, 64, 128, 8192, t=1, path=2, reps=6, layers=2)]
    if args.what == "tcsweep":        # keys-on-lanes kernel: 70B shape, M = 8 t
        out["tck"] = [attn_at(8, 8, 64, 128, cap, t=t, path=4, reps=8, layers=4)
                      for cap in (8192, 32768) for t in (1, 2, 4, 5, 8, 9)]
    if args.what == "tc72ab":         # M = 72: auto vs forced 2 groups (A/B harness)
        out["tck"] = [attn_at(8, 8, 64, 128, cap, t=9, path=4, reps=10, layers=4, groups=g)
                      for cap in (8192, 32768) for g in (0, 2, 0, 2)]
    if args.what == "tcgroups":       # softmax column groups 2 vs 4, 70B shape
        out["tck"] = [attn_at(8, 8, 64, 128, cap, t=t, path=4, reps=8, layers=4, groups=g)
                      for cap in (8192, 32768) for t in (1, 2, 4, 6, 8, 9) for g in (2, 4)]
    if args.what == "tcrepro":
        out["verify"] = [attn_at(8, 8, 64, 128, 1024, t=9, path=1, reps=4, layers=2)]
    if args.what == "attn4096":       # ncu target: 7B shape at full context
        out["attn_7b"] = [attn_at(16, 32, 32, 128, 4096, reps=10)]
    if args.what in ("all", "copy"):
        out["copy_7b"] = [copy_at(16, 32, 128, c, 64, arena=a) for a in (0, 1)
                          for c in (1024, 4032)]
    if args.what in ("all", "host"):
        out["host"] = host_cost()
        out["host_step"] = host_cost_step()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
