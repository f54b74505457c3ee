"""Allocation-policy sweep on B200 (the paper's E3/E4 experiments, synthetic):
full decodes 0 -> N_max of the Llama-2-7B-shaped workload (BASELINE configs[1])
under ITERATIVE (r = 1 cadence, exact-size reallocation), UPFRONT (r = N_max)
and BMC for r in {8, 32, 64, 128, 512}, same kernels, same inputs.

Prints one JSON object: tokens/s per point, the ledger (allocations, copied
bytes, SDPA bytes) and the paper's reference ratios for context
(P:L600 upfront vs iterative 1.9x; P:L616 BMC(T=16) vs iterative/upfront
3.25x/1.34x; P:L1103-1122 SD latency vs T; all CPU/MI210)."""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2511_12031_b200 import bmc  # noqa: E402


def run_point(cfg, policy, r, reps=1, skip_padding=False):
    """One sweep point.  Each point sets up its growth memory as bench.py does
    (the two-ended growth region when twice the final cache fits, else a
    trimmed pool with the peak footprint reserved), so no point pays or
    inherits another's allocator state."""
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev)
    B = cfg["B"]
    torch.cuda.synchronize()
    bmc.bmc_region_reserve(0, 0)
    bmc.bmc_pool_trim(0)
    ring = bench.make_ring(cfg, B, dev)
    t_all = 1 + cfg["k"]
    outs = {t: [torch.empty(B, cfg["H_q"], t, cfg["D"], dtype=torch.float32, device=dev)
                for _ in range(cfg["L"])] for t in range(1, t_all + 1)}
    kind, arena, _ = bench.growth_memory(cfg, B, dev, "auto", margin=4 << 30, policy=policy)
    gen = bench.Generation(cfg, B, r, policy, ring, outs, stream, 0)
    gen.arena = kind
    gen.skip_padding = skip_padding
    gen.run()                                   # warm-up
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    tok = 0
    for _ in range(reps):
        tok += gen.run()[0]
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    return {"policy": policy + ("+length-aware" if skip_padding else ""), "r": r, "arena": arena, "T": -(-cfg["N"] // r) if policy == "bmc" else None,
            "tokens_per_s": tok / (ms / 1e3), "ms_per_generation": ms / reps}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="7b")
    ap.add_argument("--rs", default="8,32,64,128,512")
    ap.add_argument("--baselines", default="iterative,upfront")
    ap.add_argument("--n-max", type=int, default=0, help="override N_max (quick runs)")
    ap.add_argument("--ablation", action="store_true",
                    help="also run the length-aware ablation (SURVEY NEXT-4)")
    args = ap.parse_args()
    cfg = dict(bench.CONFIGS[args.config])
    if args.n_max:
        cfg["N"] = args.n_max
        cfg["workload"] += f" [N_max overridden to {args.n_max}]"
    bmc.load()
    pts = []
    # BMC points first; the iterative baseline (one pool allocation per layer
    # and token) runs last so its allocator churn cannot affect the others
    for r in [int(x) for x in args.rs.split(",") if x]:
        pts.append(run_point(cfg, "bmc", r))
        print(json.dumps(pts[-1]), file=sys.stderr, flush=True)
    for pol in sorted([p for p in args.baselines.split(",") if p], key=lambda x: x == "iterative"):
        r = cfg["N"] if pol == "upfront" else 1
        pts.append(run_point(cfg, pol, r))
        print(json.dumps(pts[-1]), file=sys.stderr, flush=True)
    if args.ablation:
        # what the padded-GEMV contract costs: the same runs streaming only
        # visible rows (UPFRONT + length-aware = a contiguous exact-prefix kernel)
        for pol, r in (("bmc", 128), ("upfront", cfg["N"])):
            pts.append(run_point(cfg, pol, r, skip_padding=True))
            print(json.dumps(pts[-1]), file=sys.stderr, flush=True)
    best = max((p for p in pts if p["policy"] == "bmc"), key=lambda p: p["tokens_per_s"])
    out = {"config": cfg["workload"], "points": pts, "best_bmc": best}
    it = next((p for p in pts if p["policy"] == "iterative"), None)
    up = next((p for p in pts if p["policy"] == "upfront"), None)
    if it and up:
        out["speedup_best_bmc_vs_iterative"] = best["tokens_per_s"] / it["tokens_per_s"]
        out["speedup_best_bmc_vs_upfront"] = best["tokens_per_s"] / up["tokens_per_s"]
        out["speedup_upfront_vs_iterative"] = up["tokens_per_s"] / it["tokens_per_s"]
    out["paper_context"] = {
        "upfront_vs_iterative_attention_block": "1.9x lower latency (Genoa CPU, P:L600)",
        "bmc_T16_vs_iterative_upfront": "3.25x / 1.34x (Genoa CPU, OPT-13B B=8 N=1024, P:L616)",
        "bandwidth_model_expectation_B200": "BMC ~2.9x iterative, ~1.9x upfront (SURVEY 8(d))"}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
