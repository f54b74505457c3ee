"""Token-tree speculation vs the number of allocations T (the paper's E8,
P:L1102-1122, and E21), synthetic, on B200: full generations
0 -> N through bench.py's token-tree mode (append, spec_write_tree of the
k-node tree, verify SDPA, commit_path of the accepted chain) for r = N / T,
latency normalised to T = 1 (one allocation: BMC with r = N, i.e. upfront).
Prints one JSON object with the paper's normalised latencies beside ours
(the paper's are CPU / MI210 numbers: context, not targets)."""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import bench  # noqa: E402
from sweep import run_point  # noqa: E402
from paper_2511_12031_b200 import bmc  # noqa: E402

PAPER = {
    "7b-tree": {"source": "P:L1115-1118 (Table tab:number_of_allocations_latency, Genoa CPU)",
                "T": [1, 2, 4, 8, 16, 128, 256, 512, 1024],
                "norm": [1.00, 0.56, 0.54, 0.45, 0.46, 0.47, 0.64, 0.83, 2.04]},
    "opt13b-tree": {"source": "P:L1710-1713 (Table tab:SpecDec_latency, MI210)",
                    "T": [1, 2, 4, 8, 16, 32, 64, 128, 256],
                    "norm": [1.00, 0.65, 0.55, 0.509, 0.501, 0.503, 0.52, 0.57, 0.74]},
}
PAPER["7b-tree-b32"] = PAPER["7b-tree"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="7b-tree", choices=sorted(PAPER))
    ap.add_argument("--reps", type=int, default=1)
    args = ap.parse_args()
    cfg = dict(bench.CONFIGS[args.config])
    bmc.load()
    pts = []
    for T in PAPER[args.config]["T"]:
        r = cfg["N"] // T
        p = run_point(cfg, "bmc", r, reps=args.reps)
        p["T"] = T
        pts.append(p)
        print(json.dumps(p), file=sys.stderr, flush=True)
    base = pts[0]["ms_per_generation"]
    for p in pts:
        p["norm_latency"] = p["ms_per_generation"] / base
    best = min(pts, key=lambda p: p["ms_per_generation"])
    print(json.dumps({"config": cfg["workload"], "tree": {"k": cfg["k"], "m": cfg["m"]},
                      "points": pts, "best_T": best["T"],
                      "norm_latency_row": [round(p["norm_latency"], 3) for p in pts],
                      "paper": PAPER[args.config]}))


if __name__ == "__main__":
    main()
