"""Validation of the r advisor on B200 (the paper's E5-E7 /
E20 model validations):
measured r sweeps at several context lengths and shapes, against the
advisor's pick from measured bandwidths.

Advisor (paper_2511_12031_b200/advisor.py, byte form): a separate realloc
copy gives r* = sqrt(2 N BW_read / BW_copy); with copy-on-read growth (the
default) the growth adds only the write of the new buffer, r* =
sqrt(N BW_read / BW_write); T = N / r* is rounded to a power of two.
BW_read / BW_write are measured here: the decode attention kernel's achieved
read bandwidth and the copy-on-read growth launches' achieved bandwidth."""
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
from paper_2511_12031_b200 import advisor, bmc  # noqa: E402

CASES = [  # (name, config, N, k for SD or None, r values)
    ("7B MHA", "7b", 512, [8, 16, 32, 64, 128, 512]),
    ("7B MHA", "7b", 2048, [16, 32, 64, 128, 256, 2048]),
    ("7B MHA", "7b", 8192, [32, 64, 128, 256, 512, 8192]),
    ("L3-8B GQA", "l3-8b", 1024, [16, 32, 64, 128, 256, 1024]),
    ("L3-8B GQA", "l3-8b", 4096, [32, 64, 128, 256, 512, 4096]),
    ("7B-SD k=4", "7b-sd", 4096, [16, 32, 64, 128, 256, 4096]),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bw-read", type=float, default=7.0e12,
                    help="decode attention read bandwidth (bench roofline achieved)")
    ap.add_argument("--bw-write", type=float, default=5.47e12,
                    help="copy-on-read growth launch bandwidth (bench growth sub-record)")
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    bmc.load()
    out = []
    for name, cname, N, rs in CASES:
        if args.only and args.only not in name:
            continue
        cfg = dict(bench.CONFIGS[cname])
        cfg["N"] = N
        # short generations are repeated (>= ~8K tokens per timed point) so a
        # point is not one clock ramp
        reps = max(1, 8192 // N)
        pts = [run_point(cfg, "bmc", r, reps=reps) for r in rs]
        best = max(pts, key=lambda p: p["tokens_per_s"])
        m = 1.0
        if cfg["k"]:   # mean tokens per speculative iteration E[m+1] (P_ACCEPT = 0.7)
            p = bench.P_ACCEPT
            m = sum(p ** i for i in range(cfg["k"] + 1))
        # the paper's SD form scales T with sqrt(N/m): per token
        # the growth is amortised over m tokens while the verify reads per iteration
        n_eff = N / m if cfg["k"] else N
        r_cor = advisor.advise_r(N, args.bw_read, args.bw_write, copy_on_read=True,
                                 tokens_per_iter=m)
        r_sep = advisor.advise_r(N, args.bw_read, args.bw_write)
        at = {p["r"]: p["tokens_per_s"] for p in pts}
        row = {"case": name, "N": N, "points": [(p["r"], round(p["tokens_per_s"], 1)) for p in pts],
               "best_r": best["r"], "advised_r_copy_on_read": r_cor,
               "advised_r_separate_copy": r_sep,
               "regret_at_advised": (1 - at[r_cor] / best["tokens_per_s"]) if r_cor in at else None,
               "tokens_per_iteration": m, "n_eff": n_eff}
        out.append(row)
        print(json.dumps(row), flush=True)
    print(json.dumps({"bw_read": args.bw_read, "bw_write": args.bw_write, "cases": out}))


if __name__ == "__main__":
    main()
