"""Per-iteration device time of the fused 70B-SD verify step vs capacity for
r = 128 and r = 256 (N_max 8192): which caps are slow?"""
import json
import os
import sys
from collections import defaultdict
sys.path.insert(0, os.getcwd())
import torch  # noqa: E402
import bench  # noqa: E402
from paper_2511_12031_b200 import bmc  # noqa: E402
bmc.load()
cfg = dict(bench.CONFIGS["70b-long"])
cfg["N"] = 8192
dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream(dev)
B = cfg["B"]
ring = bench.make_ring(cfg, B, dev)
outs = {t: [torch.empty(B, cfg["H_q"], t, cfg["D"], dtype=torch.float32, device=dev)
            for _ in range(cfg["L"])] for t in range(1, 2 + cfg["k"])}
res = {}
for r in (128, 256):
    torch.cuda.synchronize()
    bmc.bmc_region_reserve(0, 0)
    kind, arena, _ = bench.growth_memory(cfg, B, dev, "auto", margin=4 << 30)
    gen = bench.Generation(cfg, B, r, "bmc", ring, outs, stream, 0)
    gen.arena = kind
    gen.run()
    ev = [[torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True), None]
          for _ in range(3000)]
    gev = [[torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True), None]
           for _ in range(200)]
    gen.run(1, ev, gev)
    torch.cuda.synchronize()
    g = [(x[2]["cap_old"], x[2]["capacity"], round(x[0].elapsed_time(x[1]), 3)) for x in gev if x[2]]
    print("r", r, "growth steps", len(g), "total ms", round(sum(x[2] for x in g), 1), g[:6], g[-6:], flush=True)
    by = defaultdict(list)
    for e0, e1, st in ev:
        if st is None:
            continue
        by[(st["capacity"], 1 + st["staged"])].append(e0.elapsed_time(e1))
    res[r] = {f"{c}/{t}": (len(v), round(sum(v) / len(v), 3)) for (c, t), v in sorted(by.items())}
caps = sorted({k for r in res for k in res[r]}, key=lambda s: tuple(map(int, s.split("/"))))
for c in caps:
    a, b = res[128].get(c), res[256].get(c)
    print(c, "r128", a, "r256", b)
