"""70B-SD (k=8, B=8, 80 layers) at N_max 8192: wall vs device time and the
library's host-time categories per r (the r=128 point ran 25% slower than
r=64 / r=256 in two sweeps)."""
import json
import os
import sys
import time
sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tools"))
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
for r in [int(x) for x in sys.argv[1].split(",")]:
    torch.cuda.synchronize()
    bmc.bmc_region_reserve(0, 0)
    kind, arena, _ = bench.growth_memory(cfg, B, dev, "auto", margin=4 << 30)
    gen = bench.Generation(cfg, B, r, "bmc", ring, outs, stream, 0)
    gen.arena = kind
    gen.run()
    torch.cuda.synchronize()
    bmc.bmc_host_profile(reset=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(stream)
    tok = gen.run()[0]
    e1.record(stream)
    t_host = time.perf_counter() - t0
    torch.cuda.synchronize()
    t_all = time.perf_counter() - t0
    prof = bmc.bmc_host_profile(reset=True)
    print(json.dumps({"r": r, "tok_s": tok / (e0.elapsed_time(e1) / 1e3), "gpu_ms": e0.elapsed_time(e1),
                      "host_enqueue_ms": 1e3 * t_host, "wall_ms": 1e3 * t_all,
                      "host_prof_ms": {k: round(v[0], 1) for k, v in prof.items()}}), flush=True)
